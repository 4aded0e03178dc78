// Multi-rank sharding of static non-uniform sims.
//
// Partition: the leaves are stored in Morton order of their SW fine corner, so
// rank r owns the contiguous range [floor(n r / R), floor(n (r+1) / R)) — a
// space-filling-curve partition with compact pieces.  A rank keeps every
// global segment with at least one owned leaf; the remote leaves of those
// segments are its halo.  A cut segment is evaluated by both ranks from
// identical inputs (its two leaves' states), so both see the same bits and no
// flux is communicated.
//
// Per DG2 step: two halo exchanges (the state each RK stage gathers: U after
// the friction head, U* after stage 1), 72 B per halo leaf, as one grouped
// ncclSend / ncclRecv per peer that lands directly in the halo slots; then one
// ncclAllReduce(min) over the 64 B reduction slots (the CFL minimum, the
// complemented ACC depth maximum and the first non-finite key are all mins,
// and min is exact, so dt is bit-identical for any rank count).  FV1 needs one
// exchange, ACC one (h at the step start).  Everything is enqueued on the
// library stream, so a whole step — NCCL calls included — is captured in the
// sim's CUDA graph.
//
// Transports: NCCL (one process per GPU; libnccl is loaded at run time, the
// copy already in the process when there is one, e.g. torch's), a local
// group (all ranks as shards of one process on one device, driven phase by
// phase by fm_group_run) — the single-GPU harness that checks the partition,
// halo and reduction logic bit-for-bit against the unsharded sim — or a host
// transport (one process per rank, any devices, the halo slices and the
// reduction slots staged through a POSIX shared-memory segment with a
// process-shared barrier): the library's own pack / halo-slot / reduction
// code across real process boundaries, on however many GPUs there are,
// including one (no kernel ever waits on another rank; only host threads do).
#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <string>

#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <type_traits>

#include <algorithm>
#include <cstring>
#include <numeric>

#include "fm_device.cuh"
#include "fm_sim.hpp"

namespace fmh {

// ---- the transport ------------------------------------------------------------

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*ErrorString)(ncclResult_t) = nullptr;
};

static const NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) {
    if (!api.h) throw Error(FM_ERR_CONFIG, "NCCL is not available (libnccl.so.2 not found)");
    return api;
  }
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process
  if (!h) {
    if (const char* p = std::getenv("FM_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
  }
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) throw Error(FM_ERR_CONFIG, "NCCL is not available (libnccl.so.2 not found)");
  auto sym = [&](const char* n) {
    void* f = dlsym(h, n);
    if (!f) throw Error(FM_ERR_CONFIG, std::string("NCCL symbol missing: ") + n);
    return f;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.ErrorString = reinterpret_cast<decltype(api.ErrorString)>(sym("ncclGetErrorString"));
  api.h = h;
  return api;
}

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(FM_ERR_CUDA, std::string("[nccl] ") + what + ": " + nccl().ErrorString(r));
}

enum CommKind { COMM_LOCAL = 0, COMM_NCCL = 1, COMM_HOST = 2 };

// Host transport: one shared-memory segment per partition.  Layout: the
// barrier header, the reduction area (nranks x 8 u64), then nranks x nranks
// slots (src, dst) of slot_bytes each for the halo slices.
struct ShmHeader {
  std::atomic<int> count;
  std::atomic<int> gen;
  int nranks;
  int pad;
};
constexpr size_t kShmReduce = 64;  // bytes per rank in the reduction area
// segment size: 32 MB by default (a container's /dev/shm is often 64 MB), or
// $FM_HOST_COMM_MB; each (src, dst) slot gets 1 / nranks^2 of it
static size_t shm_bytes() {
  const char* e = std::getenv("FM_HOST_COMM_MB");
  const long mb = e ? std::atol(e) : 32;
  return size_t(mb > 0 ? mb : 32) << 20;
}

struct Comm {
  int kind = COMM_LOCAL;
  int nranks = 1, rank = 0;
  ncclComm_t nc = nullptr;
  std::vector<Sim*> members;  // local group: the shard sim of each rank (or null)
  // host transport
  std::string shm_name;
  void* shm = nullptr;
  size_t shm_size = 0;
  size_t slot_bytes = 0;
  std::vector<double> stage;  // host staging of the packed send buffer
  ShmHeader* hdr() const { return static_cast<ShmHeader*>(shm); }
  unsigned char* reduce_area() const { return static_cast<unsigned char*>(shm) + 64; }
  unsigned char* slot(int src, int dst) const {
    return reduce_area() + kShmReduce * size_t(nranks) + (size_t(src) * nranks + dst) * slot_bytes;
  }
};

// Sense-counting barrier of the ranks' host threads over the segment.  A rank
// that waits longer than two minutes gives up (a peer died).
static void shm_barrier(Comm& c) {
  ShmHeader* h = c.hdr();
  const int g = h->gen.load(std::memory_order_acquire);
  if (h->count.fetch_add(1, std::memory_order_acq_rel) == c.nranks - 1) {
    h->count.store(0, std::memory_order_relaxed);
    h->gen.fetch_add(1, std::memory_order_acq_rel);
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  int spins = 0;
  while (h->gen.load(std::memory_order_acquire) == g) {
    if (++spins > 1000) {
      sched_yield();
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
        throw Error(FM_ERR_OTHER, "host transport: a peer rank did not reach the barrier");
    }
  }
}

Comm* comm_create_host(int nranks, int rank, const char* name) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(FM_ERR_CONFIG, "comm: bad rank / size");
  if (!name || name[0] != '/') throw Error(FM_ERR_CONFIG, "host comm: the name must start with '/'");
  auto c = std::make_unique<Comm>();
  c->kind = COMM_HOST;
  c->nranks = nranks;
  c->rank = rank;
  c->shm_name = name;
  const int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
  if (fd < 0) throw Error(FM_ERR_IO, std::string("host comm: shm_open failed for ") + name);
  const size_t bytes = shm_bytes();
  if (ftruncate(fd, off_t(bytes)) != 0) {
    close(fd);
    throw Error(FM_ERR_IO, "host comm: ftruncate failed");
  }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) throw Error(FM_ERR_IO, "host comm: mmap failed");
  c->shm = p;
  c->shm_size = bytes;
  c->slot_bytes = ((bytes - 64 - kShmReduce * nranks) / (size_t(nranks) * nranks)) & ~size_t(63);
  shm_barrier(*c);  // every rank has the segment mapped (a fresh one is zero-filled)
  return c.release();
}

static void host_allreduce_u64_min(Comm& c, unsigned long long* dev, int count) {
  if (count > int(kShmReduce / 8)) throw Error(FM_ERR_OTHER, "host comm: reduction too wide");
  unsigned long long v[8];
  FM_CUDA(cudaMemcpyAsync(v, dev, count * 8, cudaMemcpyDeviceToHost, stream()));
  FM_CUDA(cudaStreamSynchronize(stream()));
  std::memcpy(c.reduce_area() + kShmReduce * c.rank, v, count * 8);
  shm_barrier(c);
  for (int r = 0; r < c.nranks; ++r) {
    unsigned long long w[8];
    std::memcpy(w, c.reduce_area() + kShmReduce * r, count * 8);
    for (int q = 0; q < count; ++q) v[q] = std::min(v[q], w[q]);
  }
  shm_barrier(c);  // the area may be reused
  FM_CUDA(cudaMemcpyAsync(dev, v, count * 8, cudaMemcpyHostToDevice, stream()));
  FM_CUDA(cudaStreamSynchronize(stream()));
}

static double host_allreduce_sum(Comm& c, double x) {
  std::memcpy(c.reduce_area() + kShmReduce * c.rank, &x, 8);
  shm_barrier(c);
  double sum = 0.0;  // rank order: the same bits on every rank
  for (int r = 0; r < c.nranks; ++r) {
    double w;
    std::memcpy(&w, c.reduce_area() + kShmReduce * r, 8);
    sum += w;
  }
  shm_barrier(c);
  return sum;
}

Comm* comm_create_local(int nranks) {
  if (nranks < 1) throw Error(FM_ERR_CONFIG, "comm: nranks must be >= 1");
  auto c = std::make_unique<Comm>();
  c->kind = COMM_LOCAL;
  c->nranks = nranks;
  c->members.assign(nranks, nullptr);
  return c.release();
}

void comm_unique_id(uint8_t* out) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

Comm* comm_create_nccl(int nranks, int rank, const uint8_t* id) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(FM_ERR_CONFIG, "comm: bad rank / size");
  auto c = std::make_unique<Comm>();
  c->kind = COMM_NCCL;
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  nccl_check(nccl().CommInitRank(&c->nc, nranks, u, rank), "ncclCommInitRank");
  return c.release();
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->kind == COMM_NCCL && c->nc) nccl().CommDestroy(c->nc);
  if (c->kind == COMM_HOST && c->shm) {
    munmap(c->shm, c->shm_size);
    if (c->rank == 0) shm_unlink(c->shm_name.c_str());
  }
  for (Sim* s : c->members)
    if (s && s->shard) s->shard->comm = nullptr;
  delete c;
}

void comm_forget(Comm* c, Sim* s) {
  if (!c) return;
  for (auto& m : c->members)
    if (m == s) m = nullptr;
}

// ---- the partition plan (host) --------------------------------------------------

int64_t shard_first(int64_t n, int nranks, int r) {
  return int64_t((static_cast<__int128>(n) * r) / nranks);
}

static int owner_of(const std::vector<int64_t>& firsts, int64_t g) {
  // firsts has nranks + 1 entries, firsts[nranks] = n
  return int(std::upper_bound(firsts.begin(), firsts.end(), g) - firsts.begin()) - 1;
}

ShardPlan shard_plan(int64_t n, int64_t nseg, const int32_t* seg_l, const int32_t* seg_r, int nranks,
                     int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(FM_ERR_CONFIG, "shard plan: bad rank / size");
  if (n < nranks) throw Error(FM_ERR_CONFIG, "shard plan: fewer leaves than ranks");
  std::vector<int64_t> firsts(nranks + 1);
  for (int r = 0; r <= nranks; ++r) firsts[r] = shard_first(n, nranks, r);
  ShardPlan p;
  p.first = firsts[rank];
  p.count = firsts[rank + 1] - firsts[rank];
  p.send.assign(nranks, {});
  for (int64_t q = 0; q < nseg; ++q) {
    const int64_t a = seg_l[q], b = seg_r[q];
    if (a < 0 || b < 0 || a >= n || b >= n) throw Error(FM_ERR_STRUCTURE, "shard plan: bad segment");
    const int oa = owner_of(firsts, a), ob = owner_of(firsts, b);
    if (oa != rank && ob != rank) continue;
    p.segs.push_back(q);
    if (oa == rank && ob != rank) {
      p.halo.push_back(b);
      p.send[ob].push_back(a);
    } else if (ob == rank && oa != rank) {
      p.halo.push_back(a);
      p.send[oa].push_back(b);
    }
  }
  auto uniq = [](std::vector<int64_t>& v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  };
  uniq(p.halo);
  for (auto& v : p.send) uniq(v);
  // halo grouped by owner: ascending global ids are already grouped
  p.halo_owner.resize(p.halo.size());
  for (size_t k = 0; k < p.halo.size(); ++k) p.halo_owner[k] = owner_of(firsts, p.halo[k]);
  return p;
}

// ---- sharded sim construction -------------------------------------------------

namespace {

inline unsigned nblk(uint64_t n, int t) { return unsigned((n + t - 1) / t); }

__global__ void k_pack(const double* __restrict__ u, int w, const int32_t* __restrict__ idx, long long m,
                       double* __restrict__ buf) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= w * m) return;
  const long long k = t / w, q = t % w;
  buf[t] = u[w * (long long)idx[k] + q];
}

// Local group: min-combine the reduction slots of every shard into all of them.
__global__ void k_red_combine(DevRed* const* reds, int n) {
  const int f = threadIdx.x;  // 0..7: 2 slots x 4 fields
  if (f >= 8) return;
  unsigned long long m = ~0ull;
  for (int r = 0; r < n; ++r) m = min(m, reinterpret_cast<const unsigned long long*>(reds[r])[f]);
  for (int r = 0; r < n; ++r) reinterpret_cast<unsigned long long*>(reds[r])[f] = m;
}


}  // namespace

// One eager exchange + reduction right after construction: NCCL sets up its
// peer connections on first use, outside any graph capture.
static void shard_warmup(Sim& s) {
  shard_op(s, OP_EXCH_U);
  shard_op(s, OP_REDUCE);  // joins the exchange first
  FM_CUDA(cudaStreamSynchronize(stream()));
}

// The uniform raster shards into row bands: rank r owns the global rows
// [floor(ny r / R), floor(ny (r+1) / R)) (a contiguous range of the raster's
// own j-major cell order), stored first, then one ghost row south and one
// north where a neighbour band exists.  The exchange per stage is one row of
// 72 B cells each way; faces on a band edge are solved by both bands from the
// same inputs.
static Sim* uniform_shard(const fm_sim_desc* d, const fm_raster* dem, Comm* comm, int rank) {
  cudaStream_t st = stream();
  std::unique_ptr<Sim> G(sim_create(d, dem, nullptr));
  const int R = comm->nranks, nx = G->nx, nyg = G->ny;
  if (nyg < R) throw Error(FM_ERR_CONFIG, "shard: fewer raster rows than ranks");
  const int g0 = int(shard_first(nyg, R, rank)), g1 = int(shard_first(nyg, R, rank + 1));
  const int nyo = g1 - g0, hs = g0 > 0 ? 1 : 0, hn = g1 < nyg ? 1 : 0;
  auto S = std::make_unique<Sim>();
  Sim& s = *S;
  s.solver = G->solver;
  s.scheme = G->scheme;
  s.libm = G->libm;
  s.g = G->g;
  s.hdry = G->hdry;
  s.courant = G->courant;
  std::copy(G->bc, G->bc + 4, s.bc);
  s.uniform = true;
  s.L = 0;
  s.M = nx;
  s.N = nyo;
  s.R = G->R;
  s.x0 = G->x0;
  s.y0 = G->y0;
  s.p2 = G->p2;
  s.nx = nx;
  s.ny = nyo;
  s.gy0 = g0;
  s.nyg = nyg;
  s.ghost_s = hs;
  s.ghost_n = hn;
  s.ninflow = G->ninflow;
  s.hy_t = G->hy_t;
  s.hy_q = G->hy_q;
  s.region = G->region;
  s.rect = G->rect;
  s.manning = G->manning;
  s.hydro.alloc(1);
  FM_CUDA(cudaMemcpyAsync(s.hydro.p, G->hydro.p, sizeof(Hydro), cudaMemcpyDeviceToDevice, st));
  s.clk.alloc(2);
  s.red.alloc(2);
  s.n = int64_t(nx) * nyo;
  s.nseg = int64_t(nx + 1) * nyo + int64_t(nx) * (nyo + 1);
  // owned rows first, then the ghost rows: contiguous row copies on the device
  const size_t nt = size_t(nyo + hs + hn) * nx;
  auto rows = [&](auto& dst, const auto& src, int width) {
    using T = std::remove_pointer_t<decltype(src.p)>;
    dst.alloc(nt * width);
    const size_t rw = size_t(nx) * width * sizeof(T);
    FM_CUDA(cudaMemcpyAsync(dst.p, src.p + size_t(g0) * nx * width, rw * nyo, cudaMemcpyDeviceToDevice, st));
    if (hs)
      FM_CUDA(cudaMemcpyAsync(dst.p + size_t(nyo) * nx * width, src.p + size_t(g0 - 1) * nx * width, rw,
                              cudaMemcpyDeviceToDevice, st));
    if (hn)
      FM_CUDA(cudaMemcpyAsync(dst.p + size_t(nyo + hs) * nx * width, src.p + size_t(g1) * nx * width, rw,
                              cudaMemcpyDeviceToDevice, st));
  };
  rows(s.u, G->u, 9);
  s.us.alloc(9 * nt);
  FM_CUDA(cudaMemcpyAsync(s.us.p, s.u.p, 9 * nt * sizeof(double), cudaMemcpyDeviceToDevice, st));
  rows(s.z, G->z, 3);
  rows(s.nman, G->nman, 1);
  s.li.alloc(s.n);
  s.lj.alloc(s.n);
  FM_CUDA(cudaMemcpyAsync(s.li.p, G->li.p + size_t(g0) * nx, size_t(s.n) * sizeof(int32_t),
                          cudaMemcpyDeviceToDevice, st));
  FM_CUDA(cudaMemcpyAsync(s.lj.p, G->lj.p + size_t(g0) * nx, size_t(s.n) * sizeof(int32_t),
                          cudaMemcpyDeviceToDevice, st));
  if (s.scheme == FM_ACC) {
    s.aqx.alloc(size_t(nx + 1) * nyo);
    s.aqy.alloc(size_t(nx) * (nyo + 1));
    s.aqx.zero();
    s.aqy.zero();
  }
  auto sh = std::make_unique<Shard>();
  sh->comm = comm;
  sh->rank = rank;
  sh->nranks = R;
  sh->first = int64_t(g0) * nx;
  sh->n_global = int64_t(nyg) * nx;
  sh->n_halo = int64_t(hs + hn) * nx;
  std::vector<int32_t> sidx;
  if (hs) {  // row g0 to rank - 1, its row g0 - 1 into the south ghost
    sh->peers.push_back(rank - 1);
    sh->soff.push_back(int64_t(sidx.size()));
    sh->scnt.push_back(nx);
    for (int i = 0; i < nx; ++i) sidx.push_back(i);
    sh->hoff.push_back(0);
    sh->hcnt.push_back(nx);
  }
  if (hn) {  // row g1 - 1 to rank + 1, its row g1 into the north ghost
    sh->peers.push_back(rank + 1);
    sh->soff.push_back(int64_t(sidx.size()));
    sh->scnt.push_back(nx);
    for (int i = 0; i < nx; ++i) sidx.push_back(int32_t(int64_t(nyo - 1) * nx + i));
    sh->hoff.push_back(int64_t(hs) * nx);
    sh->hcnt.push_back(nx);
  }
  if (sidx.empty()) sidx.push_back(0);
  sh->send_idx.upload(sidx.data(), sidx.size());
  sh->send_buf.alloc(9 * sidx.size());
  s.shard = std::move(sh);
  if (comm->kind == COMM_LOCAL) comm->members[rank] = &s;
  G.reset();
  FM_CUDA(cudaStreamSynchronize(st));
  if (comm->kind == COMM_NCCL) shard_warmup(s);
  return S.release();
}

// ---- device-side shard construction ---------------------------------------
// The plan of shard_plan, built with flags + stream compactions over the
// global topology already on the device (no host round trip of the grid).
namespace {

constexpr int kMaxRanks = 64;
struct Owners {
  long long firsts[kMaxRanks + 1];
  int nranks;
};
__device__ __forceinline__ int owner_d(const Owners& o, long long g) {
  int r = 0;
  while (r + 1 < o.nranks && g >= o.firsts[r + 1]) ++r;
  return r;
}

// per segment: inner (both leaves owned), boundary (one owned); per boundary
// segment its remote leaf joins the halo and its owned leaf the peer's send list
__global__ void k_seg_class(long long nseg, const int32_t* __restrict__ sl, const int32_t* __restrict__ sr,
                            Owners o, int rank, long long first, long long count, uint8_t* inner,
                            uint8_t* bound, uint8_t* halo_mark, uint8_t* send_mark) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= nseg) return;
  const long long a = sl[q], b = sr[q];
  const bool ma = a >= first && a < first + count, mb = b >= first && b < first + count;
  inner[q] = ma && mb;
  bound[q] = ma != mb;
  if (ma != mb) {
    const long long rem = ma ? b : a, own = ma ? a : b;
    halo_mark[rem] = 1;
    send_mark[(long long)owner_d(o, rem) * count + (own - first)] = 1;
  }
}

__global__ void k_fill_i32(long long n, int32_t v, int32_t* out) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k < n) out[k] = v;
}

// dense global -> local maps
__global__ void k_leaf_map(long long first, long long count, const int32_t* __restrict__ halo,
                           long long nhalo, int32_t* map) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r < count)
    map[first + r] = int32_t(r);
  else if (r < count + nhalo)
    map[halo[r - count]] = int32_t(r);
}
__global__ void k_seg_map(const int32_t* __restrict__ ids, long long n, long long base, int32_t* map) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r < n) map[ids[r]] = int32_t(base + r);
}

// local rows: owned [first, first + count) then the halo
template <typename T>
__global__ void k_gather_local(long long ntot, int width, long long first, long long count,
                               const int32_t* __restrict__ halo, const T* __restrict__ src, T* __restrict__ dst) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= ntot * width) return;
  const long long r = t / width, e = t % width;
  const long long g = r < count ? first + r : halo[r - count];
  dst[t] = src[g * width + e];
}

__global__ void k_remap_owned(long long first, long long count, const int32_t* __restrict__ nb,
                              const int32_t* __restrict__ sid, const int32_t* __restrict__ lmap,
                              const int32_t* __restrict__ smap, int32_t* nbl, int32_t* sidl) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= 8 * count) return;
  const int32_t gn = nb[8 * first + t], gs = sid[8 * first + t];
  nbl[t] = gn < 0 ? -1 : lmap[gn];
  sidl[t] = gs < 0 ? -1 : smap[gs];
}

__global__ void k_local_segs(long long nloc, long long ninner, const int32_t* __restrict__ inner_ids,
                             const int32_t* __restrict__ bound_ids, const int32_t* __restrict__ sl,
                             const int32_t* __restrict__ sr, const int32_t* __restrict__ lmap, int32_t* osl,
                             int32_t* osr) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= nloc) return;
  const long long g = k < ninner ? inner_ids[k] : bound_ids[k - ninner];
  osl[k] = lmap[sl[g]];
  osr[k] = lmap[sr[g]];
}

__global__ void k_halo_owner(long long nhalo, const int32_t* __restrict__ halo, Owners o, int32_t* out) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k < nhalo) out[k] = owner_d(o, halo[k]);
}

// indices i in [0, n) with flag[i] != 0, ascending; returns the count
int64_t select_flagged(const uint8_t* flags, int64_t n, DBuf<int32_t>& out) {
  cudaStream_t st = stream();
  out.alloc(std::max<int64_t>(n, 1));
  DBuf<int> cnt(1);
  cub::CountingInputIterator<int32_t> it(0);
  size_t tmp = 0;
  FM_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, flags, out.p, cnt.p, int(n), st));
  DBuf<unsigned char> t(std::max<size_t>(tmp, 1));
  FM_CUDA(cub::DeviceSelect::Flagged(t.p, tmp, it, flags, out.p, cnt.p, int(n), st));
  FM_LAUNCHED();
  int c = 0;
  cnt.download(&c, 1);
  FM_CUDA(cudaStreamSynchronize(st));
  return c;
}

}  // namespace

Sim* sim_create_shard(const fm_sim_desc* d, const fm_raster* dem, const Grid* grid, Comm* comm, int rank) {
  if (!comm) throw Error(FM_ERR_CONFIG, "shard: null communicator");
  if (rank < 0 || rank >= comm->nranks) throw Error(FM_ERR_CONFIG, "shard: rank out of range");
  if ((comm->kind == COMM_NCCL || comm->kind == COMM_HOST) && rank != comm->rank)
    throw Error(FM_ERR_CONFIG, "shard: rank differs from the communicator's");
  if (d->solver == FM_MWDG2 || d->solver == FM_HWFV1)
    throw Error(FM_ERR_CONFIG, "shard: adaptive sims re-grid every step and run as replicas");
  if (!grid) return uniform_shard(d, dem, comm, rank);
  if (comm->nranks > kMaxRanks) throw Error(FM_ERR_CONFIG, "shard: more than 64 ranks");
  cudaStream_t st = stream();
  std::unique_ptr<Sim> G(sim_create(d, dem, grid));
  const int64_t n = G->n, nseg = G->nseg;
  const int R = comm->nranks;
  if (n < R) throw Error(FM_ERR_CONFIG, "shard plan: fewer leaves than ranks");
  Owners own{};
  own.nranks = R;
  for (int r = 0; r <= R; ++r) own.firsts[r] = shard_first(n, R, r);
  const int64_t first = own.firsts[rank], count = own.firsts[rank + 1] - first;

  // classify segments; mark the halo and the send lists
  DBuf<uint8_t> inner_f(std::max<int64_t>(nseg, 1)), bound_f(std::max<int64_t>(nseg, 1));
  DBuf<uint8_t> halo_f(n), send_f(size_t(R) * count);
  halo_f.zero();
  send_f.zero();
  k_seg_class<<<nblk(nseg, 256), 256, 0, st>>>(nseg, G->seg_l.p, G->seg_r.p, own, rank, first, count,
                                               inner_f.p, bound_f.p, halo_f.p, send_f.p);
  FM_LAUNCHED();
  DBuf<int32_t> inner_ids, bound_ids, halo, owner;
  const int64_t ninner = select_flagged(inner_f.p, nseg, inner_ids);
  const int64_t nbound = select_flagged(bound_f.p, nseg, bound_ids);
  const int64_t nhalo = select_flagged(halo_f.p, n, halo);
  std::vector<DBuf<int32_t>> sends(R);
  std::vector<int64_t> nsend(R, 0);
  for (int r = 0; r < R; ++r)
    if (r != rank) nsend[r] = select_flagged(send_f.p + size_t(r) * count, count, sends[r]);
  std::vector<int32_t> hown(static_cast<size_t>(nhalo));
  if (nhalo) {
    owner.alloc(nhalo);
    k_halo_owner<<<nblk(nhalo, 256), 256, 0, st>>>(nhalo, halo.p, own, owner.p);
    FM_LAUNCHED();
    owner.download(hown.data(), size_t(nhalo));
    FM_CUDA(cudaStreamSynchronize(st));
  }

  auto S = std::make_unique<Sim>();
  Sim& s = *S;
  // scalar parameters
  s.solver = G->solver;
  s.scheme = G->scheme;
  s.libm = G->libm;
  s.g = G->g;
  s.hdry = G->hdry;
  s.courant = G->courant;
  std::copy(G->bc, G->bc + 4, s.bc);
  s.L = G->L;
  s.M = G->M;
  s.N = G->N;
  s.R = G->R;
  s.x0 = G->x0;
  s.y0 = G->y0;
  s.p2 = G->p2;
  s.ninflow = G->ninflow;
  s.hy_t = G->hy_t;
  s.hy_q = G->hy_q;
  s.region = G->region;
  s.rect = G->rect;
  s.manning = G->manning;
  s.hydro.alloc(1);
  FM_CUDA(cudaMemcpyAsync(s.hydro.p, G->hydro.p, sizeof(Hydro), cudaMemcpyDeviceToDevice, st));
  s.clk.alloc(2);
  s.red.alloc(2);

  // maps and local arrays
  DBuf<int32_t> lmap(n), smap(std::max<int64_t>(nseg, 1));
  k_fill_i32<<<nblk(n, 256), 256, 0, st>>>(n, -1, lmap.p);
  FM_LAUNCHED();
  k_fill_i32<<<nblk(std::max<int64_t>(nseg, 1), 256), 256, 0, st>>>(std::max<int64_t>(nseg, 1), -1, smap.p);
  FM_LAUNCHED();
  const int64_t ntot = count + nhalo;
  k_leaf_map<<<nblk(ntot, 256), 256, 0, st>>>(first, count, halo.p, nhalo, lmap.p);
  FM_LAUNCHED();
  if (ninner) {
    k_seg_map<<<nblk(ninner, 256), 256, 0, st>>>(inner_ids.p, ninner, 0, smap.p);
    FM_LAUNCHED();
  }
  if (nbound) {
    k_seg_map<<<nblk(nbound, 256), 256, 0, st>>>(bound_ids.p, nbound, ninner, smap.p);
    FM_LAUNCHED();
  }
  s.n = count;
  s.nseg = ninner + nbound;
  s.nseg_inner = ninner;
  auto gather = [&](auto& dst, const auto& src, int width) {
    using T = std::remove_pointer_t<decltype(src.p)>;
    dst.alloc(size_t(ntot) * width);
    k_gather_local<T><<<nblk(ntot * width, 256), 256, 0, st>>>(ntot, width, first, count, halo.p, src.p,
                                                                 dst.p);
    FM_LAUNCHED();
  };
  gather(s.lvl, G->lvl, 1);
  gather(s.li, G->li, 1);
  gather(s.lj, G->lj, 1);
  gather(s.z, G->z, 3);
  gather(s.nman, G->nman, 1);
  gather(s.u, G->u, 9);
  s.us.alloc(9 * size_t(ntot));
  FM_CUDA(cudaMemcpyAsync(s.us.p, s.u.p, 9 * size_t(ntot) * sizeof(double), cudaMemcpyDeviceToDevice, st));
  s.sk.alloc(count);
  FM_CUDA(cudaMemcpyAsync(s.sk.p, G->sk.p + first, size_t(count), cudaMemcpyDeviceToDevice, st));
  s.nb.alloc(8 * count);
  s.sid.alloc(8 * count);
  k_remap_owned<<<nblk(8 * count, 256), 256, 0, st>>>(first, count, G->nb.p, G->sid.p, lmap.p, smap.p, s.nb.p,
                                                      s.sid.p);
  FM_LAUNCHED();
  s.seg_l.alloc(std::max<int64_t>(s.nseg, 1));
  s.seg_r.alloc(std::max<int64_t>(s.nseg, 1));
  if (s.nseg) {
    k_local_segs<<<nblk(s.nseg, 256), 256, 0, st>>>(s.nseg, ninner, inner_ids.p, bound_ids.p, G->seg_l.p,
                                                    G->seg_r.p, lmap.p, s.seg_l.p, s.seg_r.p);
    FM_LAUNCHED();
  }
  build_seg_geo(s);
  build_seg_z(s);
  s.infc.alloc(std::max<int64_t>(1, int64_t(s.ninflow) * count));
  if (s.ninflow == 0) s.infc.zero();
  for (int f = 0; f < s.ninflow; ++f)
    FM_CUDA(cudaMemcpyAsync(s.infc.p + size_t(f) * count, G->infc.p + size_t(f) * n + first,
                            size_t(count) * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  if (s.scheme == FM_ACC) {
    s.accq.alloc(std::max<int64_t>(s.nseg, 1));
    s.accq.zero();
    s.accqb.alloc(4 * s.n);
    s.accqb.zero();
  } else {
    s.segst.alloc(6 * size_t(std::max<int64_t>(s.nseg, 1)));
  }

  // exchange plan: peers ascending; halo slices grouped by owner (ascending)
  auto sh = std::make_unique<Shard>();
  sh->comm = comm;
  sh->rank = rank;
  sh->nranks = R;
  sh->first = first;
  sh->n_global = n;
  sh->n_halo = nhalo;
  int64_t total_send = 0;
  for (int r = 0; r < R; ++r) total_send += nsend[r];
  sh->send_idx.alloc(std::max<int64_t>(total_send, 1));
  int64_t at = 0;
  for (int r = 0; r < R; ++r) {
    const int64_t h0 = std::lower_bound(hown.begin(), hown.end(), r) - hown.begin();
    const int64_t h1 = std::upper_bound(hown.begin(), hown.end(), r) - hown.begin();
    if (r == rank || (nsend[r] == 0 && h1 == h0)) continue;
    sh->peers.push_back(r);
    sh->soff.push_back(at);
    sh->scnt.push_back(nsend[r]);
    if (nsend[r])
      FM_CUDA(cudaMemcpyAsync(sh->send_idx.p + at, sends[r].p, size_t(nsend[r]) * sizeof(int32_t),
                              cudaMemcpyDeviceToDevice, st));
    at += nsend[r];
    sh->hoff.push_back(h0);
    sh->hcnt.push_back(h1 - h0);
  }
  sh->send_buf.alloc(9 * size_t(std::max<int64_t>(total_send, 1)));
  s.shard = std::move(sh);
  shard_stage_lists(s);
  if (comm->kind == COMM_LOCAL) comm->members[rank] = &s;
  FM_CUDA(cudaStreamSynchronize(st));
  G.reset();
  if (comm->kind == COMM_NCCL) shard_warmup(s);
  return S.release();
}

// ---- step operations ---------------------------------------------------------

// The array a halo exchange moves and its width in doubles per leaf: the
// 72 B rows of U (or U*), or ACC's compact depth (8 B per halo leaf, SURVEY
// §8 e3) while the ACC state is in its compact layout.
double* exch_array(Sim& s, int op, int* w) {
  if (op == OP_EXCH_U && s.acc_soa) {
    *w = 1;
    return s.ch.p;
  }
  if (op == OP_EXCH_U && s.fv1c) {  // FV1 compact: the head's output rows of 3
    *w = 3;
    return s.cu3.p;
  }
  *w = 9;
  return op == OP_EXCH_U ? s.u.p : s.us.p;
}

void shard_pack(Sim& s, const double* arr, int w) {
  Shard& sh = *s.shard;
  const long long m = (long long)(sh.soff.empty() ? 0 : sh.soff.back() + sh.scnt.back());
  if (m == 0) return;
  k_pack<<<nblk(w * m, 256), 256, 0, stream()>>>(arr, w, sh.send_idx.p, m, sh.send_buf.p);
  FM_LAUNCHED();
}

// Local group: copy every peer's packed slice for this shard into its halo.
void shard_local_recv(Sim& s, double* arr, int w) {
  Shard& sh = *s.shard;
  Comm& c = *sh.comm;
  for (size_t k = 0; k < sh.peers.size(); ++k) {
    const Sim* peer = c.members[sh.peers[k]];
    if (!peer) throw Error(FM_ERR_CONFIG, "local group: a peer shard is missing");
    const Shard& ps = *peer->shard;
    const auto it = std::find(ps.peers.begin(), ps.peers.end(), sh.rank);
    if (it == ps.peers.end()) throw Error(FM_ERR_STRUCTURE, "local group: asymmetric exchange plan");
    const size_t j = size_t(it - ps.peers.begin());
    if (ps.scnt[j] != sh.hcnt[k]) throw Error(FM_ERR_STRUCTURE, "local group: halo size mismatch");
    if (sh.hcnt[k])
      FM_CUDA(cudaMemcpyAsync(arr + w * (s.n + sh.hoff[k]), ps.send_buf.p + w * ps.soff[j],
                              w * sh.hcnt[k] * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
  }
}

void shard_local_reduce(const std::vector<Sim*>& sims) {
  std::vector<DevRed*> reds;
  for (Sim* s : sims) reds.push_back(s->red.p);
  DBuf<DevRed*> d;
  d.upload(reds.data(), reds.size());
  k_red_combine<<<1, 32, 0, stream()>>>(d.p, int(reds.size()));
  FM_LAUNCHED();
  FM_CUDA(cudaStreamSynchronize(stream()));
}

Shard::~Shard() {
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (side) cudaStreamDestroy(side);
}

void shard_finish(Sim& s) {
  Shard& sh = *s.shard;
  if (!sh.pending) return;
  FM_CUDA(cudaStreamWaitEvent(stream(), sh.ev_join, 0));
  sh.pending = false;
}

// A host-transport exchange: pack, stage the slices through the segment,
// land the peers' slices in the halo slots.
static void host_exchange(Sim& s, double* arr, int w) {
  Shard& sh = *s.shard;
  Comm& c = *sh.comm;
  shard_pack(s, arr, w);
  const long long m = (long long)(sh.soff.empty() ? 0 : sh.soff.back() + sh.scnt.back());
  c.stage.resize(size_t(std::max<long long>(m, 1)) * w);
  if (m) FM_CUDA(cudaMemcpyAsync(c.stage.data(), sh.send_buf.p, size_t(m) * w * 8, cudaMemcpyDeviceToHost, stream()));
  FM_CUDA(cudaStreamSynchronize(stream()));
  for (size_t k = 0; k < sh.peers.size(); ++k) {
    const size_t bytes = size_t(sh.scnt[k]) * w * 8;
    if (bytes > c.slot_bytes)
      throw Error(FM_ERR_OTHER, "host comm: halo slice larger than a slot (raise $FM_HOST_COMM_MB)");
    if (bytes) std::memcpy(c.slot(sh.rank, sh.peers[k]), c.stage.data() + size_t(w) * sh.soff[k], bytes);
  }
  shm_barrier(c);
  for (size_t k = 0; k < sh.peers.size(); ++k)
    if (sh.hcnt[k])
      FM_CUDA(cudaMemcpyAsync(arr + size_t(w) * (s.n + sh.hoff[k]), c.slot(sh.peers[k], sh.rank),
                              size_t(sh.hcnt[k]) * w * 8, cudaMemcpyHostToDevice, stream()));
  FM_CUDA(cudaStreamSynchronize(stream()));
  shm_barrier(c);  // the slots may be reused
}

// The stage split's leaf lists from the send plan (once, at creation).
void shard_stage_lists(Sim& s) {
  Shard& sh = *s.shard;
  const int64_t m = sh.soff.empty() ? 0 : sh.soff.back() + sh.scnt.back();
  std::vector<int32_t> idx(size_t(std::max<int64_t>(m, 0)));
  if (m) {
    sh.send_idx.download(idx.data(), size_t(m));
    FM_CUDA(cudaStreamSynchronize(stream()));
  }
  std::vector<uint8_t> sent(size_t(s.n), 0);
  for (int32_t k : idx)
    if (k >= 0 && k < s.n) sent[size_t(k)] = 1;
  std::vector<int32_t> first, rest;
  for (int64_t k = 0; k < s.n; ++k) (sent[size_t(k)] ? first : rest).push_back(int32_t(k));
  sh.n_first = int64_t(first.size());
  sh.n_rest = int64_t(rest.size());
  if (first.empty()) first.push_back(0);
  if (rest.empty()) rest.push_back(0);
  sh.stage_first.upload(first.data(), first.size());
  sh.stage_rest.upload(rest.data(), rest.size());
}

bool shard_nccl(const Sim& s) { return s.shard && s.shard->comm && s.shard->comm->kind == COMM_NCCL; }

bool shard_eager(const Sim& s) { return s.shard && s.shard->comm && s.shard->comm->kind == COMM_HOST; }

void shard_op(Sim& s, int op) {
  FM_RANGE(op == OP_REDUCE ? "shard_reduce" : "shard_exchange");
  Shard& sh = *s.shard;
  if (!sh.comm) throw Error(FM_ERR_CONFIG, "shard: the communicator was destroyed");
  if (sh.comm->kind == COMM_HOST) {
    if (op == OP_REDUCE) {
      host_allreduce_u64_min(*sh.comm, reinterpret_cast<unsigned long long*>(s.red.p), 8);
    } else {
      int w = 9;
      double* arr = exch_array(s, op, &w);
      host_exchange(s, arr, w);
    }
    return;
  }
  if (sh.comm->kind != COMM_NCCL)
    throw Error(FM_ERR_CONFIG, "shard: a local-group shard steps only through fm_group_run");
  const NcclApi& api = nccl();
  cudaStream_t st = stream();
  shard_finish(s);
  if (op == OP_REDUCE) {
    // both parity slots: the other slot is already identical on every rank
    nccl_check(api.AllReduce(s.red.p, s.red.p, 2 * sizeof(DevRed) / 8, ncclUint64, ncclMin,
                             sh.comm->nc, st), "ncclAllReduce");
    return;
  }
  int w = 9;
  double* arr = exch_array(s, op, &w);
  shard_pack(s, arr, w);
  // fork: the exchange runs on the side stream, the main stream goes on with
  // the segments that need no halo; shard_finish joins
  if (!sh.side) {
    FM_CUDA(cudaStreamCreateWithFlags(&sh.side, cudaStreamNonBlocking));
    FM_CUDA(cudaEventCreateWithFlags(&sh.ev_fork, cudaEventDisableTiming));
    FM_CUDA(cudaEventCreateWithFlags(&sh.ev_join, cudaEventDisableTiming));
  }
  FM_CUDA(cudaEventRecord(sh.ev_fork, st));
  FM_CUDA(cudaStreamWaitEvent(sh.side, sh.ev_fork, 0));
  nccl_check(api.GroupStart(), "ncclGroupStart");
  for (size_t k = 0; k < sh.peers.size(); ++k) {
    if (sh.scnt[k])
      nccl_check(api.Send(sh.send_buf.p + w * sh.soff[k], size_t(w * sh.scnt[k]), ncclFloat64,
                          sh.peers[k], sh.comm->nc, sh.side), "ncclSend");
    if (sh.hcnt[k])
      nccl_check(api.Recv(arr + w * (s.n + sh.hoff[k]), size_t(w * sh.hcnt[k]), ncclFloat64,
                          sh.peers[k], sh.comm->nc, sh.side), "ncclRecv");
  }
  nccl_check(api.GroupEnd(), "ncclGroupEnd");
  FM_CUDA(cudaEventRecord(sh.ev_join, sh.side));
  sh.pending = true;
}

// Host-API reductions of a sharded sim across its NCCL ranks (a local-group
// shard answers for itself).
void shard_allreduce_u64_min(Sim& s, unsigned long long* dev, int count) {
  if (s.shard && s.shard->comm && s.shard->comm->kind == COMM_HOST) {
    host_allreduce_u64_min(*s.shard->comm, dev, count);
    return;
  }
  if (!s.shard || !s.shard->comm || s.shard->comm->kind != COMM_NCCL) return;
  shard_finish(s);
  nccl_check(nccl().AllReduce(dev, dev, size_t(count), ncclUint64, ncclMin, s.shard->comm->nc, stream()),
             "ncclAllReduce");
}
double shard_allreduce_sum(Sim& s, double v) {
  if (s.shard && s.shard->comm && s.shard->comm->kind == COMM_HOST) return host_allreduce_sum(*s.shard->comm, v);
  if (!s.shard || !s.shard->comm || s.shard->comm->kind != COMM_NCCL) return v;
  DBuf<double> d;
  d.upload(&v, 1);
  nccl_check(nccl().AllReduce(d.p, d.p, 1, ncclFloat64, ncclSum, s.shard->comm->nc, stream()),
             "ncclAllReduce");
  d.download(&v, 1);
  FM_CUDA(cudaStreamSynchronize(stream()));
  return v;
}

}  // namespace fmh
