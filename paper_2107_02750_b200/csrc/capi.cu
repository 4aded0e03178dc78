// The C ABI of include/fm_gpu.h.  Every entry point converts C++ exceptions
// into status codes + a thread-local message; no exception crosses the ABI.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "fm_device.cuh"
#include "fm_io.hpp"
#include "fm_sim.hpp"

using namespace fmh;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return FM_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return FM_ERR_OTHER;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FM_ERR_OTHER;
  }
}

// No CPU fallback: a call without a usable CUDA device fails loudly.
void require_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    throw Error(FM_ERR_CUDA, "libfm_gpu requires a CUDA device (sm_100a); none is available");
}

__global__ void k_dhat_level(const double* __restrict__ det, const uint64_t nodes, double norm,
                             int M, int level, double* out) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= nodes) return;
  double d[9];
  for (int q = 0; q < 9; ++q) d[q] = det[9 * n + q];
  int i, j;
  fmd::node_ij(level, n, M, i, j);
  out[size_t(j) * (M << level) + i] = fmd::dhat(d, norm);
}

__global__ void k_flags_level(const uint8_t* __restrict__ f, const uint64_t nodes, int M, int level,
                              uint8_t* out) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= nodes) return;
  int i, j;
  fmd::node_ij(level, n, M, i, j);
  out[size_t(j) * (M << level) + i] = f[n];
}

__global__ void k_near(const double* __restrict__ det, uint64_t nodes, double norm, double eps,
                       double rel, unsigned long long* count) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= nodes) return;
  double d[9];
  for (int q = 0; q < 9; ++q) d[q] = det[9 * n + q];
  if (fabs(fmd::dhat(d, norm) - eps) <= rel * eps) atomicAdd(count, 1ull);
}

inline unsigned nblk(uint64_t n) { return unsigned((n + 255) / 256); }

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// Random operands: random sign and mantissa, exponent drawn across (and a
// little beyond) the fast-path window, with hard mantissa patterns mixed in.
__device__ __forceinline__ double rand_operand(uint64_t r, uint64_t r2) {
  uint64_t mant = r & 0x000fffffffffffffull;
  switch (r2 & 7) {
    case 0: mant = 0; break;                                // exact powers of two
    case 1: mant = 0x000fffffffffffffull; break;            // all ones
    case 2: mant &= 0xffffffffull << 20; break;             // short mantissas
    default: break;
  }
  // every biased exponent 0..2046 (zero/subnormal at 0), weighted toward the
  // fast-path window edges half of the time
  uint64_t e = (r2 >> 3) % 2047;
  if ((r2 >> 20) & 1) e = ((r2 >> 21) & 1 ? 40 : 2020) + ((r2 >> 22) % 40);
  const uint64_t sign = (r2 >> 40) & 1;
  return __longlong_as_double(static_cast<long long>((sign << 63) | (e << 52) | mant));
}

// FM_GUARD's positive control: one write just past a buffer's end (into its
// guard band, which exists only under FM_GUARD=1)
__global__ void k_write_past_end(double* p, int64_t n) { p[n] = 1.0; }

__global__ void k_selftest_div(int which, int64_t n, uint64_t seed, unsigned long long* fails) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const uint64_t a1 = mix64(seed ^ (2 * k)), a2 = mix64(a1), b1 = mix64(a2), b2 = mix64(b1);
  const double a = rand_operand(a1, a2), b = rand_operand(b1, b2);
  if (which == 1) {  // the constant-divisor path of project4
    const double q1 = fmd::div_4s3(a), r1 = a / (4.0 * fmd::kS3);
    if (__double_as_longlong(q1) != __double_as_longlong(r1)) atomicAdd(fails, 1ull);
    return;
  }
  if (which == 2) {  // the shared-divisor division fmd::zdiv2, both quotients
    const uint64_t c1 = mix64(b2), c2 = mix64(c1);
    const double a2 = rand_operand(c1, c2);
    double q1, q2;
    fmd::zdiv2(a, a2, b, q1, q2);
    const double r1 = a == 0.0 ? a : a / b, r2 = a2 == 0.0 ? a2 : a2 / b;
    if (__double_as_longlong(q1) != __double_as_longlong(r1) || __double_as_longlong(q2) != __double_as_longlong(r2))
      atomicAdd(fails, 1ull);
    return;
  }
  // the inline division kernel builds use with -DFM_INLINE_DIV (fmd::quot)
  const double q = (fmd::div_fast_ok(a) && fmd::div_fast_ok(b)) ? fmd::quot(a, b, fmd::recip(b)) : a / b;
  const double ref = a / b;
  if (__double_as_longlong(q) != __double_as_longlong(ref)) atomicAdd(fails, 1ull);
}

__global__ void k_eval_libm(int fn, int64_t n, const double* __restrict__ x, double* __restrict__ out) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const double v = x[k];
  out[k] = fn == 0 ? fmd::pow73_m(v, FM_LIBM_NATIVE) : fn == 1 ? fmd::cbrt_m(v, FM_LIBM_NATIVE)
         : fn == 2 ? pow(v, 7.0 / 3.0) : fn == 3 ? fmd::pow73_m(v, FM_LIBM_PORTABLE) : fmd::pow73_cr(v);
}
}  // namespace

struct fm_grid {
  std::unique_ptr<Grid> g;
};
struct fm_sim {
  std::unique_ptr<Sim> s;
};
struct fm_comm {
  Comm* c = nullptr;
  ~fm_comm() { comm_destroy(c); }
};

extern "C" {

const char* fm_last_error(void) { return g_err.c_str(); }

int fm_init(int32_t device) {
  return guard([&] {
    require_device();
    FM_CUDA(cudaSetDevice(device));
    upload_banks();
    order_preload();
  });
}

int fm_set_stream(void* s) {
  return guard([&] { set_stream(static_cast<cudaStream_t>(s)); });
}

int fm_synchronize(void) {
  return guard([&] { FM_CUDA(cudaStreamSynchronize(stream())); });
}

int64_t fm_launch_count(void) { return launches(); }

int fm_debug_guard_report(int64_t* checked, int64_t* overruns) {
  return guard([&] { guard_report(checked, overruns); });
}

int fm_selftest(int32_t which, int64_t n, uint64_t seed, int64_t* failures) {
  return guard([&] {
    require_device();
    if (which < 0 || which > 3) throw Error(FM_ERR_CONFIG, "unknown self-test");
    if (which == 3) {
      // the guard checker finds a deliberate overrun (FM_GUARD=1 only: the
      // write lands in the buffer's guard band); *failures = overruns found
      if (!guard_enabled()) throw Error(FM_ERR_CONFIG, "self-test 3 needs FM_GUARD=1 when the library loads");
      int64_t c0 = 0, o0 = 0, c1 = 0, o1 = 0;
      guard_report(&c0, &o0);
      {
        DBuf<double> b(4);
        k_write_past_end<<<1, 1, 0, stream()>>>(b.p, 4);
        FM_LAUNCHED();
      }
      guard_report(&c1, &o1);
      *failures = o1 - o0;
      return;
    }
    DBuf<unsigned long long> f(1);
    f.zero();
    k_selftest_div<<<unsigned((n + 255) / 256), 256, 0, stream()>>>(which, n, seed, f.p);
    FM_LAUNCHED();
    unsigned long long v = 0;
    f.download(&v, 1);
    FM_CUDA(cudaStreamSynchronize(stream()));
    *failures = int64_t(v);
  });
}

int fm_mra_static(const fm_raster* dem, int32_t L, double eps, int32_t graded, int32_t kind,
                  fm_grid** out) {
  return guard([&] {
    require_device();
    auto h = std::make_unique<fm_grid>();
    h->g.reset(mra_static(dem, L, eps, graded != 0, kind));
    *out = h.release();
  });
}

int fm_grid_import(int32_t L, int32_t M, int32_t N, double Rfine, double x0, double y0, int64_t n,
                   const int32_t* level, const int32_t* i, const int32_t* j, const double* topo3,
                   fm_grid** out) {
  return guard([&] {
    require_device();
    auto h = std::make_unique<fm_grid>();
    h->g.reset(grid_from_leaves(L, M, N, Rfine, x0, y0, n, level, i, j, topo3));
    *out = h.release();
  });
}
int fm_grid_destroy(fm_grid* g) {
  return guard([&] { delete g; });
}

int64_t fm_grid_num_leaves(const fm_grid* g) { return g ? g->g->nleaves : -1; }

int fm_grid_info(const fm_grid* h, int32_t* L, int32_t* M, int32_t* N, double* R, double* x0,
                 double* y0, double* norm) {
  return guard([&] {
    const Grid& g = *h->g;
    if (L) *L = g.L;
    if (M) *M = g.M;
    if (N) *N = g.N;
    if (R) *R = g.R;
    if (x0) *x0 = g.x0;
    if (y0) *y0 = g.y0;
    if (norm) *norm = g.field_norm;
  });
}

int fm_grid_leaves(const fm_grid* h, int32_t order, int32_t* lo, int32_t* io, int32_t* jo,
                   double* topo3) {
  return guard([&] {
    const Grid& g = *h->g;
    std::vector<int8_t> l;
    std::vector<int32_t> i, j;
    std::vector<int64_t> perm;
    if (order == FM_ORDER_REFERENCE) {
      perm = reference_order(g, &l, &i, &j);
    } else {
      l = g.lf_l.to_host();
      i = g.lf_i.to_host();
      j = g.lf_j.to_host();
      perm.resize(g.nleaves);
      for (int64_t k = 0; k < g.nleaves; ++k) perm[k] = k;
    }
    std::vector<double> z = topo3 ? g.lf_z.to_host() : std::vector<double>();
    for (int64_t r = 0; r < g.nleaves; ++r) {
      const int64_t k = perm[r];
      if (lo) lo[r] = l[k];
      if (io) io[r] = i[k];
      if (jo) jo[r] = j[k];
      if (topo3) std::memcpy(topo3 + 3 * r, &z[3 * k], 24);
    }
  });
}

int fm_grid_flags(const fm_grid* h, int32_t level, uint8_t* out) {
  return guard([&] {
    const Grid& g = *h->g;
    if (level < 0 || level >= g.L) throw Error(FM_ERR_DOMAIN, "level out of range");
    const uint64_t nodes = g.nodes(level);
    DBuf<uint8_t> tmp(nodes);
    k_flags_level<<<nblk(nodes), 256, 0, stream()>>>(g.flag[level].p, nodes, g.M, level, tmp.p);
    FM_LAUNCHED();
    tmp.download(out, nodes);
    FM_CUDA(cudaStreamSynchronize(stream()));
  });
}

int fm_grid_dhat(const fm_grid* h, int32_t level, double* out) {
  return guard([&] {
    const Grid& g = *h->g;
    if (level < 0 || level >= g.L) throw Error(FM_ERR_DOMAIN, "level out of range");
    const uint64_t nodes = g.nodes(level);
    DBuf<double> tmp(nodes);
    k_dhat_level<<<nblk(nodes), 256, 0, stream()>>>(g.det[level].p, nodes, g.field_norm, g.M,
                                                     level, tmp.p);
    FM_LAUNCHED();
    tmp.download(out, nodes);
    FM_CUDA(cudaStreamSynchronize(stream()));
  });
}

int fm_grid_near_threshold(const fm_grid* h, double rel, int64_t* count) {
  return guard([&] {
    const Grid& g = *h->g;
    DBuf<unsigned long long> c(1);
    c.zero();
    for (int l = 0; l < g.L; ++l) {
      k_near<<<nblk(g.nodes(l)), 256, 0, stream()>>>(g.det[l].p, g.nodes(l), g.field_norm, g.eps,
                                                      rel, c.p);
      FM_LAUNCHED();
    }
    unsigned long long v = 0;
    c.download(&v, 1);
    FM_CUDA(cudaStreamSynchronize(stream()));
    *count = int64_t(v);
  });
}

int fm_grid_timing(const fm_grid* h, double* ms, double* bytes) {
  return guard([&] {
    if (ms) *ms = h->g->mra_ms;
    if (bytes) *bytes = h->g->mra_bytes;
  });
}

int fm_grade_flags(int32_t L, int32_t M, int32_t N, int32_t graded, uint8_t* flags) {
  return guard([&] {
    require_device();
    if (L < 1) return;
    grade_flags_host(L, M, N, graded != 0, flags);
  });
}

int fm_sim_create(const fm_sim_desc* d, const fm_raster* dem, const fm_grid* grid, fm_sim** out) {
  return guard([&] {
    require_device();
    auto h = std::make_unique<fm_sim>();
    h->s.reset(sim_create(d, dem, grid ? grid->g.get() : nullptr));
    // the reference-order permutation of a static leaf set, built with the
    // sim (scratch allocations and a sort) rather than inside the first
    // download; adaptive sims rebuild it after a re-grid on demand
    if (!h->s->adaptive) sim_ref_perm(*h->s);
    *out = h.release();
  });
}

int fm_sim_destroy(fm_sim* s) {
  return guard([&] { delete s; });
}

int64_t fm_sim_num_cells(const fm_sim* s) { return s ? s->s->n : -1; }
int64_t fm_sim_num_segments(const fm_sim* s) { return s ? s->s->nseg : -1; }

int fm_sim_compute_dt(fm_sim* s, double* dt) {
  return guard([&] { *dt = sim_compute_dt(*s->s); });
}
int fm_sim_step(fm_sim* s, double dt) {
  return guard([&] { sim_step(*s->s, dt); });
}
int fm_sim_apply_inflows(fm_sim* s, double t, double dt, double* added) {
  return guard([&] { *added = sim_apply_inflows(*s->s, t, dt); });
}
int fm_sim_adapt(fm_sim* s, double t) {
  return guard([&] { sim_adapt(*s->s, t); });
}
int fm_sim_volume(fm_sim* s, double* v) {
  return guard([&] { *v = sim_volume(*s->s); });
}
int fm_sim_finite(fm_sim* s, int32_t* ok, double* bx, double* by) {
  return guard([&] { *ok = sim_finite(*s->s, bx, by) ? 1 : 0; });
}
int fm_sim_download(fm_sim* s, int32_t* l, int32_t* i, int32_t* j, double* u9, double* z3) {
  return guard([&] { sim_download(*s->s, l, i, j, u9, z3); });
}
int fm_sim_upload(fm_sim* s, const double* u9) {
  return guard([&] { sim_upload(*s->s, u9); });
}
int fm_sim_raster_shape(fm_sim* s, int32_t* nc, int32_t* nr, double* xll, double* yll, double* cs,
                        double* nodata) {
  return guard([&] { sim_raster_shape(*s->s, nc, nr, xll, yll, cs, nodata); });
}
int fm_sim_raster(fm_sim* s, int32_t which, double* out, int32_t on_device) {
  return guard([&] { sim_raster(*s->s, which, out, on_device != 0); });
}
int fm_sim_sample_gauges(fm_sim* s, int32_t n, const double* x, const double* y, double* out4) {
  return guard([&] { sim_sample_gauges(*s->s, n, x, y, out4); });
}
int fm_comm_unique_id(uint8_t id[128]) {
  return guard([&] { comm_unique_id(id); });
}
int fm_comm_create_nccl(int32_t nranks, int32_t rank, const uint8_t id[128], fm_comm** out) {
  return guard([&] {
    require_device();
    auto h = std::make_unique<fm_comm>();
    h->c = comm_create_nccl(nranks, rank, id);
    *out = h.release();
  });
}
int fm_comm_create_host(int32_t nranks, int32_t rank, const char* name, fm_comm** out) {
  return guard([&] {
    auto h = std::make_unique<fm_comm>();
    h->c = comm_create_host(nranks, rank, name);
    *out = h.release();
  });
}
int fm_comm_create_local(int32_t nranks, fm_comm** out) {
  return guard([&] {
    auto h = std::make_unique<fm_comm>();
    h->c = comm_create_local(nranks);
    *out = h.release();
  });
}
int fm_comm_destroy(fm_comm* c) {
  return guard([&] { delete c; });
}
int fm_sim_create_shard(const fm_sim_desc* d, const fm_raster* dem, const fm_grid* grid, fm_comm* comm,
                        int32_t rank, fm_sim** out) {
  return guard([&] {
    require_device();
    if (!comm) throw Error(FM_ERR_CONFIG, "shard: null communicator");
    auto h = std::make_unique<fm_sim>();
    h->s.reset(sim_create_shard(d, dem, grid ? grid->g.get() : nullptr, comm->c, rank));
    *out = h.release();
  });
}
int fm_sim_acc_faces(fm_sim* s, double* gx, double* gy, const double* sx, const double* sy) {
  return guard([&] {
    Sim& m = *s->s;
    if (!m.uniform || m.scheme != FM_ACC || m.shard)
      throw Error(FM_ERR_CONFIG, "acc_faces: an unsharded uniform ACC simulation only");
    if (sx) m.aqx.upload(sx, m.aqx.n);
    if (sy) m.aqy.upload(sy, m.aqy.n);
    if (gx) m.aqx.download(gx, m.aqx.n);
    if (gy) m.aqy.download(gy, m.aqy.n);
    FM_CUDA(cudaStreamSynchronize(stream()));
  });
}
int fm_sim_geometry(const fm_sim* s, int32_t* L, int32_t* M, int32_t* N, double* Rfine, double* x0,
                    double* y0) {
  return guard([&] {
    const Sim& m = *s->s;
    if (L) *L = m.uniform ? 0 : m.L;
    if (M) *M = m.uniform ? m.nx : m.M;
    if (N) *N = m.uniform ? (m.nyg ? m.nyg : m.ny) : m.N;
    if (Rfine) *Rfine = m.R;
    if (x0) *x0 = m.x0;
    if (y0) *y0 = m.y0;
  });
}
int fm_sim_shard_info(const fm_sim* s, int32_t* rank, int32_t* nranks, int64_t* first, int64_t* owned,
                      int64_t* halo, int64_t* n_global) {
  return guard([&] {
    const Sim& m = *s->s;
    const Shard* sh = m.shard.get();
    if (rank) *rank = sh ? sh->rank : 0;
    if (nranks) *nranks = sh ? sh->nranks : 1;
    if (first) *first = sh ? sh->first : 0;
    if (owned) *owned = m.n;
    if (halo) *halo = sh ? sh->n_halo : 0;
    if (n_global) *n_global = sh ? sh->n_global : m.n;
  });
}
int fm_group_run(fm_sim* const* sims, int32_t n, fm_clock* clk, int64_t max_steps, int32_t stop_at_events,
                 fm_run_result* out) {
  fm_run_result r{};
  const int st = guard([&] {
    std::vector<Sim*> v;
    for (int32_t k = 0; k < n; ++k) v.push_back(sims[k]->s.get());
    group_run(v, clk, max_steps, stop_at_events, &r);
  });
  if (out) *out = r;
  return st;
}
int fm_shard_plan(int64_t n_leaves, int64_t n_segments, const int32_t* seg_l, const int32_t* seg_r,
                  int32_t nranks, int32_t rank, int64_t* first, int64_t* count, int64_t* n_local_segments,
                  int64_t* n_halo, int64_t* halo, int32_t* halo_owner, int64_t* send_counts,
                  int64_t* send) {
  return guard([&] {
    const ShardPlan p = shard_plan(n_leaves, n_segments, seg_l, seg_r, nranks, rank);
    if (first) *first = p.first;
    if (count) *count = p.count;
    if (n_local_segments) *n_local_segments = int64_t(p.segs.size());
    if (n_halo) *n_halo = int64_t(p.halo.size());
    if (halo) std::copy(p.halo.begin(), p.halo.end(), halo);
    if (halo_owner) std::copy(p.halo_owner.begin(), p.halo_owner.end(), halo_owner);
    int64_t at = 0;
    for (int r = 0; r < nranks; ++r) {
      if (send_counts) send_counts[r] = int64_t(p.send[r].size());
      if (send) std::copy(p.send[r].begin(), p.send[r].end(), send + at);
      at += int64_t(p.send[r].size());
    }
  });
}
int fm_sim_topology(fm_sim* s, int32_t* level, int32_t* i, int32_t* j, int32_t* seg_l, int32_t* seg_r) {
  return guard([&] {
    Sim& m = *s->s;
    if (m.uniform) throw Error(FM_ERR_CONFIG, "topology: uniform sims have no leaf list");
    if (level) {
      const std::vector<int8_t> l = m.lvl.to_host();
      for (int64_t k = 0; k < m.n; ++k) level[k] = l[k];
    }
    if (i) m.li.download(i, m.n);
    if (j) m.lj.download(j, m.n);
    if (seg_l || seg_r) {
      if (m.seg_l.n < size_t(m.nseg)) throw Error(FM_ERR_CONFIG, "topology: no segment list");
      if (seg_l) m.seg_l.download(seg_l, m.nseg);
      if (seg_r) m.seg_r.download(seg_r, m.nseg);
    }
    FM_CUDA(cudaStreamSynchronize(stream()));
  });
}
int fm_raster_read(const char* path, fm_raster* out) {
  return guard([&] {
    if (!path || !out) throw Error(FM_ERR_IO, "fm_raster_read: null argument");
    raster_read(path, out);
  });
}
int fm_raster_release(fm_raster* r) {
  return guard([&] { raster_release(r); });
}
int fm_raster_write(const fm_raster* r, const char* path, int32_t binary) {
  return guard([&] {
    if (!path) throw Error(FM_ERR_IO, "fm_raster_write: null path");
    if (binary) raster_write_bin(r, path);
    else raster_write_ascii(r, path);
  });
}
int fm_grid_write(const fm_grid* g, const char* path, int32_t binary) {
  return guard([&] {
    if (!g || !path) throw Error(FM_ERR_IO, "fm_grid_write: null argument");
    require_device();
    grid_write(g, path, binary != 0);
  });
}
int fm_grid_read(const char* path, fm_grid** out) {
  return guard([&] {
    if (!path || !out) throw Error(FM_ERR_IO, "fm_grid_read: null argument");
    grid_read(path, out);
  });
}
int fm_rmse(const double* tt, const double* tv, int64_t nt, const double* rt, const double* rv, int64_t nr,
            double* out) {
  return guard([&] {
    if (nt <= 0 || nr <= 0 || !tt || !tv || !rt || !rv || !out) throw Error(FM_ERR_IO, "rmse: empty series");
    // interpolate (metrics.cpp:20-28)
    auto interp = [&](double t) {
      const double* hi = std::upper_bound(tt, tt + nt, t);
      if (hi == tt) return tv[0];
      if (hi == tt + nt) return tv[nt - 1];
      const int64_t k = hi - tt;
      const double t0 = tt[k - 1], t1 = tt[k];
      const double w = (t - t0) / (t1 - t0);
      return tv[k - 1] + w * (tv[k] - tv[k - 1]);
    };
    const double lo = std::max(tt[0], rt[0]);
    const double hi = std::min(tt[nt - 1], rt[nr - 1]);
    double sum = 0.0;
    long long n = 0;
    for (int64_t k = 0; k < nr; ++k) {
      if (rt[k] < lo || rt[k] > hi) continue;
      const double d = interp(rt[k]) - rv[k];
      sum += d * d;
      ++n;
    }
    if (n == 0) throw Error(FM_ERR_IO, "rmse: series do not overlap in time");
    *out = std::sqrt(sum / double(n));
  });
}
int fm_extent_metrics(const fm_raster* test, const fm_raster* ref, double wet_threshold, int64_t* counts,
                      double* rates) {
  return guard([&] {
    require_device();
    extent_metrics(test, ref, wet_threshold, counts, rates);
  });
}
int fm_eval_libm(int32_t fn, int64_t n, const double* x, double* out) {
  return guard([&] {
    require_device();
    if (fn < 0 || fn > 4) throw Error(FM_ERR_CONFIG, "eval_libm: unknown function");
    DBuf<double> dx, dy(std::max<int64_t>(n, 1));
    dx.upload(x, n);
    k_eval_libm<<<unsigned((n + 255) / 256), 256, 0, stream()>>>(fn, n, dx.p, dy.p);
    FM_LAUNCHED();
    dy.download(out, n);
    FM_CUDA(cudaStreamSynchronize(stream()));
  });
}
int fm_sim_adapt_stats(fm_sim* s, int64_t* n_encoded, int64_t* n_internal) {
  return guard([&] { adaptive_stats(*s->s, n_encoded, n_internal); });
}
int fm_sim_checkpoint(fm_sim* s, const char* path) {
  return guard([&] { sim_checkpoint(*s->s, path); });
}
int fm_sim_resume(fm_sim* s, const char* path) {
  return guard([&] { sim_resume(*s->s, path); });
}
int fm_sim_snapshot(fm_sim* s) {
  return guard([&] { sim_snapshot(*s->s); });
}
int fm_sim_restore(fm_sim* s) {
  return guard([&] { sim_restore(*s->s); });
}
int64_t fm_sim_element_log(fm_sim* h, double* t, int64_t* count, int64_t cap) {
  const auto& log = h->s->element_log;
  const int64_t n = int64_t(log.size());
  for (int64_t k = 0; k < std::min(n, cap); ++k) {
    if (t) t[k] = log[k].first;
    if (count) count[k] = log[k].second;
  }
  return n;
}
int fm_sim_run(fm_sim* s, fm_clock* clk, int64_t max_steps, int32_t stop_at_events,
               fm_run_result* out) {
  return guard([&] { sim_run(*s->s, clk, max_steps, stop_at_events, out); });
}
int fm_sim_last_run_ms(fm_sim* s, double* ms) {
  return guard([&] { *ms = s->s->last_run_ms; });
}
int fm_sim_profile(fm_sim* s, int64_t steps, double* ms, int64_t* launches, int32_t cap,
                   int32_t* n) {
  return guard([&] {
    int nf = 0;
    sim_profile(*s->s, steps, ms, launches, cap, &nf);
    *n = nf;
  });
}
const char* fm_sim_kernel_name(fm_sim*, int32_t family) { return kernel_family_name(family); }

}  // extern "C"
