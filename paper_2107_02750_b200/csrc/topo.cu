// Device topology of a graded leaf set.
//
// Replaces neighbors / is_graded / enumerate_faces (quadgrid.cpp:121-260)
// and the inflow / Manning resolution of make_nonuniform_sim
// (solver_nonuniform.cpp:575-584, 611-628).  Instead of hash probes, every
// query is an O(1) look-up in the dense flag pyramid: a level-l node exists
// iff its parent is flagged, it is a leaf iff it exists and is unflagged, and
// its leaf index is off[l][node] (or off[L-1][parent] + k at level L).
//
// Per leaf and side the result is a 2-bit kind (0 boundary, 1 one coarser
// neighbour, 2 one same-level neighbour, 3 two finer neighbours) and up to two
// neighbour indices ordered south-to-north / west-to-east, which is the order
// enumerate_faces sorts each side's segment list in (quadgrid.cpp:250-258).
// Segments (needed by ACC's persistent face discharges) are owned by the
// coarser leaf, or by the west/south leaf at equal level, exactly as in
// enumerate_faces (quadgrid.cpp:206-208).
#include "fm_device.cuh"
#include "fm_sim.hpp"
#include "leafinfo.cuh"
#include "step_common.cuh"

using namespace fmd;

namespace fmh {

namespace {

struct TopoIn {
  const uint8_t* flag[16];
  const int32_t* off[16];
  int L, M, N;
};

__device__ __forceinline__ int32_t leaf_index(const TopoIn& t, int l, uint64_t n) {
  if (t.L == 0) return int32_t(n);
  if (l < t.L) return t.off[l][n];
  return t.off[t.L - 1][n >> 2] + int32_t(n & 3);
}
__device__ __forceinline__ bool is_flagged(const TopoIn& t, int l, uint64_t n) {
  return l < t.L && t.flag[l][n] != 0;
}

__global__ void k_topo(TopoIn t, long long n, const int8_t* __restrict__ lvl,
                       const int32_t* __restrict__ li, const int32_t* __restrict__ lj,
                       int32_t* __restrict__ nb, uint8_t* __restrict__ sk,
                       int32_t* __restrict__ owned, int* err) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int l = lvl[k], i = li[k], j = lj[k];
  const int w = t.M << l, h = t.N << l;
  uint8_t code = 0;
  int own = 0;
#pragma unroll
  for (int sd = 0; sd < 4; ++sd) {
    const int di = sd == 1 ? 1 : sd == 3 ? -1 : 0;
    const int dj = sd == 0 ? 1 : sd == 2 ? -1 : 0;
    const int ni = i + di, nj = j + dj;
    int kind = 0, a = -1, b = -1;
    if (ni >= 0 && nj >= 0 && ni < w && nj < h) {
      const bool exists = l == 0 || is_flagged(t, l - 1, node_index(l - 1, ni >> 1, nj >> 1, t.M));
      if (exists) {
        const uint64_t q = node_index(l, ni, nj, t.M);
        if (!is_flagged(t, l, q)) {
          kind = 2;
          a = leaf_index(t, l, q);
        } else {
          kind = 3;
          int c0i, c0j, c1i, c1j;
          if (sd == 1 || sd == 3) {
            c0i = c1i = 2 * ni + (sd == 3 ? 1 : 0);
            c0j = 2 * nj;
            c1j = 2 * nj + 1;
          } else {
            c0j = c1j = 2 * nj + (sd == 2 ? 1 : 0);
            c0i = 2 * ni;
            c1i = 2 * ni + 1;
          }
          const uint64_t q0 = node_index(l + 1, c0i, c0j, t.M), q1 = node_index(l + 1, c1i, c1j, t.M);
          if (is_flagged(t, l + 1, q0) || is_flagged(t, l + 1, q1)) atomicOr(err, 1);
          a = leaf_index(t, l + 1, q0);
          b = leaf_index(t, l + 1, q1);
        }
      } else {
        // coarser: the level-(l-1) ancestor must exist (2:1 grading)
        const int la = l - 1;
        const bool up = la == 0 || is_flagged(t, la - 1, node_index(la - 1, ni >> 2, nj >> 2, t.M));
        if (!up) atomicOr(err, 1);
        kind = 1;
        a = leaf_index(t, la, node_index(la, ni >> 1, nj >> 1, t.M));
      }
    }
    nb[8 * k + 2 * sd] = a;
    nb[8 * k + 2 * sd + 1] = b;
    code |= uint8_t(kind << (2 * sd));
    own += kind == 3 ? 2 : (kind == 2 && (sd == 0 || sd == 1)) ? 1 : 0;
  }
  sk[k] = code;
  owned[k] = own;
}

__device__ __forceinline__ int owned_on(uint8_t code, int sd) {
  const int kind = (code >> (2 * sd)) & 3;
  return kind == 3 ? 2 : (kind == 2 && (sd == 0 || sd == 1)) ? 1 : 0;
}
__device__ __forceinline__ int owned_before(uint8_t code, int sd) {
  int s = 0;
  for (int q = 0; q < sd; ++q) s += owned_on(code, q);
  return s;
}

// The adaptive re-grid's extra per-leaf / per-segment statics, computed in
// the segment pass (one launch instead of four): the owned segments'
// geometry byte and (P2) topography limits, the leaf's side topography
// limits (P2) and its encode_pairing partners z* for two-segment sides
// (side_effective, solver_nonuniform.cpp:155-163: face_limit of region_topo).
struct SegExtras {
  uint8_t* geo;       // null: not fused
  double2* segz;      // P2 only
  double* zside;      // P2 only
  double* zpair;      // 4 per leaf
  const double* zp[16];  // the z encode-up pyramid per level (3 per node)
  const double* z;
  const int8_t* lvl;
  int L, M;
};

// Segment ids per leaf side + the owned segments' (left, right) leaves.
__global__ void k_segments(long long n, const int32_t* __restrict__ li,
                           const int32_t* __restrict__ lj, const int32_t* __restrict__ nb,
                           const uint8_t* __restrict__ sk, const int32_t* __restrict__ base,
                           int32_t* __restrict__ sid, int32_t* __restrict__ seg_l,
                           int32_t* __restrict__ seg_r, SegExtras ex) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint8_t code = sk[k];
  const bool fused = ex.geo != nullptr;
  int lk = 0, ik = 0, jk = 0;
  if (fused) {
    lk = ex.lvl[k];
    ik = li[k];
    jk = lj[k];
  }
  // an owned segment's statics from its two leaves (fused mode)
  auto statics = [&](int32_t q, int32_t a, int32_t b) {
    const int la = a == k ? lk : ex.lvl[a], ia = a == k ? ik : li[a], ja = a == k ? jk : lj[a];
    const int lb = b == k ? lk : ex.lvl[b], ib = b == k ? ik : li[b], jb = b == k ? jk : lj[b];
    const uint8_t gc = seg_geo_code(ex.L, la, ia, ja, lb, ib, jb);
    ex.geo[q] = gc;
    if (ex.segz) ex.segz[q] = seg_z2(gc, ex.z + 3 * (long long)a, ex.z + 3 * (long long)b);
  };
  for (int sd = 0; sd < 4; ++sd) {
    const int kind = (code >> (2 * sd)) & 3;
    int a = -1, b = -1;
    const int32_t n0 = nb[8 * k + 2 * sd], n1 = nb[8 * k + 2 * sd + 1];
    const bool mine_left = sd == 0 || sd == 1;
    if (kind == 3 || (kind == 2 && mine_left)) {
      const int32_t s0 = base[k] + owned_before(code, sd);
      a = s0;
      seg_l[s0] = mine_left ? int32_t(k) : n0;
      seg_r[s0] = mine_left ? n0 : int32_t(k);
      if (fused) statics(s0, mine_left ? int32_t(k) : n0, mine_left ? n0 : int32_t(k));
      if (kind == 3) {
        b = s0 + 1;
        seg_l[s0 + 1] = mine_left ? int32_t(k) : n1;
        seg_r[s0 + 1] = mine_left ? n1 : int32_t(k);
        if (fused) statics(s0 + 1, mine_left ? int32_t(k) : n1, mine_left ? n1 : int32_t(k));
      }
    } else if (kind == 2) {
      const int opp = (sd + 2) & 3;
      a = base[n0] + owned_before(sk[n0], opp);
    } else if (kind == 1) {
      const int opp = (sd + 2) & 3;
      const int t = (sd == 1 || sd == 3) ? (lj[k] & 1) : (li[k] & 1);
      a = base[n0] + owned_before(sk[n0], opp) + t;
    }
    sid[8 * k + 2 * sd] = a;
    sid[8 * k + 2 * sd + 1] = b;
    if (fused) {
      // k_zpair: the partner z* of a two-segment side
      double v = 0.0;
      if (kind == 3) {
        const int ni = ik + (sd == 1 ? 1 : sd == 3 ? -1 : 0);
        const int nj = jk + (sd == 0 ? 1 : sd == 2 ? -1 : 0);
        const double* p = ex.zp[lk] + 3 * node_index(lk, ni, nj, ex.M);
        v = face_val(P3{p[0], p[1], p[2]}, (sd + 2) & 3);
      }
      ex.zpair[4 * k + sd] = v;
    }
  }
  if (fused && ex.zside) side_z4(ex.z + 3 * k, ex.zside + 4 * k);
}

// Static per-segment geometry for the segment kernel (k_seg, P2 geometry):
// bit 0 x-normal; bits 1-2 / 3-4 the tangential offset code of the W/S and
// E/N leaf's limit point (0: centre of its face, 1: -1/4, 2: +1/4 of its
// size).  The segment centre (enumerate_faces, quadgrid.cpp:222-245) lies at
// the finer leaf's face centre, i.e. a quarter off the coarser leaf's.
__global__ void k_seg_geo(long long nseg, int L, const int32_t* __restrict__ seg_l,
                          const int32_t* __restrict__ seg_r, const int8_t* __restrict__ lvl,
                          const int32_t* __restrict__ li, const int32_t* __restrict__ lj,
                          uint8_t* __restrict__ geo, const long long* __restrict__ nsd) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= nseg || (nsd && q >= *nsd)) return;
  const int a = seg_l[q], b = seg_r[q];
  geo[q] = seg_geo_code(L, lvl[a], li[a], lj[a], lvl[b], li[b], lj[b]);
}

// Static topography limits of every segment (P2 geometry): z of each leaf's
// plane at the segment centre, evaluated exactly as k_seg's limit_rel would
// (limit_at, solver_nonuniform.cpp:52-66): the topography never changes on a
// static grid, so k_seg reads these 16 B instead of both leaves' z rows.
__global__ void k_seg_z(long long nseg, const int32_t* __restrict__ seg_l, const int32_t* __restrict__ seg_r,
                        const uint8_t* __restrict__ geo, const double* __restrict__ z, double2* __restrict__ out,
                        const long long* __restrict__ nsd) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= nseg || (nsd && q >= *nsd)) return;
  out[q] = seg_z2(geo[q], z + 3 * (long long)seg_l[q], z + 3 * (long long)seg_r[q]);
}

// ... and of every leaf side: z of the leaf's plane at its side midpoints
// (N E S W), as k_stage's side evaluation would compute it.
__global__ void k_side_z(long long n, const double* __restrict__ z, double* __restrict__ out) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  side_z4(z + 3 * k, out + 4 * k);
}

// --- scan -----------------------------------------------------------------
__global__ void k_block_sums(const int32_t* __restrict__ in, long long n,
                             long long* __restrict__ sums) {
  __shared__ long long s[32];
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long v = k < n ? in[k] : 0;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    long long x = threadIdx.x < (blockDim.x >> 5) ? s[threadIdx.x] : 0;
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (threadIdx.x == 0) sums[blockIdx.x] = x;
  }
}
__global__ void k_scan_sums(long long* sums, long long nb, long long* total) {
  __shared__ long long part[1024];
  __shared__ long long base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (long long b0 = 0; b0 < nb; b0 += blockDim.x) {
    const long long k = b0 + threadIdx.x;
    const long long v = k < nb ? sums[k] : 0;
    part[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < int(blockDim.x); o <<= 1) {
      const long long add = threadIdx.x >= unsigned(o) ? part[threadIdx.x - o] : 0;
      __syncthreads();
      part[threadIdx.x] += add;
      __syncthreads();
    }
    if (k < nb) sums[k] = base + part[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) base += part[threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = base;
}
__global__ void k_scan_apply(const int32_t* __restrict__ in, int32_t* __restrict__ out,
                             long long n, const long long* __restrict__ sums) {
  __shared__ long long s[1024];
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long v = k < n ? in[k] : 0;
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < int(blockDim.x); o <<= 1) {
    const long long add = threadIdx.x >= unsigned(o) ? s[threadIdx.x - o] : 0;
    __syncthreads();
    s[threadIdx.x] += add;
    __syncthreads();
  }
  if (k < n) out[k] = int32_t(sums[blockIdx.x] + s[threadIdx.x] - v);
}

// --- inflow targets (solver_nonuniform.cpp:611-628) ---------------------------
// The reference walks every fine cell of the rectangle to its containing leaf
// (QuadGrid::find_containing, quadgrid.cpp:62-69) and counts cells per leaf.
// A leaf's count is the area of the intersection of its fine-cell square with
// the rectangle, computed directly per leaf (integer, so identical).
__global__ void k_inflow_overlap(long long n, int L, const int8_t* __restrict__ lvl,
                                 const int32_t* __restrict__ li, const int32_t* __restrict__ lj, int i0,
                                 int j0, int i1, int j1, int32_t* __restrict__ cnt) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  cnt[k] = inflow_overlap(L, lvl[k], li[k], lj[k], i0, j0, i1, j1);
}

// Manning per leaf from a cell-centred raster (solver_nonuniform.cpp:575-584).
__global__ void k_manning(long long n, int L, double R, double x0, double y0,
                          const int8_t* __restrict__ lvl, const int32_t* __restrict__ li,
                          const int32_t* __restrict__ lj, const double* __restrict__ mr, int nc,
                          int nr, double xll, double yll, double cs, double uniform,
                          double* __restrict__ out) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  out[k] = manning_at(L, R, x0, y0, lvl[k], li[k], lj[k], mr, nc, nr, xll, yll, cs, uniform);
}

TopoIn topo_in(const Grid& g) {
  TopoIn t{};
  for (int l = 0; l < g.L; ++l) {
    t.flag[l] = g.flag[l].p;
    t.off[l] = g.off[l].p;
  }
  t.L = g.L;
  t.M = g.M;
  t.N = g.N;
  return t;
}

inline unsigned nblk(long long n, int t) { return unsigned((n + t - 1) / t); }

}  // namespace

// Exclusive scan; the total lands in *total_dev (device), no host sync.
void scan_exclusive_async(const int32_t* in, int32_t* out, int64_t n, long long* total_dev,
                          DBuf<long long>* scratch = nullptr) {
  cudaStream_t st = stream();
  const int T = 1024;
  const long long nb = (n + T - 1) / T;
  if (n == 0) {
    FM_CUDA(cudaMemsetAsync(total_dev, 0, sizeof(long long), st));
    return;
  }
  DBuf<long long> own;
  DBuf<long long>& sums = scratch ? *scratch : own;
  sums.ensure(std::max<long long>(nb, 1));
  k_block_sums<<<unsigned(nb), T, 0, st>>>(in, n, sums.p);
  FM_LAUNCHED();
  k_scan_sums<<<1, 1024, 0, st>>>(sums.p, nb, total_dev);
  FM_LAUNCHED();
  k_scan_apply<<<unsigned(nb), T, 0, st>>>(in, out, n, sums.p);
  FM_LAUNCHED();
}

int64_t scan_exclusive(const int32_t* in, int32_t* out, int64_t n) {
  DBuf<long long> total(1);
  scan_exclusive_async(in, out, n, total.p);
  long long tot = 0;
  total.download(&tot, 1);
  FM_CUDA(cudaStreamSynchronize(stream()));
  return tot;
}

void build_seg_geo(Sim& s) {
  s.seg_geo.ensure(std::max<int64_t>(s.nseg, 1));
  if (s.nseg) {
    k_seg_geo<<<nblk(s.nseg, 256), 256, 0, stream()>>>(s.nseg, s.L, s.seg_l.p, s.seg_r.p, s.lvl.p, s.li.p,
                                                      s.lj.p, s.seg_geo.p, s.nseg_lazy ? s.nseg_dev.p : nullptr);
    FM_LAUNCHED();
  }
}

// after the topography is final (initial conditions zero FV1/ACC's z slopes)
void build_seg_z(Sim& s) {
  if (s.p2 && s.n) {
    s.zside.ensure(4 * size_t(s.n));
    k_side_z<<<nblk(s.n, 256), 256, 0, stream()>>>(s.n, s.z.p, s.zside.p);
    FM_LAUNCHED();
  }
  if (s.nseg && s.p2) {
    s.segz.ensure(2 * size_t(s.nseg));
    k_seg_z<<<nblk(s.nseg, 256), 256, 0, stream()>>>(s.nseg, s.seg_l.p, s.seg_r.p, s.seg_geo.p, s.z.p,
                                                    reinterpret_cast<double2*>(s.segz.p),
                                                    s.nseg_lazy ? s.nseg_dev.p : nullptr);
    FM_LAUNCHED();
  }
}

void build_topology(Sim& s, const Grid& g, const double* const* zp) {
  FM_RANGE("build_topology");
  cudaStream_t st = stream();
  const long long n = s.n;
  s.nb.ensure(8 * n);
  s.sk.ensure(n);
  // adaptive re-grids keep the scratch (no allocation calls per adapt: the
  // host enqueues this work right after the adapt's sync, with the GPU idle)
  DBuf<int32_t> owned_tmp, base_tmp;
  DBuf<int32_t>& owned = s.adaptive ? s.topo_owned : owned_tmp;
  DBuf<int32_t>& base = s.adaptive ? s.topo_base : base_tmp;
  owned.ensure(n);
  base.ensure(n);
  // [0]: segment total (scan), [1]: the ungraded-grid error flag; one sync for both
  DBuf<long long> tot2(s.adaptive ? 0 : 2);
  // an adaptive re-grid keeps the total on the device and does not wait for
  // it: its grid is graded by construction (grade_flags in the adapt's
  // prefix), and the segment launches take an upper bound (a leaf is the
  // finer-or-equal side of at most one segment per side: nseg <= 4 n) with
  // the true count read on the device (NuView::nseg_dev)
  const bool lazy = s.adaptive;
  if (lazy) s.nseg_dev.ensure(2);
  long long* tot = lazy ? s.nseg_dev.p : tot2.p;
  FM_CUDA(cudaMemsetAsync(tot, 0, 2 * sizeof(long long), st));
  const TopoIn t = topo_in(g);
  k_topo<<<nblk(n, 256), 256, 0, st>>>(t, n, s.lvl.p, s.li.p, s.lj.p, s.nb.p, s.sk.p, owned.p,
                                        reinterpret_cast<int*>(tot + 1));
  FM_LAUNCHED();
  scan_exclusive_async(owned.p, base.p, n, tot, s.adaptive ? &s.topo_sums : nullptr);
  if (lazy) {
    s.nseg = std::max<int64_t>(4 * n, 1);
    s.nseg_lazy = true;
    FM_CUDA(cudaMemcpyAsync(&s.slots().nseg, tot, sizeof(long long), cudaMemcpyDeviceToHost, st));
  } else {
    long long h2[2] = {0, 0};
    tot2.download(h2, 2);
    FM_CUDA(cudaStreamSynchronize(st));
    s.nseg = h2[0];
    s.nseg_lazy = false;
    if (h2[1]) throw Error(FM_ERR_STRUCTURE, "non-uniform solvers require a graded (2:1) grid");
  }
  {
    s.sid.ensure(8 * n);
    s.seg_l.ensure(std::max<int64_t>(s.nseg, 1));
    s.seg_r.ensure(std::max<int64_t>(s.nseg, 1));
    SegExtras ex{};
    if (zp) {
      // the adaptive re-grid: the segment statics, side limits and pairing
      // partners in this pass (build_seg_geo / build_seg_z / k_zpair fused)
      s.seg_geo.ensure(std::max<int64_t>(s.nseg, 1));
      s.zpair.ensure(4 * size_t(n));
      ex.geo = s.seg_geo.p;
      if (s.p2) {
        s.segz.ensure(2 * size_t(std::max<int64_t>(s.nseg, 1)));
        s.zside.ensure(4 * size_t(n));
        ex.segz = reinterpret_cast<double2*>(s.segz.p);
        ex.zside = s.zside.p;
      }
      ex.zpair = s.zpair.p;
      for (int l = 0; l < s.L && l < 16; ++l) ex.zp[l] = zp[l];
      ex.z = s.z.p;
      ex.lvl = s.lvl.p;
      ex.L = s.L;
      ex.M = s.M;
    }
    k_segments<<<nblk(n, 256), 256, 0, st>>>(n, s.li.p, s.lj.p, s.nb.p, s.sk.p, base.p, s.sid.p,
                                              s.seg_l.p, s.seg_r.p, ex);
    FM_LAUNCHED();
    if (!zp) build_seg_geo(s);
    if (s.scheme != FM_ACC) s.segst.ensure(6 * size_t(std::max<int64_t>(s.nseg, 1)));
  }
}

void resolve_inflows(Sim& s, const Grid& g) {
  (void)g;
  cudaStream_t st = stream();
  s.infc.ensure(std::max<int64_t>(1, int64_t(s.ninflow) * s.n));
  if (s.ninflow == 0) s.infc.zero();
  for (int f = 0; f < s.ninflow; ++f) {
    const int* r = &s.rect[4 * f];
    k_inflow_overlap<<<nblk(s.n, 256), 256, 0, st>>>(s.n, s.L, s.lvl.p, s.li.p, s.lj.p, r[0], r[1], r[2],
                                                     r[3], s.infc.p + f * s.n);
    FM_LAUNCHED();
  }
}

void resolve_manning(Sim& s) {
  k_manning<<<nblk(s.n, 256), 256, 0, stream()>>>(
      s.n, s.L, s.R, s.x0, s.y0, s.lvl.p, s.li.p, s.lj.p, s.has_mr ? (s.mr_ext ? s.mr_ext : s.mr.p) : nullptr, s.mr_ncols,
      s.mr_nrows, s.mr_xll, s.mr_yll, s.mr_cs, s.manning, s.nman.p);
  FM_LAUNCHED();
}

}  // namespace fmh
