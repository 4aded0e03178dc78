// Dynamically adaptive MWDG2 / HWFV1 entirely on the device
// (AdaptiveSim, solver_adaptive.cpp).
//
// Every adapt (solver_adaptive.cpp:136-171) runs on the device over dense
// block-Morton pyramids, with no host round trip for data.  The per-level
// passes run each large level as one launch and all levels of <= 256 nodes in
// one single-CTA launch (run_levels); level-independent passes run every level
// in one launch (run_levels_flat):
//   norms        (:139-144) in k_mark_leaves_dn (exact max reductions)
//   encode_up    (:16-57)   k_mark_leaves + EncodeFlagBody per level, which
//   flag         (:59-73)   also flags the node (static topography significance
//                           precomputed once: max(a,b) >= eps <=> a >= eps || b >= eps)
//   closure      (detail_tree.cpp:56-64) and closes it over its children
//   buffer_ring  (:75-94)   inside grade_count_levels (ring = tmp)
//   grade_flags  (detail_tree.cpp:97-113) + leaf counts: grade_count_levels
//   assemble_grid(detail_tree.cpp:132-164): build_leaves (topography decode)
//   transfer     (:96-134)  k_transfer_leaves: one thread per new leaf walks
//                           its ancestor chain, decoding with stored or zero
//                           details; unchanged leaves keep their coefficients
//                           bit-for-bit (the encode_up copy of the old leaf IS
//                           the old value)
//   remap + rebuild_topology (:173-202, solver_nonuniform.cpp:521-527):
//                           the Manning values and inflow targets of the new
//                           leaves in the transfer's install, then
//                           build_topology with the encode_pairing partner z*
//                           of two-segment sides (region_topo,
//                           solver_nonuniform.cpp:80-89, from a z encode-up
//                           pyramid, ZpyrBody) and the segment statics written
//                           in its segment pass.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>

#include "fm_device.cuh"
#include "fm_sim.hpp"
#include "leafinfo.cuh"
#include "levels.cuh"

using namespace fmd;

namespace fmh {

bool geometry_is_p2(double R, double x0, double y0, int L, int M, int N);
void ic_surface_or_depth(Sim& s, const fm_sim_desc* d);
void ic_finish(Sim& s);

struct AdaptState {
  int kind = 0;
  double eps = 1e-3;
  std::vector<DBuf<uint8_t>> zsig;   // [L] static topography significance
  // [L+1] 0 unknown, 1 leaf, 2 internal: every level in one allocation
  // (known_all), so an adapt clears them all with one memset
  DBuf<uint8_t> known_all;
  std::vector<uint8_t*> known;
  std::vector<DBuf<double>> sc;      // [L+1] flow scaling, 9 per node
  std::vector<DBuf<double>> fdet;    // [L] flow details, 27 per node
  std::vector<DBuf<double>> zp;      // [L] z encode-up pyramid, 3 per node
  std::vector<DBuf<uint8_t>> tmp;    // [L] flags before the ring dilation
  DBuf<unsigned long long> norms;    // 3
  // the device-sized prefix of every adapt (encode up to the leaf list) as
  // one CUDA graph: dn[0] = current leaf count (set before each replay),
  // dn[1] = the new leaf count (read back after it)
  DBuf<long long> dn;
  cudaGraphExec_t prefix = nullptr;
  std::vector<const void*> prefix_key;  // the buffers the graph was captured on
  int64_t prefix_kernels = 0;
  ~AdaptState() {
    if (prefix) cudaGraphExecDestroy(prefix);
  }
};

void adaptive_destroy(AdaptState* a) { delete a; }

namespace {

inline unsigned nblk(uint64_t n, int t) { return unsigned((n + t - 1) / t); }

struct PtrTab {
  uint8_t* known[16];
  double* sc[16];
};

// max over the block of three non-negative values as bit patterns, one
// atomicMax per field (per-warp atomics on three addresses serialised ~9k
// atomics per adapt)
__device__ __forceinline__ void block_max3(double a, double b, double c, unsigned long long* out) {
  for (int o = 16; o; o >>= 1) {
    a = smax(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = smax(b, __shfl_xor_sync(0xffffffffu, b, o));
    c = smax(c, __shfl_xor_sync(0xffffffffu, c, o));
  }
  __shared__ unsigned long long sm[3][32];
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if ((threadIdx.x & 31) == 0) {
    sm[0][w] = dbits(a);
    sm[1][w] = dbits(b);
    sm[2][w] = dbits(c);
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    unsigned long long m = 0;
    for (int q = 0; q < nw; ++q) m = m > sm[threadIdx.x][q] ? m : sm[threadIdx.x][q];
    atomicMax(out + threadIdx.x, m);
  }
}

// the leaf count from the device (graph replays): grid-stride.  The current
// leaves into the pyramid (known = 1, their rows as level scaling) and, from
// the same rows, the norms (solver_adaptive.cpp:139-144): exact maxima over
// bit patterns, block-reduced, one atomic per block and field.
__global__ void k_mark_leaves_dn(const long long* __restrict__ dn, int M, const int8_t* __restrict__ lvl,
                                 const int32_t* __restrict__ li, const int32_t* __restrict__ lj,
                                 const double* __restrict__ u, PtrTab t, unsigned long long* norms) {
  const long long n = dn[0];
  double a = 0.0, b = 0.0, c = 0.0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const int l = lvl[k];
    const uint64_t node = node_index(l, li[k], lj[k], M);
    t.known[l][node] = 1;
    double* o = t.sc[l] + 9 * node;
    double r[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) r[q] = u[9 * k + q];
#pragma unroll
    for (int q = 0; q < 9; ++q) o[q] = r[q];
    a = smax(a, fabs(r[0]));
    b = smax(b, fabs(r[3]));
    c = smax(c, fabs(r[6]));
  }
  block_max3(a, b, c, norms);
}



__global__ void k_all_ones(uint64_t n, uint8_t* f) {
  const uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (k < n) f[k] = 1;
}

__global__ void k_leaf_ij(long long n, int L, int M, int8_t* lvl, int32_t* li, int32_t* lj) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int i, j;
  node_ij(L, uint64_t(k), M, i, j);
  lvl[k] = int8_t(L);
  li[k] = i;
  lj[k] = j;
}

// ---- level-fused passes ---------------------------------------------------
// The re-grid walks the pyramid level by level; the coarse levels are tiny
// (level l of one root block has 4^l nodes) and a launch per level makes the
// adapt launch-bound.  A pass therefore runs each large level as its own
// launch and all the small levels (<= kSmallNodes nodes) in ONE single-CTA
// launch that walks them in the pass's order with a __syncthreads between
// levels; per-level-independent passes run every level in one launch.  The
// per-node bodies are the kernels' previous bodies, unchanged.
#ifndef FM_SMALL_NODES
#define FM_SMALL_NODES 256
#endif
constexpr uint64_t kSmallNodes = FM_SMALL_NODES;
#ifndef FM_SMALL_THREADS
#define FM_SMALL_THREADS 256
#endif
constexpr int kMaxLv = 16;

struct Install {
  int8_t* lvl;
  int32_t* li;
  int32_t* lj;
  double* z;
  const double* gz;  // the grid's leaf topography
  // the new leaf set's Manning values and inflow target counts, computed as
  // each leaf is installed (resolve_manning / resolve_inflows fused)
  double* nman;
  const double* mr;  // cell-centred raster (null: uniform `manning`)
  int mr_nc, mr_nr, L, ninflow;
  double mr_xll, mr_yll, mr_cs, manning, R, x0, y0;
  int32_t* infc;     // ninflow x n
  long long n;
  int rect[4 * kMaxInflows];
};

struct LvTab {
  int L, M, N;
  uint8_t* known[kMaxLv + 1];
  double* sc[kMaxLv + 1];
  double* fdet[kMaxLv];
  const uint8_t* zsig[kMaxLv];
  uint8_t* flag[kMaxLv];
  uint8_t* tmp[kMaxLv];
  double* zp[kMaxLv];
  const int32_t* off[kMaxLv];
  const unsigned long long* norms;
  double eps;
  double* unew;
  const double* z;  // leaf topography (3 per leaf, device order)
  int zero_slopes;  // HWFV1: the leaves' z planes are taken with zero slopes
  int do_install;   // k_transfer_leaves also installs the leaf set (inst)
  Install inst;
  __host__ __device__ uint64_t nodes(int l) const { return uint64_t(M) * N << (2 * l); }
};

// encode_up + flag + ancestor_closure in ONE fine-to-coarse sweep
// (solver_adaptive.cpp:16-73, detail_tree.cpp:56-64): at level l a node that
// is not a current leaf and whose four children are known is encoded
// (encode_flow, wavelets.cpp:102-120); its flag is the static topography
// significance, or a flow detail of the node just encoded with d_hat >= eps
// (the norms are taken over the current leaves first), or -- the closure --
// any flagged child at l + 1, whose flags are final because the sweep
// visited level l + 1 before.  Equal to the three passes in turn.  Every
// load a node needs (its flags, the children's flags and rows) issues before
// the first store, and d_hat is taken from the details in registers: the
// sweep is a chain of levels, so each node's latency is on the critical path.
template <int KIND>
struct EncodeFlagBody {
  __device__ static void node(int l, uint64_t n, const LvTab& t) {
    uint8_t* kn = t.known[l];
    const uint8_t kself = kn[n];
    const uint32_t k4 = *reinterpret_cast<const uint32_t*>(t.known[l + 1] + 4 * n);
    const uint8_t zs = t.zsig[l][n];
    const uint32_t ct = l + 1 < t.L ? *reinterpret_cast<const uint32_t*>(t.tmp[l + 1] + 4 * n) : 0u;
    // the norms now, not after the stores below (which the compiler cannot
    // move them past): one round trip fewer on the level's critical path
    const double nrm[3] = {bitsd(t.norms[0]), bitsd(t.norms[1]), bitsd(t.norms[2])};
    uint8_t f = zs;  // (a non-zero significance value is kept as is)
    bool sig = false;
    const bool enc = kself == 0 && (k4 & 0xffu) && (k4 & 0xff00u) && (k4 & 0xff0000u) && (k4 & 0xff000000u);
    if (enc) {
      // the four children's rows are 36 contiguous, 16 B aligned doubles:
      // load them all before any store (the stores below could alias them)
      double ch[36];
      const double2* src = reinterpret_cast<const double2*>(t.sc[l + 1] + 36 * n);
#pragma unroll
      for (int q = 0; q < 18; ++q) {
        const double2 w = src[q];
        ch[2 * q] = w.x;
        ch[2 * q + 1] = w.y;
      }
#pragma unroll
      for (int fi = 0; fi < 3; ++fi) {
        P3 kids[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) kids[c] = P3{ch[9 * c + 3 * fi], ch[9 * c + 3 * fi + 1], ch[9 * c + 3 * fi + 2]};
        P3 p;
        double d[9];
        encode_k<KIND>(kids, p, d);
        t.sc[l][9 * n + 3 * fi] = p.c0;
        t.sc[l][9 * n + 3 * fi + 1] = p.cx;
        t.sc[l][9 * n + 3 * fi + 2] = p.cy;
#pragma unroll
        for (int q = 0; q < 9; ++q) t.fdet[l][27 * n + 9 * fi + q] = d[q];
        if (dhat(d, nrm[fi]) >= t.eps) sig = true;
      }
      kn[n] = 2;
    }
    if (!f && (sig || ct)) f = 1;
    t.tmp[l][n] = f;
  }
};

// buffer_ring, one level: dilate to the same-level 8-neighbourhood (:75-94),
// from the closed flags (tmp) into the grid's flags
// transfer as a walk per NEW leaf (one launch instead of one per level):
// from the level-0 scaling down the leaf's ancestor chain, decoding at each
// ancestor only the child on the path, with the stored flow details where the
// ancestor was internal (kInternal) and zero details otherwise — the
// reference's own DFS order (transfer, solver_adaptive.cpp:96-134).  A leaf that was
// an old leaf keeps its bits (:114-116).  Each child's decode is decode_k's
// arithmetic for that child, so this equals a level-by-level decode.
template <int KIND>
__global__ void __launch_bounds__(256) k_transfer_leaves(LvTab t, long long n, const int8_t* __restrict__ lvl,
                                                         const int32_t* __restrict__ li,
                                                         const int32_t* __restrict__ lj) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int l = lvl[k];
  const uint64_t nl = node_index(l, li[k], lj[k], t.M);
  double v[9];
  if (l > 0 && t.known[l][nl] == 1) {
    const double* o = t.sc[l] + 9 * nl;
#pragma unroll
    for (int q = 0; q < 9; ++q) v[q] = o[q];
  } else {
    const double* o = t.sc[0] + 9 * (nl >> (2 * l));
#pragma unroll
    for (int q = 0; q < 9; ++q) v[q] = o[q];
    // every ancestor's "internal" flag up front (independent loads, one
    // round trip for the whole chain), and each level's details prefetched
    // into L1 one level ahead of its decode
    uint32_t internal_mask = 0;
#pragma unroll
    for (int m = 0; m < kMaxLv; ++m)
      if (m < l && t.known[m][nl >> (2 * (l - m))] == 2) internal_mask |= 1u << m;
    auto prefetch_det = [&](int m) {
      if (m < l && ((internal_mask >> m) & 1u)) {
        const double* dd = t.fdet[m] + 27 * (nl >> (2 * (l - m)));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(dd));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(dd + 13));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(dd + 26));
      }
    };
    prefetch_det(0);
    for (int m = 0; m < l; ++m) {
      prefetch_det(m + 1);
      const uint64_t a = nl >> (2 * (l - m));
      const int c = int(nl >> (2 * (l - m - 1))) & 3;
      const bool internal = (internal_mask >> m) & 1u;
      const double* dd = t.fdet[m] + 27 * a;
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        double d[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) d[q] = internal ? dd[9 * f + q] : 0.0;
        const P3 o3 = decode_child_k<KIND>(P3{v[3 * f], v[3 * f + 1], v[3 * f + 2]}, d, c);
        v[3 * f] = o3.c0;
        v[3 * f + 1] = o3.cx;
        v[3 * f + 2] = o3.cy;
      }
    }
  }
  double* o = t.unew + 9 * k;
  if (t.do_install) {
    // the sim takes the new leaf set in the same pass (copy_leaves_from_grid)
    // and, for FV1, the piecewise-constant representation
    // (solver_adaptive.cpp:157-164: slopes of U and z zeroed)
    const double* zg = t.inst.gz + 3 * k;
    double* zo = t.inst.z + 3 * k;
    t.inst.lvl[k] = int8_t(l);
    t.inst.li[k] = li[k];
    t.inst.lj[k] = lj[k];
    zo[0] = zg[0];
    zo[1] = t.zero_slopes ? 0.0 : zg[1];
    zo[2] = t.zero_slopes ? 0.0 : zg[2];
    if (t.zero_slopes) v[1] = v[2] = v[4] = v[5] = v[7] = v[8] = 0.0;
    const Install& in = t.inst;
    if (in.nman) {
      const int i = li[k], j = lj[k];
      in.nman[k] = manning_at(in.L, in.R, in.x0, in.y0, l, i, j, in.mr, in.mr_nc, in.mr_nr, in.mr_xll,
                              in.mr_yll, in.mr_cs, in.manning);
      for (int f = 0; f < in.ninflow; ++f)
        in.infc[f * in.n + k] = inflow_overlap(in.L, l, i, j, in.rect[4 * f], in.rect[4 * f + 1],
                                               in.rect[4 * f + 2], in.rect[4 * f + 3]);
    }
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) o[q] = v[q];
}

// region_topo (solver_nonuniform.cpp:80-89) for every flagged node
template <int KIND>
struct ZpyrBody {
  __device__ static void node(int l, uint64_t n, const LvTab& t) {
    const int L = t.L;
    if ((l > 0 && !t.flag[l - 1][n >> 2]) || !t.flag[l][n]) return;
    P3 kids[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint64_t ch = 4 * n + c;
      const bool leaf = l + 1 == L || !t.flag[l + 1][ch];
      const double* s;
      if (leaf)
        s = t.z + 3 * (l + 1 < L ? t.off[l + 1][ch] : t.off[l][n] + c);
      else
        s = t.zp[l + 1] + 3 * ch;
      // FV1 leaves carry zero topography slopes (set by the transfer, +0 exactly)
      kids[c] = (leaf && t.zero_slopes) ? P3{s[0], 0.0, 0.0} : P3{s[0], s[1], s[2]};
    }
    const P3 p = encode_parent_k<KIND>(kids);
    t.zp[l][3 * n] = p.c0;
    t.zp[l][3 * n + 1] = p.cx;
    t.zp[l][3 * n + 2] = p.cy;
  }
};

template <class Body>
__global__ void k_level(LvTab t, int l) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n < t.nodes(l)) Body::node(l, n, t);
}
// the small levels from `first` to `last` (either direction), one CTA
template <class Body>
__global__ void __launch_bounds__(FM_SMALL_THREADS) k_levels_small(LvTab t, int first, int last) {
  const int step = last >= first ? 1 : -1;
  for (int l = first;; l += step) {
    const uint64_t nodes = t.nodes(l);
    for (uint64_t n = threadIdx.x; n < nodes; n += blockDim.x) Body::node(l, n, t);
    __syncthreads();
    if (l == last) break;
  }
}
// every level at once (per-level independent bodies): blockIdx.y = level
template <class Body>
__global__ void k_levels_flat(LvTab t, int l0) {
  const int l = l0 + blockIdx.y;
  const uint64_t nodes = t.nodes(l);
  for (uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; n < nodes;
       n += uint64_t(gridDim.x) * blockDim.x)
    Body::node(l, n, t);
}

// The middle levels of a vertical pass (each node reads only its children or
// its parent) as subtrees: CTA b owns the level-r node b and walks its
// subtree's levels r..rt in the pass's order with a block barrier between
// levels — the level-(l+1) results it reads were written by its own threads,
// so no launch boundary (and its ~µs gap) is needed per level.  rt: the
// finest level with at most kTreeThreads nodes per subtree.
#ifndef FM_TREE_THREADS
#define FM_TREE_THREADS 64
#endif
constexpr int kTreeThreads = FM_TREE_THREADS;
template <class Body>
__global__ void __launch_bounds__(kTreeThreads) k_levels_tree(LvTab t, int r, int rt, int fine_to_coarse) {
  const uint64_t b = blockIdx.x;
  for (int q = 0; q <= rt - r; ++q) {
    const int l = fine_to_coarse ? rt - q : r + q;
    const uint64_t per = uint64_t(1) << (2 * (l - r));
    for (uint64_t j = threadIdx.x; j < per; j += blockDim.x) Body::node(l, b * per + j, t);
    __syncthreads();
  }
}

// Run Body over levels lo..hi in the given order: the small coarse levels
// (<= kSmallNodes nodes) in one single-CTA launch, the middle levels as
// subtrees in one launch (k_levels_tree), the fine levels one launch each.
template <class Body>
void run_levels(const LvTab& t, int lo, int hi, bool fine_to_coarse) {
  if (hi < lo) return;
  cudaStream_t st = stream();
  int ls = -1;  // the finest small level
  for (int l = lo; l <= hi; ++l)
    if (t.nodes(l) <= kSmallNodes) ls = l;
  const int r = std::max(ls + 1, lo);  // subtree roots
  int rt = r - 1;                      // the finest subtree level
  for (int l = r; l <= hi; ++l)
    if ((uint64_t(1) << (2 * (l - r))) <= uint64_t(kTreeThreads)) rt = l;
  if (rt == r) rt = r - 1;  // one level: a plain launch
  auto big = [&](int l) {
    k_level<Body><<<nblk(t.nodes(l), 256), 256, 0, st>>>(t, l);
    FM_LAUNCHED();
  };
  auto small = [&](int a, int b) {
    k_levels_small<Body><<<1, FM_SMALL_THREADS, 0, st>>>(t, a, b);
    FM_LAUNCHED();
  };
  auto tree = [&]() {
    if (rt < r) return;
    k_levels_tree<Body><<<unsigned(t.nodes(r)), kTreeThreads, 0, st>>>(t, r, rt, fine_to_coarse ? 1 : 0);
    FM_LAUNCHED();
  };
  const int fb = std::max(rt + 1, r);  // the first per-level launch
  if (fine_to_coarse) {
    for (int l = hi; l >= fb; --l) big(l);
    tree();
    if (ls >= lo) small(ls, lo);
  } else {
    if (ls >= lo) small(lo, ls);
    tree();
    for (int l = fb; l <= hi; ++l) big(l);
  }
}
template <class Body>
void run_levels_flat(const LvTab& t, int lo, int hi) {
  if (hi < lo) return;
  const unsigned bx = unsigned(std::min<uint64_t>(nblk(t.nodes(hi), 256), 148 * 8));
  k_levels_flat<Body><<<dim3(bx, hi - lo + 1), 256, 0, stream()>>>(t, lo);
  FM_LAUNCHED();
}

LvTab lv_tab(Sim& s, Grid& g, AdaptState& a) {
  LvTab t{};
  t.L = g.L;
  t.M = g.M;
  t.N = g.N;
  for (int l = 0; l <= g.L; ++l) {
    t.known[l] = a.known[l];
    t.sc[l] = a.sc[l].p;
  }
  for (int l = 0; l < g.L; ++l) {
    t.fdet[l] = a.fdet[l].p;
    t.zsig[l] = a.zsig[l].p;
    t.flag[l] = g.flag[l].p;
    t.tmp[l] = a.tmp[l].p;
    t.zp[l] = a.zp[l].p;
    t.off[l] = g.off.size() > size_t(l) ? g.off[l].p : nullptr;
  }
  t.norms = a.norms.p;
  t.eps = a.eps;
  t.z = s.z.p;
  return t;
}

// rebuild_topology + encode_pairing partners (the remap of the Manning values
// and inflow targets ran in the transfer): one segment pass also writes the
// segment statics, the side limits and the z* partners from the z encode-up
// pyramid (built in the adapt's prefix graph, right after the leaf list)
void refresh_topology(Sim& s) {
  Grid& g = *s.grid;
  AdaptState& a = *s.ad;
  const double* zp[16] = {};
  for (int l = 0; l < s.L && l < 16; ++l) zp[l] = a.zp[l].p;
  build_topology(s, g, zp);
}

}  // namespace

// make_adaptive_sim (solver_adaptive.cpp:209-236)
void adaptive_init(Sim& s, const fm_sim_desc* d, const fm_raster* dem) {
  cudaStream_t st = stream();
  if (d->max_level < 0) throw Error(FM_ERR_CONFIG, "adaptive solvers require max_level");
  if (d->adapt_every < 1) throw Error(FM_ERR_CONFIG, "adapt_every must be >= 1");
  if (d->max_level < 1) throw Error(FM_ERR_CONFIG, "adaptive solvers need max_level >= 1");
  const int kind = d->solver == FM_MWDG2 ? FM_MW : FM_HW;
  s.adapt_every = d->adapt_every;
  s.ad = new AdaptState();
  AdaptState& a = *s.ad;
  a.kind = kind;
  a.eps = d->epsilon;
  // the topography tree, once (topography_tree, detail_tree.cpp:166-170)
  s.grid = std::make_unique<Grid>();
  Grid& g = *s.grid;
  g.graded = true;
  mra_encode(dem, d->max_level, d->epsilon, kind, g, nullptr);
  const int L = g.L;
  s.L = L;
  s.M = g.M;
  s.N = g.N;
  s.R = g.R;
  s.x0 = g.x0;
  s.y0 = g.y0;
  s.p2 = geometry_is_p2(s.R, s.x0, s.y0, L, s.M, s.N);
  a.zsig.resize(L);
  a.known.resize(L + 1);
  a.sc.resize(L + 1);
  a.fdet.resize(L);
  a.zp.resize(L);
  a.tmp.resize(L);
  {
    std::vector<uint64_t> off(L + 2, 0);  // 16 B aligned levels
    for (int l = 0; l <= L; ++l) off[l + 1] = (off[l] + (uint64_t(g.M) * g.N << (2 * l)) + 15) & ~uint64_t(15);
    a.known_all.alloc(off[L + 1]);
    for (int l = 0; l <= L; ++l) a.known[l] = a.known_all.p + off[l];
  }
  for (int l = 0; l <= L; ++l) {
    const uint64_t nodes = uint64_t(g.M) * g.N << (2 * l);
    a.sc[l].alloc(9 * nodes);
    if (l < L) {
      a.zsig[l].alloc(nodes);
      FM_CUDA(cudaMemcpyAsync(a.zsig[l].p, g.flag[l].p, nodes, cudaMemcpyDeviceToDevice, st));
      a.fdet[l].alloc(27 * nodes);
      a.zp[l].alloc(3 * nodes);
      a.tmp[l].alloc(nodes);
    }
  }
  a.norms.alloc(3);
  a.dn.alloc(2);
  // the initial uniform level-L grid (make_uniform_quadgrid) with nug0.topo =
  // the projected fine planes (not a decode)
  for (int l = 0; l < L; ++l) {
    k_all_ones<<<nblk(g.nodes(l), 256), 256, 0, st>>>(g.nodes(l), g.flag[l].p);
    FM_LAUNCHED();
  }
  grade_count_levels(g, true);
  build_leaves(g);
  s.n = g.nleaves;
  s.lvl.alloc(s.n);
  s.li.alloc(s.n);
  s.lj.alloc(s.n);
  k_leaf_ij<<<nblk(s.n, 256), 256, 0, st>>>(s.n, L, s.M, s.lvl.p, s.li.p, s.lj.p);
  FM_LAUNCHED();
  project_planes(dem, L, s.M, s.N, s.z);
  // make_nonuniform_sim on that grid (solver_nonuniform.cpp:558-636)
  s.u.alloc(9 * s.n);
  s.us.alloc(9 * s.n);
  s.u.zero();
  if (d->initial_depth_raster) {
    const fm_raster* hr = d->initial_depth_raster;
    if (hr->ncols != dem->ncols || hr->nrows != dem->nrows)
      throw Error(FM_ERR_CONFIG, "initial_depth_raster geometry must match the DEM");
    DBuf<double> fine;
    project_planes(hr, L, s.M, s.N, fine);  // level-L leaves: the planes themselves
    FM_CUDA(cudaMemcpy2DAsync(s.u.p, 9 * sizeof(double), fine.p, 3 * sizeof(double),
                              3 * sizeof(double), s.n, cudaMemcpyDeviceToDevice, st));
  }
  if (!d->initial_depth_raster) ic_surface_or_depth(s, d);
  ic_finish(s);
  for (int f = 0; f < s.ninflow; ++f) {
    const int* r = &s.rect[4 * f];
    if (r[0] < 0 || r[1] < 0 || r[2] >= (s.M << L) || r[3] >= (s.N << L))
      throw Error(FM_ERR_CONFIG, "inflow region outside the domain");
  }
  s.nman.alloc(s.n);
  resolve_manning(s);
  resolve_inflows(s, g);
  build_topology(s, g);
  adaptive_adapt(s, 0.0);
}


// FM_ADAPT_PROFILE=1: per-phase device time of every adapt on stderr (CUDA
// events between the phases; diagnostics only)
namespace {
struct PhaseClock {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<const char*> name;
  explicit PhaseClock(cudaStream_t st) : st_(st) {
    const char* e = std::getenv("FM_ADAPT_PROFILE");
    on = e && e[0] == '1';
    mark("start");
  }
  void mark(const char* n) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st_);
    ev.push_back(e);
    name.push_back(n);
  }
  ~PhaseClock() {
    if (!on) return;
    cudaEventSynchronize(ev.back());
    for (size_t k = 1; k < ev.size(); ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[k - 1], ev[k]);
      std::fprintf(stderr, "%s=%.1f ", name[k], 1000.0 * ms);
    }
    float tot = 0.f;
    cudaEventElapsedTime(&tot, ev.front(), ev.back());
    std::fprintf(stderr, "| adapt %.1f us\n", 1000.0 * tot);
    for (auto e : ev) cudaEventDestroy(e);
  }

 private:
  cudaStream_t st_;
};
}  // namespace

namespace {
__global__ void k_set_dn(long long* dn, long long n) { dn[0] = n; }

// The device-sized part of an adapt, in the reference's order: encode_up +
// flag + closure (one sweep), buffer_ring, grade_flags + leaf counts, and
// leaves_from_flags + assemble_grid (build_leaves_device).  The current leaf
// count is read from dn[0], the new one written to dn[1]; every buffer is of
// fixed size (the dense pyramids; leaf arrays of capacity M N 4^L), so the
// launches are captured once in a CUDA graph and replayed every adapt.
void launch_prefix(Sim& s, Grid& g, AdaptState& a, const LvTab& tab) {
  cudaStream_t st = stream();
  const int L = g.L;
  FM_CUDA(cudaMemsetAsync(a.known_all.p, 0, a.known_all.n, st));
  PtrTab pt{};
  for (int l = 0; l <= L; ++l) {
    pt.known[l] = a.known[l];
    pt.sc[l] = a.sc[l].p;
  }
  // the current leaves into the pyramid and the norms over them
  // (solver_adaptive.cpp:139-144)
  FM_CUDA(cudaMemsetAsync(a.norms.p, 0, 3 * sizeof(unsigned long long), st));
  k_mark_leaves_dn<<<148 * 4, 256, 0, st>>>(a.dn.p, s.M, s.lvl.p, s.li.p, s.lj.p, s.u.p, pt, a.norms.p);
  FM_LAUNCHED();
  // encode_up + flag + closure, one sweep (into tmp)
  if (a.kind == 0)
    run_levels<EncodeFlagBody<0>>(tab, 0, L - 1, true);
  else
    run_levels<EncodeFlagBody<1>>(tab, 0, L - 1, true);
  // buffer_ring (tmp -> the grid's flags) is taken inside the grading pass
  // (each node's own flag = the ring dilation of tmp at its level); its
  // ancestor closure is subsumed by grading: the gather form of grade_flags
  // sets G(l) = F(l) | any child G(l+1) | ring, bottom-up, so
  // G(closure(F)) = G(F) level by level (the closure's child term is
  // contained in G's)
  std::vector<const uint8_t*> ring(L);
  for (int l = 0; l < L; ++l) ring[l] = a.tmp[l].p;
  // grade + counts + leaves + exact topography (assemble_grid)
  grade_and_build_leaves_device(g, &ring, a.dn.p + 1);
  // region_topo (solver_nonuniform.cpp:80-89) of every flagged node over the
  // new leaves' topography (the grid's leaf planes; HWFV1 takes them with
  // zero slopes, as the sim's own copy will hold them)
  LvTab zt = tab;
  zt.z = g.lf_z.p;
  zt.zero_slopes = s.scheme != FM_DG2 ? 1 : 0;
  if (a.kind == 0)
    run_levels<ZpyrBody<0>>(zt, 0, L - 1, true);
  else
    run_levels<ZpyrBody<1>>(zt, 0, L - 1, true);
}

void adapt_prefix(Sim& s, Grid& g, AdaptState& a, const LvTab& tab) {
  cudaStream_t st = stream();
  k_set_dn<<<1, 1, 0, st>>>(a.dn.p, s.n);
  FM_LAUNCHED();
  const std::vector<const void*> key = {s.u.p, s.lvl.p, s.li.p, s.lj.p, g.lf_l.p, g.lf_i.p, g.lf_j.p, g.lf_z.p};
  if (!a.prefix || key != a.prefix_key) {
    if (a.prefix) cudaGraphExecDestroy(a.prefix);
    a.prefix = nullptr;
    const int64_t before = launches();
    cudaGraph_t gr;
    FM_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    launch_prefix(s, g, a, tab);
    FM_CUDA(cudaStreamEndCapture(st, &gr));
    FM_CUDA(cudaGraphInstantiate(&a.prefix, gr, 0));
    cudaGraphDestroy(gr);
    a.prefix_key = key;
    a.prefix_kernels = launches() - before;
  }
  FM_CUDA(cudaGraphLaunch(a.prefix, st));
  count_graph_launches(a.prefix_kernels);
}
}  // namespace

namespace {
__global__ void k_count_encoded(LvTab t, int l0, unsigned long long* out) {
  const int l = l0 + blockIdx.y;
  const uint64_t nodes = t.nodes(l);
  unsigned long long c = 0;
  for (uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; n < nodes;
       n += uint64_t(gridDim.x) * blockDim.x)
    c += t.known[l][n] == 2;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
}  // namespace

// The last adapt's sizes for SURVEY §8 d4's adapt bytes: parents encoded in
// encode_up (N_enc) and the internal nodes of the pyramid (N_int).
void adaptive_stats(Sim& s, int64_t* n_enc, int64_t* n_int) {
  if (!s.adaptive || !s.ad) throw Error(FM_ERR_CONFIG, "adapt_stats: not an adaptive simulation");
  Grid& g = *s.grid;
  AdaptState& a = *s.ad;
  LvTab tab = lv_tab(s, g, a);
  DBuf<unsigned long long> c(1);
  c.zero();
  const unsigned bx = unsigned(std::min<uint64_t>(nblk(g.nodes(g.L - 1), 256), 148 * 8));
  k_count_encoded<<<dim3(bx, g.L), 256, 0, stream()>>>(tab, 0, c.p);
  FM_LAUNCHED();
  unsigned long long h = 0;
  c.download(&h, 1);
  FM_CUDA(cudaStreamSynchronize(stream()));
  if (n_enc) *n_enc = int64_t(h);
  if (n_int) {
    int64_t ni = 0;
    for (int l = 0; l < g.L; ++l) ni += int64_t(g.nodes(l));
    *n_int = ni;
  }
}

void adaptive_adapt_begin(Sim& s) {
  Grid& g = *s.grid;
  AdaptState& a = *s.ad;
  LvTab tab = lv_tab(s, g, a);
  // everything up to the new leaf list, one graph replay (adapt_prefix); the
  // new leaf count is read back with the caller's next host sync
  adapt_prefix(s, g, a, tab);
  FM_CUDA(cudaMemcpyAsync(&s.slots().n_new, a.dn.p + 1, sizeof(long long), cudaMemcpyDeviceToHost, stream()));
}

void adaptive_adapt_finish(Sim& s, double t) {
  FM_RANGE("adapt");
  s.ref_perm_ok = false;  // the leaf set changes
  ++s.leaf_gen;
  cudaStream_t st = stream();
  PhaseClock pc(st);
  Grid& g = *s.grid;
  AdaptState& a = *s.ad;
  const long long n_dev = s.slots().n_new;
  g.nleaves = n_dev;
  g.lf_l.n = g.lf_i.n = g.lf_j.n = size_t(n_dev);
  g.lf_z.n = 3 * size_t(n_dev);
  // transfer the flow onto the new leaves, straight into U (the old leaves'
  // rows are in the encode-up pyramid since the prefix), and install the
  // new leaf set into the sim in the same pass; buffers only grow
  const int64_t n_new = g.nleaves;
  s.u.ensure(9 * n_new);
  s.us.ensure(9 * n_new);
  s.n = n_new;
  s.lvl.ensure(s.n);
  s.li.ensure(s.n);
  s.lj.ensure(s.n);
  s.z.ensure(3 * s.n);
  LvTab tab = lv_tab(s, g, a);
  tab.unew = s.u.p;
  tab.do_install = 1;
  s.nman.ensure(s.n);
  s.infc.ensure(std::max<int64_t>(1, int64_t(s.ninflow) * s.n));
  if (s.ninflow == 0) s.infc.zero();
  Install in{};
  in.lvl = s.lvl.p;
  in.li = s.li.p;
  in.lj = s.lj.p;
  in.z = s.z.p;
  in.gz = g.lf_z.p;
  in.nman = s.nman.p;
  in.mr = s.has_mr ? (s.mr_ext ? s.mr_ext : s.mr.p) : nullptr;
  in.mr_nc = s.mr_ncols;
  in.mr_nr = s.mr_nrows;
  in.L = s.L;
  in.ninflow = s.ninflow;
  in.mr_xll = s.mr_xll;
  in.mr_yll = s.mr_yll;
  in.mr_cs = s.mr_cs;
  in.manning = s.manning;
  in.R = s.R;
  in.x0 = s.x0;
  in.y0 = s.y0;
  in.infc = s.infc.p;
  in.n = s.n;
  for (int q = 0; q < 4 * s.ninflow && q < 4 * kMaxInflows; ++q) in.rect[q] = s.rect[q];
  tab.inst = in;
  tab.zero_slopes = s.scheme != FM_DG2 ? 1 : 0;
  if (n_new) {
    if (a.kind == 0)
      k_transfer_leaves<0><<<nblk(n_new, 256), 256, 0, st>>>(tab, n_new, g.lf_l.p, g.lf_i.p, g.lf_j.p);
    else
      k_transfer_leaves<1><<<nblk(n_new, 256), 256, 0, st>>>(tab, n_new, g.lf_l.p, g.lf_i.p, g.lf_j.p);
    FM_LAUNCHED();
  }
  pc.mark("transfer");
  refresh_topology(s);
  pc.mark("topology");
  s.fv1_in_star = false;
  for (auto& gx : s.gexec) {
    if (gx) cudaGraphExecDestroy(gx);
    gx = nullptr;
  }
  s.element_log.emplace_back(t, s.n);  // s.n is known on the host: no sync here
}

void adaptive_adapt(Sim& s, double t) {
  adaptive_adapt_begin(s);
  FM_CUDA(cudaStreamSynchronize(stream()));
  s.settle_nseg();
  adaptive_adapt_finish(s, t);
  // an API-level adapt leaves the host's segment count exact (the device
  // loop settles it at its own syncs instead)
  FM_CUDA(cudaStreamSynchronize(stream()));
  s.settle_nseg();
}

}  // namespace fmh
