// Dynamically adaptive MWDG2 / HWFV1 entirely on the device
// (AdaptiveSim, solver_adaptive.cpp).
//
// Every adapt (solver_adaptive.cpp:136-171) runs as level-by-level kernels
// over dense block-Morton pyramids, with no host round trip for data:
//   encode_up    (:16-57)   k_mark_leaves + k_encode_up per level
//   norms        (:139-144) k_norms (exact max reductions)
//   flag         (:59-73)   k_flag per level (static topography significance
//                           precomputed once: max(a,b) >= eps <=> a >= eps || b >= eps)
//   closure      (detail_tree.cpp:56-64) k_closure per level
//   buffer_ring  (:75-94)   k_ring per level, then closure again
//   grade_flags  (detail_tree.cpp:97-113) + leaf counts: grade_count_levels
//   assemble_grid(detail_tree.cpp:132-164): build_leaves (topography decode)
//   transfer     (:96-134)  k_transfer per level: flow decode top-down with
//                           stored or zero details; unchanged leaves keep
//                           their coefficients bit-for-bit (the encode_up
//                           copy of the old leaf IS the old value)
//   remap + rebuild_topology (:173-202, solver_nonuniform.cpp:521-527):
//                           resolve_manning, resolve_inflows, build_topology,
//                           and the encode_pairing partner z* of two-segment
//                           sides (region_topo, solver_nonuniform.cpp:80-89)
//                           from a z encode-up pyramid (k_zpyr, k_zpair).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "fm_device.cuh"
#include "fm_sim.hpp"

using namespace fmd;

namespace fmh {

bool geometry_is_p2(double R, double x0, double y0, int L, int M, int N);
void ic_surface_or_depth(Sim& s, const fm_sim_desc* d);
void ic_finish(Sim& s);

struct AdaptState {
  int kind = 0;
  double eps = 1e-3;
  std::vector<DBuf<uint8_t>> zsig;   // [L] static topography significance
  std::vector<DBuf<uint8_t>> known;  // [L+1] 0 unknown, 1 leaf, 2 internal
  std::vector<DBuf<double>> sc;      // [L+1] flow scaling, 9 per node
  std::vector<DBuf<double>> fdet;    // [L] flow details, 27 per node
  std::vector<DBuf<double>> fs;      // [L] top-down flow scratch, 9 per node
  std::vector<DBuf<double>> zp;      // [L] z encode-up pyramid, 3 per node
  std::vector<DBuf<uint8_t>> tmp;    // [L] ring scratch
  DBuf<unsigned long long> norms;    // 3
};

void adaptive_destroy(AdaptState* a) { delete a; }

namespace {

inline unsigned nblk(uint64_t n, int t) { return unsigned((n + t - 1) / t); }

struct PtrTab {
  uint8_t* known[16];
  double* sc[16];
};

__global__ void k_mark_leaves(long long n, int M, const int8_t* __restrict__ lvl,
                              const int32_t* __restrict__ li, const int32_t* __restrict__ lj,
                              const double* __restrict__ u, PtrTab t) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int l = lvl[k];
  const uint64_t node = node_index(l, li[k], lj[k], M);
  t.known[l][node] = 1;
  double* o = t.sc[l] + 9 * node;
#pragma unroll
  for (int q = 0; q < 9; ++q) o[q] = u[9 * k + q];
}

template <int KIND>
__global__ void k_encode_up(uint64_t nodes, uint8_t* __restrict__ kn, const uint8_t* __restrict__ kn1,
                            double* __restrict__ sc, const double* __restrict__ sc1,
                            double* __restrict__ det) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= nodes || kn[n] != 0) return;
  const uint32_t k4 = *reinterpret_cast<const uint32_t*>(kn1 + 4 * n);
  if ((k4 & 0xffu) == 0 || (k4 & 0xff00u) == 0 || (k4 & 0xff0000u) == 0 || (k4 & 0xff000000u) == 0) return;
  // encode_flow (wavelets.cpp:102-120): h, qx, qy independently
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    P3 kids[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double* s = sc1 + 9 * (4 * n + c) + 3 * f;
      kids[c] = P3{s[0], s[1], s[2]};
    }
    P3 p;
    double d[9];
    encode_k<KIND>(kids, p, d);
    sc[9 * n + 3 * f] = p.c0;
    sc[9 * n + 3 * f + 1] = p.cx;
    sc[9 * n + 3 * f + 2] = p.cy;
#pragma unroll
    for (int q = 0; q < 9; ++q) det[27 * n + 9 * f + q] = d[q];
  }
  kn[n] = 2;
}

__global__ void k_norms(long long n, const double* __restrict__ u, unsigned long long* out) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double a = 0.0, b = 0.0, c = 0.0;
  if (k < n) {
    a = fabs(u[9 * k]);
    b = fabs(u[9 * k + 3]);
    c = fabs(u[9 * k + 6]);
  }
  for (int o = 16; o; o >>= 1) {
    a = smax(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = smax(b, __shfl_xor_sync(0xffffffffu, b, o));
    c = smax(c, __shfl_xor_sync(0xffffffffu, c, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, dbits(a));
    atomicMax(out + 1, dbits(b));
    atomicMax(out + 2, dbits(c));
  }
}

// solver_adaptive.cpp:59-73 without the closure
__global__ void k_flag(uint64_t nodes, const uint8_t* __restrict__ zsig, const uint8_t* __restrict__ kn,
                       const double* __restrict__ det, const unsigned long long* __restrict__ norms,
                       double eps, uint8_t* __restrict__ flag) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= nodes) return;
  uint8_t f = zsig[n];
  if (!f && kn[n] == 2) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double d[9];
#pragma unroll
      for (int r = 0; r < 9; ++r) d[r] = det[27 * n + 9 * q + r];
      if (dhat(d, bitsd(norms[q])) >= eps) f = 1;
    }
  }
  flag[n] = f;
}

// ancestor_closure, one level: parent |= any child (detail_tree.cpp:56-64)
__global__ void k_closure(uint64_t nodes, uint8_t* __restrict__ flag, const uint8_t* __restrict__ flag1) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= nodes) return;
  if (*reinterpret_cast<const uint32_t*>(flag1 + 4 * n)) flag[n] = 1;
}

// buffer_ring, one level: dilate to the same-level 8-neighbourhood (:75-94)
__global__ void k_ring(uint64_t nodes, int l, int M, int N, const uint8_t* __restrict__ flag,
                       uint8_t* __restrict__ out) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= nodes) return;
  uint8_t f = flag[n];
  if (!f) {
    int i, j;
    node_ij(l, n, M, i, j);
    const int w = M << l, h = N << l;
    for (int dj = -1; dj <= 1 && !f; ++dj)
      for (int di = -1; di <= 1; ++di) {
        const int ni = i + di, nj = j + dj;
        if (ni < 0 || nj < 0 || ni >= w || nj >= h) continue;
        if (flag[node_index(l, ni, nj, M)]) {
          f = 1;
          break;
        }
      }
  }
  out[n] = f;
}

// transfer (solver_adaptive.cpp:96-134), one level of the new tree.
template <int KIND>
__global__ void k_transfer(uint64_t nodes, int l, int L, const uint8_t* __restrict__ flp,
                           const uint8_t* __restrict__ fl, const uint8_t* __restrict__ fl1,
                           const uint8_t* __restrict__ kn, const uint8_t* __restrict__ kn1,
                           const double* __restrict__ sc, const double* __restrict__ sc1,
                           const double* __restrict__ det, const double* __restrict__ vin,
                           double* __restrict__ vout, const int32_t* __restrict__ off,
                           const int32_t* __restrict__ off1, double* __restrict__ u) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= nodes) return;
  if (l > 0 && !flp[n >> 2]) return;  // not in the new tree
  double v[9];
  const double* src = l == 0 ? sc + 9 * n : vin + 9 * n;
#pragma unroll
  for (int q = 0; q < 9; ++q) v[q] = src[q];
  if (!fl[n]) {  // a level-0 leaf (deeper leaves are written by their parent)
    if (l == 0) {
      double* o = u + 9 * off[n];
#pragma unroll
      for (int q = 0; q < 9; ++q) o[q] = v[q];  // sc[0] = old leaf value when it was one
    }
    return;
  }
  const bool internal = kn[n] == 2;
  double kids[4][9];
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    double d[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) d[q] = internal ? det[27 * n + 9 * f + q] : 0.0;
    P3 out[4];
    decode_k<KIND>(P3{v[3 * f], v[3 * f + 1], v[3 * f + 2]}, d, out);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      kids[c][3 * f] = out[c].c0;
      kids[c][3 * f + 1] = out[c].cx;
      kids[c][3 * f + 2] = out[c].cy;
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint64_t ch = 4 * n + c;
    const bool leaf = l + 1 == L || !fl1[ch];
    if (leaf) {
      const int32_t at = l + 1 < L ? off1[ch] : off[n] + c;
      double* o = u + 9 * at;
      const bool old = kn1[ch] == 1;  // surviving leaf keeps its bits (:114-116)
#pragma unroll
      for (int q = 0; q < 9; ++q) o[q] = old ? sc1[9 * ch + q] : kids[c][q];
    } else {
      double* o = vout + 9 * ch;
#pragma unroll
      for (int q = 0; q < 9; ++q) o[q] = kids[c][q];
    }
  }
}

// Piecewise-constant representation after an adapt (solver_adaptive.cpp:157-164)
__global__ void k_zero_slopes(long long n, double* __restrict__ z, double* __restrict__ u) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  z[3 * k + 1] = z[3 * k + 2] = 0.0;
  u[9 * k + 1] = u[9 * k + 2] = 0.0;
  u[9 * k + 4] = u[9 * k + 5] = 0.0;
  u[9 * k + 7] = u[9 * k + 8] = 0.0;
}

// region_topo (solver_nonuniform.cpp:80-89) for every flagged node: the
// encode of its four children, each a leaf's z or a deeper region.
template <int KIND>
__global__ void k_zpyr(uint64_t nodes, int l, int L, const uint8_t* __restrict__ flp,
                       const uint8_t* __restrict__ fl, const uint8_t* __restrict__ fl1,
                       const double* __restrict__ zp1, double* __restrict__ zp,
                       const int32_t* __restrict__ off, const int32_t* __restrict__ off1,
                       const double* __restrict__ z) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= nodes) return;
  if ((l > 0 && !flp[n >> 2]) || !fl[n]) return;
  P3 kids[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint64_t ch = 4 * n + c;
    const bool leaf = l + 1 == L || !fl1[ch];
    const double* s;
    if (leaf)
      s = z + 3 * (l + 1 < L ? off1[ch] : off[n] + c);
    else
      s = zp1 + 3 * ch;
    kids[c] = P3{s[0], s[1], s[2]};
  }
  const P3 p = encode_parent_k<KIND>(kids);
  zp[3 * n] = p.c0;
  zp[3 * n + 1] = p.cx;
  zp[3 * n + 2] = p.cy;
}

struct ZpTab {
  const double* zp[16];
};

// partner z* for two-segment sides: max(me.z, face_limit(region_topo, opposite))
// (side_effective, solver_nonuniform.cpp:155-163) — the face_limit part.
__global__ void k_zpair(long long n, int M, const int8_t* __restrict__ lvl,
                        const int32_t* __restrict__ li, const int32_t* __restrict__ lj,
                        const uint8_t* __restrict__ sk, ZpTab t, double* __restrict__ zpair) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int l = lvl[k], i = li[k], j = lj[k];
  const uint8_t code = sk[k];
#pragma unroll
  for (int sd = 0; sd < 4; ++sd) {
    double v = 0.0;
    if (((code >> (2 * sd)) & 3) == 3) {
      const int ni = i + (sd == 1 ? 1 : sd == 3 ? -1 : 0);
      const int nj = j + (sd == 0 ? 1 : sd == 2 ? -1 : 0);
      const double* p = t.zp[l] + 3 * node_index(l, ni, nj, M);
      v = face_val(P3{p[0], p[1], p[2]}, (sd + 2) & 3);
    }
    zpair[4 * k + sd] = v;
  }
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

void copy_leaves_from_grid(Sim& s, const Grid& g) {
  cudaStream_t st = stream();
  s.n = g.nleaves;
  s.lvl.alloc(s.n);
  s.li.alloc(s.n);
  s.lj.alloc(s.n);
  s.z.alloc(3 * s.n);
  FM_CUDA(cudaMemcpyAsync(s.lvl.p, g.lf_l.p, s.n, cudaMemcpyDeviceToDevice, st));
  FM_CUDA(cudaMemcpyAsync(s.li.p, g.lf_i.p, 4 * s.n, cudaMemcpyDeviceToDevice, st));
  FM_CUDA(cudaMemcpyAsync(s.lj.p, g.lf_j.p, 4 * s.n, cudaMemcpyDeviceToDevice, st));
  FM_CUDA(cudaMemcpyAsync(s.z.p, g.lf_z.p, 24 * s.n, cudaMemcpyDeviceToDevice, st));
}

// remap_after_adapt + rebuild_topology + encode_pairing partners
void refresh_topology(Sim& s) {
  cudaStream_t st = stream();
  Grid& g = *s.grid;
  AdaptState& a = *s.ad;
  s.nman.alloc(s.n);
  resolve_manning(s);
  resolve_inflows(s, g);
  build_topology(s, g);
  // z encode-up over the new leaves, then the partner values
  const int L = s.L;
  for (int l = L - 1; l >= 0; --l) {
    const uint64_t nodes = g.nodes(l);
    const bool last = l + 1 == L;
    if (a.kind == 0)
      k_zpyr<0><<<nblk(nodes, 256), 256, 0, st>>>(nodes, l, L, l ? g.flag[l - 1].p : nullptr, g.flag[l].p,
                                                  last ? nullptr : g.flag[l + 1].p,
                                                  last ? nullptr : a.zp[l + 1].p, a.zp[l].p, g.off[l].p,
                                                  last ? nullptr : g.off[l + 1].p, s.z.p);
    else
      k_zpyr<1><<<nblk(nodes, 256), 256, 0, st>>>(nodes, l, L, l ? g.flag[l - 1].p : nullptr, g.flag[l].p,
                                                  last ? nullptr : g.flag[l + 1].p,
                                                  last ? nullptr : a.zp[l + 1].p, a.zp[l].p, g.off[l].p,
                                                  last ? nullptr : g.off[l + 1].p, s.z.p);
    FM_LAUNCHED();
  }
  ZpTab t{};
  for (int l = 0; l < L; ++l) t.zp[l] = a.zp[l].p;
  s.zpair.alloc(4 * s.n);
  k_zpair<<<nblk(s.n, 256), 256, 0, st>>>(s.n, s.M, s.lvl.p, s.li.p, s.lj.p, s.sk.p, t, s.zpair.p);
  FM_LAUNCHED();
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
  a.fs.resize(L);
  a.zp.resize(L);
  a.tmp.resize(L);
  for (int l = 0; l <= L; ++l) {
    const uint64_t nodes = uint64_t(g.M) * g.N << (2 * l);
    a.known[l].alloc(nodes);
    a.sc[l].alloc(9 * nodes);
    if (l < L) {
      a.zsig[l].alloc(nodes);
      FM_CUDA(cudaMemcpyAsync(a.zsig[l].p, g.flag[l].p, nodes, cudaMemcpyDeviceToDevice, st));
      a.fdet[l].alloc(27 * nodes);
      a.fs[l].alloc(9 * nodes);
      a.zp[l].alloc(3 * nodes);
      a.tmp[l].alloc(nodes);
    }
  }
  a.norms.alloc(3);
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

void adaptive_adapt(Sim& s, double t) {
  s.ref_perm_ok = false;  // the leaf set changes
  cudaStream_t st = stream();
  Grid& g = *s.grid;
  AdaptState& a = *s.ad;
  const int L = g.L;
  // encode_up
  for (int l = 0; l <= L; ++l) a.known[l].zero();
  PtrTab pt{};
  for (int l = 0; l <= L; ++l) {
    pt.known[l] = a.known[l].p;
    pt.sc[l] = a.sc[l].p;
  }
  k_mark_leaves<<<nblk(s.n, 256), 256, 0, st>>>(s.n, s.M, s.lvl.p, s.li.p, s.lj.p, s.u.p, pt);
  FM_LAUNCHED();
  for (int l = L - 1; l >= 0; --l) {
    const uint64_t nodes = g.nodes(l);
    if (a.kind == 0)
      k_encode_up<0><<<nblk(nodes, 256), 256, 0, st>>>(nodes, a.known[l].p, a.known[l + 1].p, a.sc[l].p,
                                                        a.sc[l + 1].p, a.fdet[l].p);
    else
      k_encode_up<1><<<nblk(nodes, 256), 256, 0, st>>>(nodes, a.known[l].p, a.known[l + 1].p, a.sc[l].p,
                                                        a.sc[l + 1].p, a.fdet[l].p);
    FM_LAUNCHED();
  }
  // norms over the current leaves
  a.norms.zero();
  k_norms<<<nblk(s.n, 256), 256, 0, st>>>(s.n, s.u.p, a.norms.p);
  FM_LAUNCHED();
  // flag + closure
  for (int l = 0; l < L; ++l) {
    k_flag<<<nblk(g.nodes(l), 256), 256, 0, st>>>(g.nodes(l), a.zsig[l].p, a.known[l].p, a.fdet[l].p,
                                                   a.norms.p, a.eps, g.flag[l].p);
    FM_LAUNCHED();
  }
  for (int l = L - 1; l >= 1; --l) {
    k_closure<<<nblk(g.nodes(l - 1), 256), 256, 0, st>>>(g.nodes(l - 1), g.flag[l - 1].p, g.flag[l].p);
    FM_LAUNCHED();
  }
  // buffer_ring + closure
  for (int l = 0; l < L; ++l) {
    k_ring<<<nblk(g.nodes(l), 256), 256, 0, st>>>(g.nodes(l), l, g.M, g.N, g.flag[l].p, a.tmp[l].p);
    FM_LAUNCHED();
    std::swap(g.flag[l], a.tmp[l]);
  }
  for (int l = L - 1; l >= 1; --l) {
    k_closure<<<nblk(g.nodes(l - 1), 256), 256, 0, st>>>(g.nodes(l - 1), g.flag[l - 1].p, g.flag[l].p);
    FM_LAUNCHED();
  }
  // grade + counts + leaves + exact topography (assemble_grid)
  grade_count_levels(g, true);
  build_leaves(g);
  // transfer the flow onto the new leaves
  const int64_t n_new = g.nleaves;
  DBuf<double> u_new(9 * n_new);
  for (int l = 0; l < L; ++l) {
    const uint64_t nodes = g.nodes(l);
    const bool last = l + 1 == L;
    auto launch = [&](auto kind_tag) {
      constexpr int K = decltype(kind_tag)::value;
      k_transfer<K><<<nblk(nodes, 256), 256, 0, st>>>(
          nodes, l, L, l ? g.flag[l - 1].p : nullptr, g.flag[l].p, last ? nullptr : g.flag[l + 1].p,
          a.known[l].p, a.known[l + 1].p, a.sc[l].p, a.sc[l + 1].p, a.fdet[l].p,
          l ? a.fs[l].p : nullptr, last ? nullptr : a.fs[l + 1].p, g.off[l].p,
          last ? nullptr : g.off[l + 1].p, u_new.p);
    };
    if (a.kind == 0)
      launch(std::integral_constant<int, 0>{});
    else
      launch(std::integral_constant<int, 1>{});
    FM_LAUNCHED();
  }
  s.u = std::move(u_new);
  s.us.alloc(9 * n_new);
  copy_leaves_from_grid(s, g);
  if (s.scheme != FM_DG2) {
    k_zero_slopes<<<nblk(s.n, 256), 256, 0, st>>>(s.n, s.z.p, s.u.p);
    FM_LAUNCHED();
  }
  refresh_topology(s);
  s.fv1_in_star = false;
  for (auto& g : s.gexec) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
  FM_CUDA(cudaStreamSynchronize(st));
  s.element_log.emplace_back(t, s.n);
}

}  // namespace fmh
