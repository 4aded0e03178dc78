// Static multiresolution analysis on sm_100a.
//
// Replaces generate_static_grid (detail_tree.cpp:172-178) and its stages:
//   project_raster      field.cpp:64-117     -> fused into k_encode_tiles
//   build_detail_tree   detail_tree.cpp:10-54 -> k_dem_stats (+ k_field_norm_fix) + k_encode_tiles
//   flag_significant    detail_tree.cpp:66-74 -> sig flags in k_encode_tiles
//   ancestor_closure +  detail_tree.cpp:56-64,
//   grade_flags                      :97-113 -> k_grade_count (one gather pass per level)
//   leaves_from_flags + make_quadgrid +
//   assemble_grid       detail_tree.cpp:115-164, quadgrid.cpp:85-110 -> k_level0_offsets + k_topdown
//
// Layout: every pyramid level is a dense array in block-Morton order (see
// fmd::node_index) so the four children of node n are 4n..4n+3: the encode
// reads 96 contiguous bytes per parent and the flags of a sibling quad are
// one 32-bit word.  Leaves come out in global Morton order of their SW fine
// corner (the depth-first order of the tree) with a dense per-level offset
// pyramid that maps any node to its leaf index in O(1) (replacing the
// reference's unordered_map index).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>

#include "fm_device.cuh"
#include "levels.cuh"
#include "fm_internal.hpp"

using namespace fmd;

namespace fmh {

namespace {

constexpr int kMaxL = 16;

__device__ __forceinline__ unsigned long long ordered_bits(double v) {
  const unsigned long long u = dbits(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_ordered(unsigned long long u) {
  return bitsd((u >> 63) ? (u & 0x7fffffffffffffffull) : ~u);
}

constexpr int kNodataSeen = 1, kBig = 2;

struct Scalars {
  unsigned long long vmax_ord;  // ordered max over non-nodata vertices
  unsigned long long norm_bits; // max |c0| (non-negative)
  int err;                      // 1: non-finite vertex
  int flags;                    // kNodataSeen | kBig (k_dem_stats)
  double wall;
  double norm;
  int redo;                     // the speculative encode met a nodata / non-finite / huge vertex
  int pad;
};

// field.cpp:48-54 (nodata wall) — max over the non-nodata vertex samples.
__global__ void k_vertex_max(const double* __restrict__ v, size_t n, double nodata, Scalars* s) {
  double m = -INFINITY;
  int bad = 0;
  for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < n;
       k += size_t(gridDim.x) * blockDim.x) {
    const double x = v[k];
    if (x != nodata) {
      m = smax(m, x);
      if (!isfinite(x)) bad = 1;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const double y = __shfl_xor_sync(0xffffffffu, m, o);
    m = smax(m, y);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&s->vmax_ord, ordered_bits(m));
    if (bad) atomicOr(&s->err, 1);
  }
}

struct VertexView {
  const double* v;
  int ncols, nrows, n, m;  // n = ncols-1 elements east, m = nrows-1 north
  double nodata;
  double wall;
  __device__ __forceinline__ double at(int row, int col) const {
    const double x = v[size_t(row) * ncols + col];
    return x == nodata ? wall : x;
  }
  // the value as stored (the speculative encode checks every vertex for
  // nodata itself and reruns the exact path if it meets one)
  __device__ __forceinline__ double raw(int row, int col) const { return v[size_t(row) * ncols + col]; }
  // field.cpp:64-91: element (i, j), edge-replicated beyond the raster.
  __device__ __forceinline__ P3 plane(int i, int j) const {
    const int ie = min(i, n - 1), je = min(j, m - 1);
    const int rs = nrows - 1 - je, rn = rs - 1;
    return project4(at(rn, ie), at(rn, ie + 1), at(rs, ie), at(rs, ie + 1));
  }
};

__global__ void k_wall(Scalars* s) {
  double z = from_ordered(s->vmax_ord);
  if (!isfinite(z)) z = 0.0;
  s->wall = z + 100.0;
  // k_dem_stats' norm left out the cells with a nodata vertex: redo it
  if (s->flags & kNodataSeen) s->norm_bits = 0;
}

// One pass over the elements for the static MRA: the nodata-wall maximum
// (field.cpp:48-54), the non-finite check, and field_norm
// (detail_tree.cpp:22-23).  Each element checks its SW vertex (plus the north
// row and east column at the raster's edges), so every vertex is checked once;
// the norm is taken over the raw vertex values, which is field_norm exactly
// when the DEM has no nodata vertex (otherwise k_wall resets it and
// k_field_norm_fix recomputes it with the wall).  kBig marks a vertex above
// 1e300 in magnitude: the encode then keeps its zero filter taps.
__global__ void k_dem_stats(VertexView vv, Scalars* s) {
  double m = -INFINITY, nm = 0.0;
  int bad = 0, fl = 0;
  auto chk = [&](double x) {
    if (x != vv.nodata) {
      m = smax(m, x);
      if (!isfinite(x)) bad = 1;
      if (fabs(x) > 1e300) fl |= kBig;
    } else {
      fl |= kNodataSeen;
    }
  };
  // element rows over CTAs, columns over threads (coalesced, no index division)
  for (int j = blockIdx.x; j < vv.m; j += gridDim.x) {
    const int rs = vv.nrows - 1 - j, rn = rs - 1;
    const double* vn = vv.v + size_t(rn) * vv.ncols;
    const double* vs = vv.v + size_t(rs) * vv.ncols;
    for (int i = threadIdx.x; i < vv.n; i += blockDim.x) {
      const double nw = vn[i], ne = vn[i + 1], sw = vs[i], se = vs[i + 1];
      chk(sw);
      if (i == vv.n - 1) chk(se);
      if (rn == 0) {
        chk(nw);
        if (i == vv.n - 1) chk(ne);
      }
      nm = smax(nm, fabs(0.25 * (ne + nw + se + sw)));  // project4's c0 (field.cpp:15)
    }
  }
  for (int o = 16; o; o >>= 1) {
    m = smax(m, __shfl_xor_sync(0xffffffffu, m, o));
    nm = smax(nm, __shfl_xor_sync(0xffffffffu, nm, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    fl |= __shfl_xor_sync(0xffffffffu, fl, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&s->vmax_ord, ordered_bits(m));
    if (nm > 0.0) atomicMax(&s->norm_bits, dbits(nm));
    if (bad) atomicOr(&s->err, 1);
    if (fl) atomicOr(&s->flags, fl);
  }
}

// detail_tree.cpp:22-23 — field_norm = max |c0| over the fine elements.
__device__ __forceinline__ void k_field_norm_body(VertexView vv, Scalars* s) {
  vv.wall = s->wall;
  const size_t total = size_t(vv.n) * vv.m;
  double m = 0.0;
  for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < total;
       k += size_t(gridDim.x) * blockDim.x) {
    const int i = int(k % size_t(vv.n)), j = int(k / size_t(vv.n));
    const P3 p = vv.plane(i, j);
    m = smax(m, fabs(p.c0));
  }
  for (int o = 16; o; o >>= 1) m = smax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&s->norm_bits, dbits(m));
}

// field_norm again, with the wall, only when the DEM has nodata vertices (see k_dem_stats)
__global__ void k_field_norm_fix(VertexView vv, Scalars* s) {
  if (!(s->flags & kNodataSeen)) return;
  k_field_norm_body(vv, s);
}

__global__ void k_norm_final(Scalars* s) { s->norm = bitsd(s->norm_bits); }

struct EncParams {
  VertexView vv;             // FROM_VERTICES
  const double* sc_in;       // input scaling (3 per node) at level lev_in
  double* sc_out;            // tile-root scaling (3 per node) at level lev_in - T
  double* det[kMaxL];        // per level, 9 per node
  uint8_t* flag[kMaxL];      // per level, significance
  double* dmx[kMaxL];        // SPEC: per level, max |d| (the numerator of d_hat)
  Scalars* scal;
  double eps;
  int lev_in, T, M, kind;
};

// One CTA encodes a tile of 4^T input nodes up T levels (detail_tree.cpp:34-51),
// writing details + significance (detail_tree.cpp:66-72) for every parent and
// the tile-root scaling.  Thread t owns first-level parent t of the tile: it
// builds its four children itself (projecting them from the DEM vertices when
// FROM_VERTICES) so the finest, largest level never touches shared memory;
// higher levels go through a 4^(T-1)-entry shared buffer.
// Details are staged in shared memory and leave the CTA as contiguous 16 B
// vectors: a level's parents of one tile are contiguous in the block-Morton
// layout, so the tile's 9 x count doubles are one contiguous range (direct
// 72 B-strided per-thread stores cost ~3x the bytes in DRAM writes).
__device__ __forceinline__ void store_details(const double* __restrict__ sdet, double* __restrict__ o,
                                              int count, int tid, int nthr) {
  const int total = 9 * count;
  if ((reinterpret_cast<uintptr_t>(o) & 15) || (total & 1)) {  // a single odd-placed node
    for (int e = tid; e < total; e += nthr) o[e] = sdet[e];
    return;
  }
  const double2* src = reinterpret_cast<const double2*>(sdet);
  double2* dst = reinterpret_cast<double2*>(o);
  for (int e = tid; e < total / 2; e += nthr) dst[e] = src[e];
}

// The same with one bulk (TMA) copy from shared to global memory issued by
// thread 0 instead of every thread's 16 B load / store loop (when the range
// is 16 B aligned and a multiple of 16 B; otherwise store_details).  Thread 0
// must call bulk_read_done before the staging buffer is written again.
#ifndef FM_ENC_BULK
#define FM_ENC_BULK 1
#endif
__device__ __forceinline__ void store_details_bulk(const double* __restrict__ sdet, double* __restrict__ o,
                                                   int count, int tid, int nthr) {
  const unsigned bytes = 72u * unsigned(count);
  if (!FM_ENC_BULK || (reinterpret_cast<uintptr_t>(o) & 15) || (bytes & 15)) {
    store_details(sdet, o, count, tid, nthr);
    return;
  }
  if (tid == 0) {
    const unsigned src = static_cast<unsigned>(__cvta_generic_to_shared(sdet));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o), "r"(src), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}
__device__ __forceinline__ void bulk_read_done(int tid) {
  if (FM_ENC_BULK && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

#ifndef FM_ENC_MINB
#define FM_ENC_MINB 6  // 40 registers (A/B on B200: MINB 5 -> 6: MRA 1.427 -> 1.402 ms; 4: 1.471)
#endif
#ifndef FM_ENC_T
#define FM_ENC_T 5  // levels per encode pass (4^(T-1) threads per CTA)
#endif
__device__ __forceinline__ double max_abs9(const double d[9]) {
  double m = 0.0;
#pragma unroll
  for (int n = 0; n < 9; ++n) m = smax(m, fabs(d[n]));
  return m;
}
// SPEC (speculative single DEM read): the DEM statistics are not known yet,
// so the encode assumes what holds for every DEM without nodata, non-finite
// or |z| > 1e300 vertices -- no wall, zero taps dropped -- and checks that
// assumption on every vertex it reads (redo if it fails: the caller reruns
// the exact two-pass path).  It takes field_norm (max |c0| over the fine
// planes, detail_tree.cpp:22-23) from the planes it projects, and writes
// max |d| per node instead of the flag; k_sig_from_dmx forms
// d_hat = max|d| / max(1, norm) >= eps once the norm is complete, the same
// operations as dhat() (wavelets.cpp:137-149).
template <bool FROM_VERTICES, bool SPEC>
__global__ void __launch_bounds__(256, FM_ENC_MINB) k_encode_tiles(EncParams p) {
  extern __shared__ double smem[];
  const int nthr = blockDim.x;
  P3* sbuf = reinterpret_cast<P3*>(smem);
  double* sdet = smem + 3 * nthr;  // 9 per first-level parent
  const int tid = threadIdx.x;
  const uint64_t tile = blockIdx.x;
  const double norm = SPEC ? 0.0 : p.scal->norm;
  // every input finite (a non-finite vertex fails the build) and bounded
  const bool skip0 = SPEC || !(p.scal->flags & kBig);
  // a register copy: writing into the by-value parameter struct would make
  // every thread spill the whole 344-byte EncParams to local memory
  VertexView vv = p.vv;
  if constexpr (FROM_VERTICES && !SPEC) vv.wall = p.scal->wall;
  // SPEC: a nodata vertex reads as NaN, which the vertex check turns into a redo
  if constexpr (FROM_VERTICES && SPEC) vv.wall = __longlong_as_double(0x7ff8000000000000ll);

  // first level: parent (lev_in - 1), local index tid
  int lev = p.lev_in - 1;
  const uint64_t par0 = tile << (2 * (p.T - 1));
  const uint64_t par = par0 + uint64_t(tid);
  P3 kids[4];
  if constexpr (FROM_VERTICES) {
    // the four children (2I + dx, 2J + dy) share a 3 x 3 vertex block: nine
    // loads instead of sixteen.  Edge replication (VertexView::plane) clamps
    // the element column / row; a clamped second child reuses the first's.
    int I, J;
    node_ij(p.lev_in - 1, par, p.M, I, J);
    const int ia = min(2 * I, vv.n - 1), ib = min(2 * I + 1, vv.n - 1);
    const int ja = min(2 * J, vv.m - 1), jb = min(2 * J + 1, vv.m - 1);
    const int rsa = vv.nrows - 1 - ja, rsb = vv.nrows - 1 - jb;
    const int rows[3] = {rsa, rsa - 1, rsb - 1};  // south to north
    const int cols[3] = {ia, ia + 1, ib + 1};      // west to east
    double V[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) V[r][c] = SPEC ? vv.raw(rows[r], cols[c]) : vv.at(rows[r], cols[c]);
    if constexpr (SPEC) {
      bool bad = false;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) bad |= (V[r][c] == vv.nodata) | !(fabs(V[r][c]) <= 1e300);
      if (bad) atomicOr(&p.scal->redo, 1);
    }
    const bool xs = ib != ia, ys = jb != ja;
    if (xs && ys) {
      // away from the raster's east / north edge: fixed offsets, no selects
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int ox = k & 1, oy = k >> 1;
        kids[k] = project4(V[oy + 1][ox], V[oy + 1][ox + 1], V[oy][ox], V[oy][ox + 1]);  // nw ne sw se
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool sx = (k & 1) && xs, sy = (k >> 1) && ys;  // shifted one column / row
        double q[2][2];  // [south, north][west, east]
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b)
            q[a][b] = sy ? (sx ? V[1 + a][1 + b] : V[1 + a][b]) : (sx ? V[a][1 + b] : V[a][b]);
        kids[k] = project4(q[1][0], q[1][1], q[0][0], q[0][1]);  // nw ne sw se
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double* s = p.sc_in + 3 * (4 * par + k);
      kids[k] = P3{s[0], s[1], s[2]};
    }
  }
  if constexpr (SPEC && FROM_VERTICES) {
    // field_norm over this tile's fine planes: block maximum, one atomic
    double nm = smax(smax(fabs(kids[0].c0), fabs(kids[1].c0)), smax(fabs(kids[2].c0), fabs(kids[3].c0)));
    for (int o = 16; o; o >>= 1) nm = smax(nm, __shfl_xor_sync(0xffffffffu, nm, o));
    double* red = smem;  // free until the first sbuf / sdet write below
    if ((tid & 31) == 0) red[tid >> 5] = nm;
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < (nthr >> 5); ++w) nm = smax(nm, red[w]);
      if (nm > 0.0) atomicMax(&p.scal->norm_bits, dbits(nm));
    }
    __syncthreads();
  }
  P3 par_s;
  double d[9];
  encode_b(kids, p.kind, skip0, par_s, d);
#pragma unroll
  for (int n = 0; n < 9; ++n) sdet[9 * tid + n] = d[n];
  if constexpr (SPEC)
    p.dmx[lev][par] = max_abs9(d);
  else
    p.flag[lev][par] = dhat(d, norm) >= p.eps ? 1 : 0;
  if (p.T == 1) {
    double* o = p.sc_out + 3 * par;
    o[0] = par_s.c0;
    o[1] = par_s.cx;
    o[2] = par_s.cy;
  } else {
    sbuf[tid] = par_s;
  }
  __syncthreads();
  store_details_bulk(sdet, p.det[lev] + 9 * par0, nthr, tid, nthr);
  if (p.T == 1) {
    bulk_read_done(tid);
    return;
  }
  int count = nthr;  // nodes at `lev`
  for (int t = 1; t < p.T; ++t) {
    --lev;
    count >>= 2;
    P3 mine;
    const bool have = tid < count;
    const uint64_t node0 = tile << (2 * (p.T - 1 - t));
    if (have) {
#pragma unroll
      for (int k = 0; k < 4; ++k) kids[k] = sbuf[4 * tid + k];
      encode_b(kids, p.kind, skip0, mine, d);
      if constexpr (SPEC)
        p.dmx[lev][node0 + tid] = max_abs9(d);
      else
        p.flag[lev][node0 + tid] = dhat(d, norm) >= p.eps ? 1 : 0;
    }
    bulk_read_done(tid);  // the previous level's bulk copy has read sdet
    __syncthreads();  // sbuf reads and the previous sdet stores are done
    if (have) {
      sbuf[tid] = mine;
#pragma unroll
      for (int n = 0; n < 9; ++n) sdet[9 * tid + n] = d[n];
    }
    __syncthreads();
    store_details_bulk(sdet, p.det[lev] + 9 * node0, count, tid, nthr);
  }
  bulk_read_done(tid);
  if (tid == 0) {
    double* o = p.sc_out + 3 * tile;
    o[0] = sbuf[0].c0;
    o[1] = sbuf[0].cx;
    o[2] = sbuf[0].cy;
  }
}

// flag_significant (detail_tree.cpp:66-74) from the speculative encode's
// max |d|: d_hat = max|d| / max(1, norm) >= eps, every level in one launch.
struct DmxLevels {
  const double* dmx[kMaxL];
  uint8_t* flag[kMaxL];
};
// The divisor is one value for the whole pass, so its reciprocal is
// computed once and each quotient is nvcc's fast-path sequence (zdiv2's
// argument: bit-identical to `/` inside the window, checked by
// fm_selftest(2)); four nodes per thread as 2 x 16 B loads and one 4 B store.
__device__ __forceinline__ uint8_t sig_of(double m, double den, double y, bool den_ok, double eps) {
  const double q = (m == 0.0) ? m : (den_ok && div_fast_ok(m)) ? quot_ieee(m, den, y) : m / den;
  return q >= eps ? 1 : 0;
}
__global__ void k_sig_from_dmx(DmxLevels t, int M, int N, const Scalars* __restrict__ s, double eps) {
  const int l = blockIdx.y;
  const uint64_t nodes = uint64_t(M) * N << (2 * l);
  const double norm = bitsd(s->norm_bits);
  const double den = smax(1.0, norm);
  const double y = recip_ieee(den);
  const bool den_ok = div_fast_ok(den);
  const double* dm = t.dmx[l];
  uint8_t* fl = t.flag[l];
  const uint64_t quads = nodes / 4;
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < quads;
       q += uint64_t(gridDim.x) * blockDim.x) {
    const double2 a = reinterpret_cast<const double2*>(dm)[2 * q], b = reinterpret_cast<const double2*>(dm)[2 * q + 1];
    const uint32_t w = uint32_t(sig_of(a.x, den, y, den_ok, eps)) | (uint32_t(sig_of(a.y, den, y, den_ok, eps)) << 8) |
                       (uint32_t(sig_of(b.x, den, y, den_ok, eps)) << 16) |
                       (uint32_t(sig_of(b.y, den, y, den_ok, eps)) << 24);
    reinterpret_cast<uint32_t*>(fl)[q] = w;
  }
  // the level's remainder (fewer than four nodes: M N odd at level 0)
  for (uint64_t n = 4 * quads + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; n < nodes;
       n += uint64_t(gridDim.x) * blockDim.x)
    fl[n] = sig_of(dm[n], den, y, den_ok, eps);
}

// L = 0: the fine field is the coarse field.
__global__ void k_copy_fine(VertexView vv, const Scalars* __restrict__ s, double* coarse, int M,
                            uint64_t total) {
  vv.wall = s->wall;
  const uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (k >= total) return;
  int i, j;
  node_ij(0, k, M, i, j);
  const P3 q = vv.plane(i, j);
  coarse[3 * k] = q.c0;
  coarse[3 * k + 1] = q.cx;
  coarse[3 * k + 2] = q.cy;
}

#ifndef FM_TOPDOWN_QUAD
#define FM_TOPDOWN_QUAD 1
#endif
#ifndef FM_TOPDOWN_QUAD_LEVELS
#define FM_TOPDOWN_QUAD_LEVELS 1  // the finest this many levels (A/B at config 4: 1: 0.970, 2: 0.983, all: 0.998, none: 1.010 ms)
#endif
#ifndef FM_GRADE_QUAD
#define FM_GRADE_QUAD 1
#endif
// one thread per sibling quad (levels >= 1): grade_count_quad
// dmx (static MRA, deferred significance): the quad's own flags are
// max|d| / den >= eps (k_sig_from_dmx's operations) instead of fl's
__global__ void k_grade_count_quad(uint8_t* __restrict__ fl, const uint8_t* __restrict__ fl1,
                                   int32_t* __restrict__ cnt, const int32_t* __restrict__ cnt1, int l, int L,
                                   int M, int N, uint64_t quads, int graded,
                                   const uint8_t* __restrict__ ring = nullptr, const double* __restrict__ dmx = nullptr,
                                   double den = 1.0, double eps = 0.0) {
  const uint64_t m = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (m >= quads) return;
  if (dmx) {
    const double y = recip_ieee(den);
    const bool den_ok = div_fast_ok(den);
    const double2 a = reinterpret_cast<const double2*>(dmx)[2 * m], b = reinterpret_cast<const double2*>(dmx)[2 * m + 1];
    const uint32_t own = uint32_t(sig_of(a.x, den, y, den_ok, eps)) | (uint32_t(sig_of(a.y, den, y, den_ok, eps)) << 8) |
                         (uint32_t(sig_of(b.x, den, y, den_ok, eps)) << 16) |
                         (uint32_t(sig_of(b.y, den, y, den_ok, eps)) << 24);
    grade_count_quad(fl, fl1, cnt, cnt1, l, L, M, N, m, graded, nullptr, &own);
    return;
  }
  grade_count_quad(fl, fl1, cnt, cnt1, l, L, M, N, m, graded, ring);
}
__global__ void k_grade_count(uint8_t* __restrict__ fl, const uint8_t* __restrict__ fl1,
                              int32_t* __restrict__ cnt, const int32_t* __restrict__ cnt1, int l,
                              int L, int M, int N, uint64_t nodes, int graded,
                              const uint8_t* __restrict__ ring = nullptr) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n < nodes) grade_count_node(fl, fl1, cnt, cnt1, l, L, M, N, n, graded, ring);
}

// The small levels (<= kSmallLevelNodes nodes, all at the coarse end) of the
// per-level passes in ONE single-CTA launch, walking the levels in the pass's
// order with a barrier between levels: at the coarse end a launch per level
// costs more than the level's work.
constexpr uint64_t kSmallLevelNodes = 256;
struct RingPtrs {
  const uint8_t* ring[kMaxL];  // per level, or all null
};
struct LevelPtrs {
  uint8_t* fl[kMaxL];
  int32_t* cnt[kMaxL];
  int32_t* off[kMaxL];
  double* zs[kMaxL];  // zs[0] = the level-0 scaling
  const double* det[kMaxL];
};
__global__ void __launch_bounds__(256) k_grade_count_small(LevelPtrs p, int lhi, int L, int M, int N, int graded,
                                                           RingPtrs r) {
  for (int l = lhi; l >= 0; --l) {
    const uint64_t nodes = uint64_t(M) * N << (2 * l);
    for (uint64_t n = threadIdx.x; n < nodes; n += blockDim.x)
      grade_count_node(p.fl[l], l + 1 < L ? p.fl[l + 1] : nullptr, p.cnt[l], l + 1 < L ? p.cnt[l + 1] : nullptr, l,
                       L, M, N, n, graded, r.ring[l]);
    __syncthreads();
  }
}

// Exclusive scan of the level-0 counts (M*N nodes) in one CTA.
__global__ void k_level0_offsets(const int32_t* __restrict__ cnt, int32_t* __restrict__ off,
                                 int64_t n, long long* total) {
  __shared__ long long part[1024];
  __shared__ long long base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < n; b0 += blockDim.x) {
    const int64_t k = b0 + threadIdx.x;
    const long long v = k < n ? cnt[k] : 0;
    part[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < int(blockDim.x); o <<= 1) {
      const long long add = threadIdx.x >= unsigned(o) ? part[threadIdx.x - o] : 0;
      __syncthreads();
      part[threadIdx.x] += add;
      __syncthreads();
    }
    if (k < n) off[k] = int32_t(base + part[threadIdx.x] - v);
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) base += part[threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = base;
}

__global__ void k_topdown(const uint8_t* __restrict__ flp, const uint8_t* __restrict__ fl,
                          const uint8_t* __restrict__ fl1, const int32_t* __restrict__ cnt1,
                          const int32_t* __restrict__ off, int32_t* __restrict__ off1,
                          const double* __restrict__ zin, double* __restrict__ zout,
                          const double* __restrict__ det, int l, int L, int M, int kind,
                          uint64_t nodes, LeafOut out) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n < nodes) topdown_node(flp, fl, fl1, cnt1, off, off1, zin, zout, det, l, L, M, kind, n, out);
}
// The same per sibling quad (levels >= 1): at the fine levels most quads
// have an unflagged parent or no flagged node, and one thread per quad
// finds that with one byte and one word instead of four threads
__global__ void k_topdown_quad(const uint8_t* __restrict__ flp, const uint8_t* __restrict__ fl,
                               const uint8_t* __restrict__ fl1, const int32_t* __restrict__ cnt1,
                               const int32_t* __restrict__ off, int32_t* __restrict__ off1,
                               const double* __restrict__ zin, double* __restrict__ zout,
                               const double* __restrict__ det, int l, int L, int M, int kind, uint64_t quads,
                               LeafOut out) {
  const uint64_t m = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (m >= quads || !flp[m]) return;
  const uint32_t f4 = *reinterpret_cast<const uint32_t*>(fl + 4 * m);
  if (!f4) return;
#pragma unroll 1
  for (int c = 0; c < 4; ++c)
    if ((f4 >> (8 * c)) & 0xffu) topdown_node(flp, fl, fl1, cnt1, off, off1, zin, zout, det, l, L, M, kind, 4 * m + c, out);
}
__global__ void __launch_bounds__(256) k_topdown_small(LevelPtrs p, int lhi, int L, int M, int N, int kind,
                                                       LeafOut out) {
  for (int l = 0; l <= lhi; ++l) {
    const uint64_t nodes = uint64_t(M) * N << (2 * l);
    const bool last = l + 1 == L;
    for (uint64_t n = threadIdx.x; n < nodes; n += blockDim.x)
      topdown_node(l ? p.fl[l - 1] : nullptr, p.fl[l], last ? nullptr : p.fl[l + 1],
                   last ? nullptr : p.cnt[l + 1], p.off[l], last ? nullptr : p.off[l + 1], p.zs[l],
                   last ? nullptr : p.zs[l + 1], p.det[l], l, L, M, kind, n, out);
    __syncthreads();
  }
}

// Level-L planes of a vertex raster in node order (field.cpp:106-117).
__global__ void k_project_level(VertexView vv, const Scalars* __restrict__ s, double* out, int L,
                                int M, uint64_t total) {
  vv.wall = s->wall;
  const uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (k >= total) return;
  int i, j;
  node_ij(L, k, M, i, j);
  const P3 q = vv.plane(i, j);
  out[3 * k] = q.c0;
  out[3 * k + 1] = q.cx;
  out[3 * k + 2] = q.cy;
}

// One level of parent scaling (encode rows 0-2 only), children 4n..4n+3.
__global__ void k_parent_level(const double* __restrict__ in, double* __restrict__ out, int kind,
                               uint64_t nodes) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= nodes) return;
  P3 kids[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double* c = in + 3 * (4 * n + k);
    kids[k] = P3{c[0], c[1], c[2]};
  }
  const P3 p = encode_parent(kids, kind);
  out[3 * n] = p.c0;
  out[3 * n + 1] = p.cx;
  out[3 * n + 2] = p.cy;
}

inline unsigned blocks_for(uint64_t n, int t) { return unsigned((n + t - 1) / t); }

// One level of the grading sweep as its own launch.
void launch_grade_level(Grid& g, int l, bool graded, const uint8_t* ring) {
  const int L = g.L;
  const uint64_t nodes = g.nodes(l);
  uint8_t* fl = g.flag[l].p;
  const uint8_t* fl1 = l + 1 < L ? g.flag[l + 1].p : nullptr;
  int32_t* cnt = g.cnt[l].p;
  const int32_t* cnt1 = l + 1 < L ? g.cnt[l + 1].p : nullptr;
  // the level's significance still to form from max |d| (mra_encode's defer_sig)
  const double* dmx = (!ring && l > g.sig_done && size_t(l) < g.dmx.size()) ? g.dmx[l].p : nullptr;
  if (dmx || (FM_GRADE_QUAD && l >= 1)) {
    k_grade_count_quad<<<blocks_for(nodes / 4, 256), 256, 0, stream()>>>(fl, fl1, cnt, cnt1, l, L, g.M, g.N,
                                                                         nodes / 4, graded ? 1 : 0, ring, dmx,
                                                                         g.sig_den, g.eps);
  } else {
    k_grade_count<<<blocks_for(nodes, 256), 256, 0, stream()>>>(fl, fl1, cnt, cnt1, l, L, g.M, g.N, nodes,
                                                               graded ? 1 : 0, ring);
  }
  FM_LAUNCHED();
}


}  // namespace

namespace {
// The middle levels of the top-down decode as subtrees (adaptive.cu's
// k_levels_tree): CTA b owns level-r node b and decodes its subtree down to
// level rt, a block barrier between levels instead of a launch per level.
#ifndef FM_TREE_THREADS
#define FM_TREE_THREADS 64
#endif
constexpr int kTreeThreads = FM_TREE_THREADS;
__global__ void __launch_bounds__(kTreeThreads) k_topdown_tree(LevelPtrs p, int r, int rt, int L, int M, int kind,
                                                               LeafOut out) {
  const uint64_t b = blockIdx.x;
  for (int l = r; l <= rt; ++l) {
    const uint64_t per = uint64_t(1) << (2 * (l - r));
    const bool last = l + 1 == L;
    for (uint64_t j = threadIdx.x; j < per; j += blockDim.x)
      topdown_node(l ? p.fl[l - 1] : nullptr, p.fl[l], last ? nullptr : p.fl[l + 1],
                   last ? nullptr : p.cnt[l + 1], p.off[l], last ? nullptr : p.off[l + 1], p.zs[l],
                   last ? nullptr : p.zs[l + 1], p.det[l], l, L, M, kind, b * per + j, out);
    __syncthreads();
  }
}
}  // namespace

// assemble_grid's top-down decode (levels 0..L-1, offsets of level 0 done):
// the small coarse levels in one single-CTA launch, the middle levels as
// subtrees in one launch, then a launch per fine level.
// quad: the fine levels one thread per sibling quad (the static MRA, where
// most fine quads are inactive; the adaptive re-grid's fine levels are
// mostly active and run one thread per node)
void launch_topdown(Grid& g, const LeafOut& out, bool small_done = false, bool quad = false) {
  cudaStream_t st = stream();
  const int L = g.L;
  std::vector<DBuf<double>>& zs = g.zs;
  LevelPtrs p{};
  for (int l = 0; l < L; ++l) {
    p.fl[l] = g.flag[l].p;
    p.cnt[l] = g.cnt[l].p;
    p.off[l] = g.off[l].p;
    p.zs[l] = l ? zs[l].p : g.coarse.p;
    p.det[l] = g.det[l].p;
  }
  int ls = -1;
  for (int l = 0; l < L; ++l)
    if (g.nodes(l) <= kSmallLevelNodes) ls = l;
  if (ls >= 0 && !small_done) {
    k_topdown_small<<<1, 256, 0, st>>>(p, ls, L, g.M, g.N, g.dkind(), out);
    FM_LAUNCHED();
  }
  const int r = ls + 1;
  int rt = r - 1;
  for (int l = r; l < L; ++l)
    if ((uint64_t(1) << (2 * (l - r))) <= uint64_t(kTreeThreads)) rt = l;
  if (rt > r && r < L) {
    k_topdown_tree<<<unsigned(g.nodes(r)), kTreeThreads, 0, st>>>(p, r, rt, L, g.M, g.dkind(), out);
    FM_LAUNCHED();
  } else {
    rt = r - 1;
  }
  for (int l = rt + 1; l < L; ++l) {
    const uint64_t nodes = g.nodes(l);
    const bool last = l + 1 == L;
    if (FM_TOPDOWN_QUAD && quad && l >= 1 && l >= L - FM_TOPDOWN_QUAD_LEVELS)
      k_topdown_quad<<<blocks_for(nodes / 4, 256), 256, 0, st>>>(
          g.flag[l - 1].p, g.flag[l].p, last ? nullptr : g.flag[l + 1].p, last ? nullptr : g.cnt[l + 1].p,
          g.off[l].p, last ? nullptr : g.off[l + 1].p, zs[l].p, last ? nullptr : zs[l + 1].p, g.det[l].p, l, L,
          g.M, g.dkind(), nodes / 4, out);
    else
      k_topdown<<<blocks_for(nodes, 256), 256, 0, st>>>(
          l ? g.flag[l - 1].p : nullptr, g.flag[l].p, last ? nullptr : g.flag[l + 1].p,
          last ? nullptr : g.cnt[l + 1].p, g.off[l].p, last ? nullptr : g.off[l + 1].p,
          l ? zs[l].p : g.coarse.p, last ? nullptr : zs[l + 1].p, g.det[l].p, l, L, g.M, g.dkind(),
          nodes, out);
    FM_LAUNCHED();
  }
}

int64_t build_leaves(Grid& g) {
  FM_RANGE("build_leaves");
  cudaStream_t st = stream();
  const int L = g.L;
  g.cnt.resize(L);
  g.off.resize(L);
  for (int l = 0; l < L; ++l) {
    g.cnt[l].alloc(g.nodes(l));
    g.off[l].alloc(g.nodes(l));
  }
  // counts (flags already final at level L-1 .. 0 after k_grade_count)
  DBuf<long long> total(1);
  if (L == 0) {
    // every level-0 node is a leaf
    g.nleaves = int64_t(g.M) * g.N;
  } else {
    k_level0_offsets<<<1, 1024, 0, st>>>(g.cnt[0].p, g.off[0].p, int64_t(g.nodes(0)), total.p);
    FM_LAUNCHED();
    long long tot = 0;
    total.download(&tot, 1);
    FM_CUDA(cudaStreamSynchronize(st));
    g.nleaves = tot;
  }
  if (g.nleaves > INT32_MAX) throw Error(FM_ERR_STRUCTURE, "leaf count exceeds int32");
  g.lf_l.ensure(g.nleaves);
  g.lf_i.ensure(g.nleaves);
  g.lf_j.ensure(g.nleaves);
  g.lf_z.ensure(3 * g.nleaves);
  LeafOut out{g.lf_l.p, g.lf_i.p, g.lf_j.p, g.lf_z.p};
  if (L == 0) {
    // copy coarse planes out as leaves (node order == Morton order at level 0)
    std::vector<double> c = g.coarse.to_host();
    std::vector<int8_t> hl(g.nleaves, 0);
    std::vector<int32_t> hi(g.nleaves), hj(g.nleaves);
    for (int64_t k = 0; k < g.nleaves; ++k) {
      hi[k] = int32_t(k % g.M);
      hj[k] = int32_t(k / g.M);
    }
    g.lf_l.upload(hl.data(), hl.size());
    g.lf_i.upload(hi.data(), hi.size());
    g.lf_j.upload(hj.data(), hj.size());
    g.lf_z.upload(c.data(), c.size());
    return g.nleaves;
  }
  // decoded-plane scratch per level (levels 1..L-1)
  std::vector<DBuf<double>>& zs = g.zs;  // kept across builds (adaptive re-grids)
  zs.resize(L);
  for (int l = 1; l < L; ++l) zs[l].alloc(3 * g.nodes(l));
  launch_topdown(g, out, false, true);
  return g.nleaves;
}

// build_leaves without a host round trip (the adaptive re-grid's graph):
// level-0 offsets, then the top-down decode into leaf arrays that hold every
// possible leaf (capacity M N 4^L); the leaf count lands in *total.  cnt /
// off / zs must already be allocated (a previous build_leaves).
void build_leaves_device(Grid& g, long long* total) {
  cudaStream_t st = stream();
  const int L = g.L;
  k_level0_offsets<<<1, 1024, 0, st>>>(g.cnt[0].p, g.off[0].p, int64_t(g.nodes(0)), total);
  FM_LAUNCHED();
  launch_topdown(g, LeafOut{g.lf_l.p, g.lf_i.p, g.lf_j.p, g.lf_z.p});
}

namespace {
// The adapt's small coarse levels as one single-CTA launch: grading + counts
// (levels ls..0), the level-0 offsets and new leaf count, then the top-down
// decode of levels 0..ls -- three launches of one CTA each before, every
// level a chain of dependent round trips either way.
__global__ void __launch_bounds__(256) k_small_chain(LevelPtrs p, RingPtrs r, int ls, int L, int M, int N,
                                                     int graded, int kind, LeafOut out, long long* total) {
  for (int l = ls; l >= 0; --l) {
    const uint64_t nodes = uint64_t(M) * N << (2 * l);
    for (uint64_t n = threadIdx.x; n < nodes; n += blockDim.x)
      grade_count_node(p.fl[l], l + 1 < L ? p.fl[l + 1] : nullptr, p.cnt[l], l + 1 < L ? p.cnt[l + 1] : nullptr, l,
                       L, M, N, n, graded, r.ring[l]);
    __syncthreads();
  }
  cta_exclusive_scan(p.cnt[0], p.off[0], int64_t(M) * N, total);
  __syncthreads();
  for (int l = 0; l <= ls; ++l) {
    const uint64_t nodes = uint64_t(M) * N << (2 * l);
    const bool last = l + 1 == L;
    for (uint64_t n = threadIdx.x; n < nodes; n += blockDim.x)
      topdown_node(l ? p.fl[l - 1] : nullptr, p.fl[l], last ? nullptr : p.fl[l + 1],
                   last ? nullptr : p.cnt[l + 1], p.off[l], last ? nullptr : p.off[l + 1], p.zs[l],
                   last ? nullptr : p.zs[l + 1], p.det[l], l, L, M, kind, n, out);
    __syncthreads();
  }
}
}  // namespace

// grade_count_levels (graded, with the ring) + build_leaves_device, the small
// levels of both in one launch (k_small_chain).
void grade_and_build_leaves_device(Grid& g, const std::vector<const uint8_t*>* ring, long long* total) {
  cudaStream_t st = stream();
  const int L = g.L;
  int ls = -1;
  for (int l = 0; l < L; ++l)
    if (g.nodes(l) <= kSmallLevelNodes) ls = l;
  if (ls < 0) {
    grade_count_levels(g, true, ring);
    build_leaves_device(g, total);
    return;
  }
  for (int l = L - 1; l > ls; --l) launch_grade_level(g, l, true, ring ? (*ring)[l] : nullptr);
  LevelPtrs p{};
  RingPtrs r{};
  for (int l = 0; l < L; ++l) {
    p.fl[l] = g.flag[l].p;
    p.cnt[l] = g.cnt[l].p;
    p.off[l] = g.off[l].p;
    p.zs[l] = l ? g.zs[l].p : g.coarse.p;
    p.det[l] = g.det[l].p;
    r.ring[l] = ring ? (*ring)[l] : nullptr;
  }
  const LeafOut out{g.lf_l.p, g.lf_i.p, g.lf_j.p, g.lf_z.p};
  k_small_chain<<<1, 256, 0, st>>>(p, r, ls, L, g.M, g.N, 1, g.dkind(), out, total);
  FM_LAUNCHED();
  launch_topdown(g, out, true);
}

// Projection + multi-level encode (detail_tree.cpp:10-54 with the fused
// field.cpp:64-117): fills g.det, g.flag (= significance, detail_tree.cpp:66-72,
// before closure), g.coarse and g.field_norm.  All buffers are allocated
// before the first kernel so `ms` (CUDA events) times kernels only.
void mra_encode(const fm_raster* dem, int L, double eps, int kind, Grid& g, double* ms, bool defer_sig) {
  FM_RANGE("mra_encode");
  if (!dem || !dem->values) throw Error(FM_ERR_CONFIG, "null DEM raster");
  if (dem->ncols < 2 || dem->nrows < 2)
    throw Error(FM_ERR_CONFIG, "DEM must have at least 2x2 samples to define elements");
  if (L < 0) throw Error(FM_ERR_CONFIG, "max_level must be >= 0");
  if (L > kMaxL - 1) throw Error(FM_ERR_CONFIG, "max_level above 15 is not supported");
  if (eps < 0.0) throw Error(FM_ERR_DOMAIN, "flag_significant: eps must be >= 0");
  if (kind != FM_MW && kind != FM_HW) throw Error(FM_ERR_CONFIG, "unknown wavelet kind");
  upload_banks();
  cudaStream_t st = stream();
  const int n = dem->ncols - 1, m = dem->nrows - 1;
  const int step = 1 << L;
  g.L = L;
  g.M = (n + step - 1) / step;
  g.N = (m + step - 1) / step;
  g.R = dem->cellsize;
  g.x0 = dem->xll;
  g.y0 = dem->yll;
  g.eps = eps;
  g.kind = kind;
  if (uint64_t(g.M) * g.N * (uint64_t(1) << (2 * L)) > (uint64_t(1) << 40))
    throw Error(FM_ERR_CONFIG, "domain too large");

  // DEM to the device (or use it in place)
  const size_t nv = size_t(dem->ncols) * dem->nrows;
  DBuf<double> vbuf;
  const double* vdev = dem->values;
  if (!dem->on_device) {
    vbuf.upload(dem->values, nv);
    vdev = vbuf.p;
  }
  DBuf<Scalars> scal(1);
  scal.zero();
  g.det.resize(L);
  g.flag.resize(L);
  for (int l = 0; l < L; ++l) {
    g.det[l].alloc(9 * g.nodes(l));
    g.flag[l].alloc(g.nodes(l));
  }
  g.coarse.alloc(3 * g.nodes(0));
  // tile-root scaling buffers of the multi-pass encode
  std::vector<int> passes;
  for (int lev_in = L; lev_in > 0;) {
    const int T = std::min(FM_ENC_T, lev_in);
    passes.push_back(T);
    lev_in -= T;
  }
  std::vector<DBuf<double>> roots(passes.size());
  {
    int lev_in = L;
    for (size_t k = 0; k < passes.size(); ++k) {
      lev_in -= passes[k];
      if (lev_in > 0) roots[k].alloc(3 * g.nodes(lev_in));
    }
  }
  EventPair ev;
  cudaEvent_t e0 = ev.a, e1 = ev.b;
  VertexView vv{vdev, dem->ncols, dem->nrows, n, m, dem->nodata, 0.0};
  // the encode passes of up to 5 levels (4^5 = 1024 inputs per CTA)
  auto encode_passes = [&](bool spec, std::vector<DBuf<double>>* dmx) {
    int lev_in = L;
    for (size_t k = 0; k < passes.size(); ++k) {
      const int T = passes[k];
      const int lev_out = lev_in - T;
      EncParams p{};
      p.vv = vv;
      p.sc_in = k ? roots[k - 1].p : nullptr;
      p.sc_out = lev_out == 0 ? g.coarse.p : roots[k].p;
      for (int l = 0; l < L; ++l) {
        p.det[l] = g.det[l].p;
        p.flag[l] = g.flag[l].p;
        p.dmx[l] = dmx ? (*dmx)[l].p : nullptr;
      }
      p.scal = scal.p;
      p.eps = eps;
      p.lev_in = lev_in;
      p.T = T;
      p.M = g.M;
      p.kind = kind;
      const uint64_t tiles = g.nodes(lev_out);
      const int threads = 1 << (2 * (T - 1));
      const size_t smem = (sizeof(P3) + 9 * sizeof(double)) * threads;
      if (spec)
        (k == 0 ? k_encode_tiles<true, true> : k_encode_tiles<false, true>)<<<unsigned(tiles), threads, smem, st>>>(p);
      else
        (k == 0 ? k_encode_tiles<true, false> : k_encode_tiles<false, false>)<<<unsigned(tiles), threads, smem, st>>>(p);
      FM_LAUNCHED();
      lev_in = lev_out;
    }
  };
  // the exact two-pass path: DEM statistics (nodata wall, non-finite check,
  // field_norm), then the encode with the flags
  auto two_pass = [&]() {
    scal.zero();
    k_dem_stats<<<148 * 8, 256, 0, st>>>(vv, scal.p);
    FM_LAUNCHED();
    k_wall<<<1, 1, 0, st>>>(scal.p);
    FM_LAUNCHED();
    k_field_norm_fix<<<148 * 8, 256, 0, st>>>(vv, scal.p);
    FM_LAUNCHED();
    k_norm_final<<<1, 1, 0, st>>>(scal.p);
    FM_LAUNCHED();
    if (L == 0) {
      k_copy_fine<<<blocks_for(g.nodes(0), 256), 256, 0, st>>>(vv, scal.p, g.coarse.p, g.M, g.nodes(0));
      FM_LAUNCHED();
    } else {
      encode_passes(false, nullptr);
    }
  };
  Scalars hs{};
  double t_ms = 0.0;
  bool done = false;
  if (L > 0) {
    // one DEM read: the speculative encode (max |d| per node, the norm from
    // the projected planes), then the flags from max |d| and the norm
    std::vector<DBuf<double>> dmx(L);
    for (int l = 0; l < L; ++l) dmx[l].alloc(g.nodes(l));
    FM_CUDA(cudaEventRecord(e0, st));
    encode_passes(true, &dmx);
    DmxLevels t{};
    for (int l = 0; l < L; ++l) {
      t.dmx[l] = dmx[l].p;
      t.flag[l] = g.flag[l].p;
    }
    // deferred: only the small levels here (the grading's single-CTA pass
    // reads flags); the others' significance is formed in the grading
    int nsig = L;
    if (defer_sig) {
      nsig = 0;
      for (int l = 0; l < L; ++l)
        if (g.nodes(l) <= kSmallLevelNodes) nsig = l + 1;
      nsig = std::max(nsig, 1);  // level 0 always here (the quads start at level 1)
    }
    if (nsig > 0) {
      const unsigned bx = unsigned(std::min<uint64_t>(blocks_for(g.nodes(nsig - 1), 256), 148 * 8));
      k_sig_from_dmx<<<dim3(bx, nsig), 256, 0, st>>>(t, g.M, g.N, scal.p, eps);
      FM_LAUNCHED();
    }
    FM_CUDA(cudaEventRecord(e1, st));
    scal.download(&hs, 1);
    FM_CUDA(cudaStreamSynchronize(st));
    t_ms = elapsed_ms(e0, e1);
    if (!hs.redo) {
      std::memcpy(&hs.norm, &hs.norm_bits, 8);
      done = true;
      g.big = false;  // every vertex finite and |z| <= 1e300 (checked by the encode)
      g.sig_done = L - 1;
      if (nsig < L) {  // the grading forms the rest
        g.sig_done = nsig - 1;
        g.sig_den = hs.norm > 1.0 ? hs.norm : 1.0;  // smax(1.0, norm)
        g.dmx = std::move(dmx);
      }
    }
  }
  if (!done) {  // nodata, non-finite or huge vertices (or L = 0): the exact two-pass path
    FM_CUDA(cudaEventRecord(e0, st));
    two_pass();
    FM_CUDA(cudaEventRecord(e1, st));
    scal.download(&hs, 1);
    FM_CUDA(cudaStreamSynchronize(st));
    t_ms += elapsed_ms(e0, e1);
  }
  if (hs.err) throw Error(FM_ERR_DOMAIN, "project_vertices: non-finite vertex value");
  if (!done) g.big = (hs.flags & kBig) != 0;
  g.field_norm = hs.norm;
  if (ms) *ms = t_ms;
}

// Final flags (closure + optional 2:1 grading) and subtree leaf counts, one
// gather pass per level fine -> coarse (k_grade_count).
void grade_count_levels(Grid& g, bool graded, const std::vector<const uint8_t*>* ring) {
  cudaStream_t st = stream();
  const int L = g.L;
  g.cnt.resize(L);
  for (int l = 0; l < L; ++l) g.cnt[l].alloc(g.nodes(l));
  int ls = -1;  // the finest small level
  for (int l = 0; l < L; ++l)
    if (g.nodes(l) <= kSmallLevelNodes) ls = l;
  for (int l = L - 1; l > ls; --l) launch_grade_level(g, l, graded, ring ? (*ring)[l] : nullptr);
  if (ls >= 0) {
    LevelPtrs p{};
    RingPtrs r{};
    for (int l = 0; l < L; ++l) {
      p.fl[l] = g.flag[l].p;
      p.cnt[l] = g.cnt[l].p;
      r.ring[l] = ring ? (*ring)[l] : nullptr;
    }
    k_grade_count_small<<<1, 256, 0, st>>>(p, ls, L, g.M, g.N, graded ? 1 : 0, r);
    FM_LAUNCHED();
  }
}

// ---- a grid from a leaf list (read_nug + make_quadgrid, quadgrid.cpp:85-110, 310-327)
namespace {
__global__ void k_mark_ancestors(int64_t n, const int8_t* __restrict__ lvl, const int32_t* __restrict__ li,
                                 const int32_t* __restrict__ lj, uint8_t* const* __restrict__ flag, int M) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const int l = lvl[k];
  for (int a = 0; a < l; ++a) flag[a][node_index(a, li[k] >> (l - a), lj[k] >> (l - a), M)] = 1;
}
}  // namespace

Grid* grid_from_leaves(int L, int M, int N, double R, double x0, double y0, int64_t n, const int32_t* lv,
                       const int32_t* li, const int32_t* lj, const double* topo3) {
  if (L < 0 || L > kMaxL - 1) throw Error(FM_ERR_CONFIG, "grid import: level out of range");
  if (M < 1 || N < 1 || n < 1) throw Error(FM_ERR_CONFIG, "grid import: empty grid");
  // make_quadgrid's checks (quadgrid.cpp:100-108)
  int64_t weight = 0;
  for (int64_t k = 0; k < n; ++k) {
    const int l = lv[k];
    if (l < 0 || l > L || li[k] < 0 || lj[k] < 0 || li[k] >= (M << l) || lj[k] >= (N << l))
      throw Error(FM_ERR_STRUCTURE, "make_quadgrid: leaf outside domain");
    weight += int64_t(1) << (2 * (L - l));
  }
  if (weight != int64_t(M) * N * (int64_t(1) << (2 * L)))
    throw Error(FM_ERR_STRUCTURE, "make_quadgrid: leaves do not tile the domain");
  cudaStream_t st = stream();
  auto g = std::make_unique<Grid>();
  g->L = L;
  g->M = M;
  g->N = N;
  g->R = R;
  g->x0 = x0;
  g->y0 = y0;
  g->kind = FM_MW;
  g->graded = false;
  // internal nodes = strict ancestors of the leaves
  std::vector<int8_t> l8(lv, lv + n);
  DBuf<int8_t> dl;
  DBuf<int32_t> di, dj;
  dl.upload(l8.data(), n);
  di.upload(li, n);
  dj.upload(lj, n);
  g->flag.resize(L);
  std::vector<uint8_t*> fptr(std::max(L, 1), nullptr);
  for (int l = 0; l < L; ++l) {
    g->flag[l].alloc(g->nodes(l));
    g->flag[l].zero();
    fptr[l] = g->flag[l].p;
  }
  if (L > 0) {
    DBuf<uint8_t*> dfp;
    dfp.upload(fptr.data(), fptr.size());
    k_mark_ancestors<<<blocks_for(n, 256), 256, 0, st>>>(n, dl.p, di.p, dj.p, dfp.p, M);
    FM_LAUNCHED();
    FM_CUDA(cudaStreamSynchronize(st));
  }
  // counts, offsets and the Morton-ordered leaf list from the flags; the
  // decode runs on zero details (the imported topography replaces it below)
  g->det.resize(L);
  for (int l = 0; l < L; ++l) {
    g->det[l].alloc(9 * g->nodes(l));
    g->det[l].zero();
  }
  g->coarse.alloc(3 * size_t(M) * N);
  g->coarse.zero();
  grade_count_levels(*g, false);
  build_leaves(*g);
  g->det.clear();
  if (g->nleaves != n) throw Error(FM_ERR_STRUCTURE, "make_quadgrid: overlapping or duplicate leaves");
  // check the derived leaves against the input and place the topography
  const std::vector<int8_t> gl = g->lf_l.to_host();
  const std::vector<int32_t> gi = g->lf_i.to_host(), gj = g->lf_j.to_host();
  std::vector<int64_t> order(n);
  std::vector<uint64_t> key(n);
  for (int64_t k = 0; k < n; ++k) {
    key[k] = node_index(lv[k], li[k], lj[k], M) << (2 * (L - lv[k]));
    order[k] = k;
  }
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return key[a] < key[b]; });
  std::vector<double> z(3 * size_t(n));
  for (int64_t r = 0; r < n; ++r) {
    const int64_t k = order[r];
    if (gl[r] != lv[k] || gi[r] != li[k] || gj[r] != lj[k])
      throw Error(FM_ERR_STRUCTURE, "make_quadgrid: overlapping or duplicate leaves");
    z[3 * r] = topo3[3 * k];
    z[3 * r + 1] = topo3[3 * k + 1];
    z[3 * r + 2] = topo3[3 * k + 2];
  }
  g->lf_z.upload(z.data(), z.size());
  FM_CUDA(cudaStreamSynchronize(st));
  return g.release();
}

Grid* mra_static(const fm_raster* dem, int L, double eps, bool graded, int kind) {
  FM_RANGE("fm_mra_static");
  auto g = std::make_unique<Grid>();
  g->graded = graded;
  double enc_ms = 0.0;
  mra_encode(dem, L, eps, kind, *g, &enc_ms, true);
  // pre-size the count/offset pyramids so the timed region holds kernels only
  g->cnt.resize(L);
  g->off.resize(L);
  for (int l = 0; l < L; ++l) {
    g->cnt[l].alloc(g->nodes(l));
    g->off[l].alloc(g->nodes(l));
  }
  cudaStream_t st = stream();
  EventPair ev;
  cudaEvent_t e0 = ev.a, e1 = ev.b;
  FM_CUDA(cudaEventRecord(e0, st));
  grade_count_levels(*g, graded);
  g->dmx.clear();  // (stream-ordered frees)
  g->sig_done = L - 1;
  build_leaves(*g);
  FM_CUDA(cudaEventRecord(e1, st));
  FM_CUDA(cudaStreamSynchronize(st));
  g->mra_ms = enc_ms + elapsed_ms(e0, e1);
  const double Nf = double(g->nodes(L)), Nint = double(uint64_t(g->M) * g->N) * ((std::pow(4.0, L) - 1) / 3);
  // SURVEY §8(d4), fused-projection form: the encode reads the (n+1)^2
  // vertices (8 B each) instead of 24 B fine planes; 73 B per internal node
  // (details + flag), 36 B per leaf (key + topography)
  (void)Nf;
  const double Nv = double(dem->ncols) * double(dem->nrows);
  g->mra_bytes = 8.0 * Nv + 73.0 * Nint + 36.0 * double(g->nleaves);
  return g.release();
}

std::vector<int64_t> reference_order(const Grid& g, std::vector<int8_t>* lo, std::vector<int32_t>* io,
                                     std::vector<int32_t>* jo) {
  std::vector<int8_t> l = g.lf_l.to_host();
  std::vector<int32_t> i = g.lf_i.to_host(), j = g.lf_j.to_host();
  std::vector<int64_t> perm(g.nleaves);
  std::iota(perm.begin(), perm.end(), 0);
  std::sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) {
    if (l[a] != l[b]) return l[a] < l[b];
    if (j[a] != j[b]) return j[a] < j[b];
    return i[a] < i[b];
  });
  if (lo) *lo = std::move(l);
  if (io) *io = std::move(i);
  if (jo) *jo = std::move(j);
  return perm;
}

namespace {
__global__ void k_rowmajor_to_node(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                   int l, int M, uint64_t nodes, int back) {
  const uint64_t n = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (n >= nodes) return;
  int i, j;
  node_ij(l, n, M, i, j);
  const size_t r = size_t(j) * (M << l) + i;
  if (back)
    out[r] = in[n];
  else
    out[n] = in[r];
}
}  // namespace

void grade_flags_host(int L, int M, int N, bool graded, uint8_t* flags) {
  cudaStream_t st = stream();
  std::vector<DBuf<uint8_t>> f(L);
  std::vector<DBuf<int32_t>> cnt(L);
  size_t at = 0;
  for (int l = 0; l < L; ++l) {
    const uint64_t nodes = uint64_t(M) * N << (2 * l);
    DBuf<uint8_t> rm;
    rm.upload(flags + at, nodes);
    f[l].alloc(nodes);
    cnt[l].alloc(nodes);
    k_rowmajor_to_node<<<blocks_for(nodes, 256), 256, 0, st>>>(rm.p, f[l].p, l, M, nodes, 0);
    FM_LAUNCHED();
    FM_CUDA(cudaStreamSynchronize(st));
    at += nodes;
  }
  for (int l = L - 1; l >= 0; --l) {
    const uint64_t nodes = uint64_t(M) * N << (2 * l);
    k_grade_count<<<blocks_for(nodes, 256), 256, 0, st>>>(
        f[l].p, l + 1 < L ? f[l + 1].p : nullptr, cnt[l].p, l + 1 < L ? cnt[l + 1].p : nullptr, l,
        L, M, N, nodes, graded ? 1 : 0);
    FM_LAUNCHED();
  }
  at = 0;
  for (int l = 0; l < L; ++l) {
    const uint64_t nodes = uint64_t(M) * N << (2 * l);
    DBuf<uint8_t> rm(nodes);
    k_rowmajor_to_node<<<blocks_for(nodes, 256), 256, 0, st>>>(f[l].p, rm.p, l, M, nodes, 1);
    FM_LAUNCHED();
    rm.download(flags + at, nodes);
    FM_CUDA(cudaStreamSynchronize(st));
    at += nodes;
  }
}

void project_planes(const fm_raster* r, int L, int M, int N, DBuf<double>& out) {
  cudaStream_t st = stream();
  const size_t nv = size_t(r->ncols) * r->nrows;
  DBuf<double> vbuf;
  const double* vdev = r->values;
  if (!r->on_device) {
    vbuf.upload(r->values, nv);
    vdev = vbuf.p;
  }
  DBuf<Scalars> scal(1);
  scal.zero();
  k_vertex_max<<<148 * 8, 256, 0, st>>>(vdev, nv, r->nodata, scal.p);
  FM_LAUNCHED();
  k_wall<<<1, 1, 0, st>>>(scal.p);
  FM_LAUNCHED();
  VertexView vv{vdev, r->ncols, r->nrows, r->ncols - 1, r->nrows - 1, r->nodata, 0.0};
  const uint64_t total = uint64_t(M) * N << (2 * L);
  out.alloc(3 * total);
  k_project_level<<<blocks_for(total, 256), 256, 0, st>>>(vv, scal.p, out.p, L, M, total);
  FM_LAUNCHED();
  Scalars hs{};
  scal.download(&hs, 1);
  FM_CUDA(cudaStreamSynchronize(st));
  if (hs.err) throw Error(FM_ERR_DOMAIN, "project_vertices: non-finite vertex value");
}

void scaling_pyramid(DBuf<double>&& level_L, int L, int M, int N, int kind,
                     std::vector<DBuf<double>>& sc) {
  upload_banks();
  sc.clear();
  sc.resize(L + 1);
  sc[L] = std::move(level_L);
  for (int l = L - 1; l >= 0; --l) {
    const uint64_t nodes = uint64_t(M) * N << (2 * l);
    sc[l].alloc(3 * nodes);
    k_parent_level<<<blocks_for(nodes, 256), 256, 0, stream()>>>(sc[l + 1].p, sc[l].p, kind, nodes);
    FM_LAUNCHED();
  }
}

namespace {
__global__ void k_project_rowmajor(VertexView vv, const Scalars* __restrict__ s, double* out) {
  vv.wall = s->wall;
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= (long long)vv.n * vv.m) return;
  const int i = int(k % vv.n), j = int(k / vv.n);
  const P3 q = vv.plane(i, j);
  out[3 * k] = q.c0;
  out[3 * k + 1] = q.cx;
  out[3 * k + 2] = q.cy;
}
}  // namespace

// project_elements (field.cpp:93-104): unpadded planes, row-major j*nx+i.
void project_planes_rowmajor(const fm_raster* r, DBuf<double>& out) {
  cudaStream_t st = stream();
  const size_t nv = size_t(r->ncols) * r->nrows;
  DBuf<double> vbuf;
  const double* vdev = r->values;
  if (!r->on_device) {
    vbuf.upload(r->values, nv);
    vdev = vbuf.p;
  }
  DBuf<Scalars> scal(1);
  scal.zero();
  k_vertex_max<<<148 * 8, 256, 0, st>>>(vdev, nv, r->nodata, scal.p);
  FM_LAUNCHED();
  k_wall<<<1, 1, 0, st>>>(scal.p);
  FM_LAUNCHED();
  VertexView vv{vdev, r->ncols, r->nrows, r->ncols - 1, r->nrows - 1, r->nodata, 0.0};
  const long long n = (long long)(r->ncols - 1) * (r->nrows - 1);
  out.alloc(3 * n);
  k_project_rowmajor<<<unsigned((n + 255) / 256), 256, 0, st>>>(vv, scal.p, out.p);
  FM_LAUNCHED();
  Scalars hs{};
  scal.download(&hs, 1);
  FM_CUDA(cudaStreamSynchronize(st));
  if (hs.err) throw Error(FM_ERR_DOMAIN, "project_vertices: non-finite vertex value");
}

}  // namespace fmh
