// Per-leaf and per-segment static quantities of a leaf set, shared by the
// static set-up kernels (topo.cu) and the adaptive re-grid, which computes
// them inside the passes that install the new leaf set (adaptive.cu, topo.cu
// k_segments with SegExtras) instead of one launch each.
#pragma once

#include "fm_device.cuh"
#include "step_common.cuh"

namespace fmh {
namespace {

using namespace fmd;

// Manning per leaf from a cell-centred raster (solver_nonuniform.cpp:575-584).
__device__ __forceinline__ double manning_at(int L, double R, double x0, double y0, int l, int i, int j,
                                             const double* __restrict__ mr, int nc, int nr, double xll,
                                             double yll, double cs, double uniform) {
  if (!mr) return uniform;
  const double xc = x0 + (i + 0.5) * R * double(1 << (L - l));
  const double yc = y0 + (j + 0.5) * R * double(1 << (L - l));
  const int col = min(max(int((xc - xll) / cs), 0), nc - 1);
  const int row = min(max(nr - 1 - int((yc - yll) / cs), 0), nr - 1);
  return mr[size_t(row) * nc + col];
}

// Inflow target cells of a leaf (solver_nonuniform.cpp:611-628): the area of
// the intersection of its fine-cell square with the rectangle (integer).
__device__ __forceinline__ int32_t inflow_overlap(int L, int l, int i, int j, int i0, int j0, int i1, int j1) {
  const int sh = L - l;
  const long long x0 = (long long)i << sh, x1 = x0 + (1ll << sh);
  const long long y0 = (long long)j << sh, y1 = y0 + (1ll << sh);
  const long long wx = max(0ll, min(x1, (long long)i1 + 1) - max(x0, (long long)i0));
  const long long wy = max(0ll, min(y1, (long long)j1 + 1) - max(y0, (long long)j0));
  return int32_t(wx * wy);
}

// z of a leaf's plane at its four side midpoints N E S W (k_stage's side
// evaluation, limit_rel at (0, 1/2), (1/2, 0), (0, -1/2), (-1/2, 0)).
__device__ __forceinline__ void side_z4(const double* __restrict__ p, double* __restrict__ out4) {
  double2* o = reinterpret_cast<double2*>(out4);
  o[0] = make_double2(eval_rel(p[0], p[1], p[2], 0.0, 0.5), eval_rel(p[0], p[1], p[2], 0.5, 0.0));
  o[1] = make_double2(eval_rel(p[0], p[1], p[2], 0.0, -0.5), eval_rel(p[0], p[1], p[2], -0.5, 0.0));
}

// A segment's static geometry byte (k_seg's P2 path): bit 0 x-normal; bits
// 1-2 / 3-4 the tangential offset code of the W/S and E/N leaf's limit point
// (0: centre of its face, 1: -1/4, 2: +1/4 of its size).
__device__ __forceinline__ uint8_t seg_geo_code(int L, int la, int ia, int ja, int lb, int ib, int jb) {
  const bool xn = (ib << (L - lb)) == ((ia + 1) << (L - la));
  const int ta = la < lb ? ((((xn ? jb : ib) & 1) ? 2 : 1)) : 0;
  const int tb = lb < la ? ((((xn ? ja : ia) & 1) ? 2 : 1)) : 0;
  return uint8_t((xn ? 1 : 0) | (ta << 1) | (tb << 3));
}

// Both leaves' topography at the segment centre (limit_at,
// solver_nonuniform.cpp:52-66, as k_seg's limit_rel evaluates it).
__device__ __forceinline__ double2 seg_z2(int gc, const double* __restrict__ za, const double* __restrict__ zb) {
  const bool xn = gc & 1;
  const int ca = (gc >> 1) & 3, cb = (gc >> 3) & 3;
  const double ta = ca == 0 ? 0.0 : ca == 2 ? 0.25 : -0.25;
  const double tb = cb == 0 ? 0.0 : cb == 2 ? 0.25 : -0.25;
  return make_double2(eval_rel(za[0], za[1], za[2], xn ? 0.5 : ta, xn ? ta : 0.5),
                      eval_rel(zb[0], zb[1], zb[2], xn ? -0.5 : tb, xn ? tb : -0.5));
}

}  // namespace
}  // namespace fmh
