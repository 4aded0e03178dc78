// Uniform-raster DG2 / FV1 / ACC on sm_100a (UniformSim, solver_uniform.cpp):
// config 4's "uniform-raster DG2 at the finest level" comparator.
//
// Layout: cell (i, j) at j*nx + i (the reference's own order), 9 flow
// coefficients + 3 topography coefficients per cell (AoS).
//
// k_uni_march<STAGE>: one warp per strip of columns marching north (below).
// Per cell: its four face revisions (revise_faces :73-137), each face's HLL
// flux solved once (fluxes :139-185), assemble (assemble_dg2 :187-229 /
// assemble_fv1 :231-251), the update, positivity (:253-281) and, on the last
// stage, the inflow sources, the non-finite guard and the next step's CFL
// reduction (the drive-loop epilogue shared with the non-uniform kernels).
#include <algorithm>
#include <cmath>
#include <vector>

#include "fm_device.cuh"
#include "fm_sim.hpp"
#include "step_common.cuh"

using namespace fmd;

namespace fmh {

void launch_head_friction(Sim& s, const double* src, double* dst, bool manual, double mdt);
void launch_decide(Sim& s);
void project_planes_rowmajor(const fm_raster* r, DBuf<double>& out);

namespace {

// A raster band: rows [gy0, gy0 + ny) of the global ny_g rows are owned and
// stored first (row-major); the ghost rows of a sharded band (the rows just
// south / north of it, hs / hn) follow them.  Unsharded: gy0 = 0, ny_g = ny.
struct UniView {
  int nx, ny, scheme, ninflow, libm;
  int gy0, nyg, hs, hn;
  double R, x0, y0, g, hdry, courant;
  int bc[4];
  const double* z;
  const double* nman;
  int rect[4 * kMaxInflows];
};

struct Star {
  double h, qx, qy;
};

// storage index of cell (i, local row jl), jl in [-1, ny]: owned rows first,
// then the south and north ghost rows
__device__ __forceinline__ size_t cidx(const UniView& v, int i, int jl) {
  const int r = jl < 0 ? v.ny : jl >= v.ny ? v.ny + v.hs : jl;
  return size_t(r) * v.nx + i;
}

// One face of revise_faces (solver_uniform.cpp:84-129): the cell's limit on
// side `sd` (side_limit, :16-26) against the opposing face value of the
// neighbour's topography.  Returns the starred state; zd and the raw limit
// feed DirMod.
struct FaceRev {
  Star st;
  double zd;
};
__device__ __forceinline__ FaceRev revise_face(const double u[9], const P3& zc, int sd,
                                               double z_other, bool has_other, double hdry) {
  const P3 h{u[0], u[1], u[2]}, qx{u[3], u[4], u[5]}, qy{u[6], u[7], u[8]};
  const double lh = smax(0.0, face_val(h, sd));
  const double lqx = face_val(qx, sd), lqy = face_val(qy, sd);
  const double lz = face_val(zc, sd);
  const double eta = lh + lz;
  double uu, vv;
  vel2(lh, lqx, lqy, hdry, uu, vv);
  const double zs = smax(lz, has_other ? z_other : lz);
  const double hs = smax(0.0, eta - zs);
  FaceRev r;
  r.st = Star{hs, hs * uu, hs * vv};
  r.zd = zs - smax(0.0, zs - eta);
  return r;
}

__device__ __forceinline__ P3 ld3(const double* a, size_t c) { return P3{a[3 * c], a[3 * c + 1], a[3 * c + 2]}; }
__device__ __forceinline__ void ld9(const double* a, size_t c, double s[9]) {
#pragma unroll
  for (int q = 0; q < 9; ++q) s[q] = a[9 * c + q];
}

// ---- the marching stage kernel ---------------------------------------------
// One warp per strip of 30 columns x FM_UNI_H rows, marching north row by
// row: lane L holds column cx0 - 1 + L (lanes 0 and 31 are the strip's west /
// east halo columns, computed but not stored).  Each row's four face
// revisions (revise_faces, solver_uniform.cpp:84-129) and its x fluxes
// (fluxes :139-185) meet across lanes by shuffles, each x face's HLL solved
// once by the lane west of it; the y fluxes need no exchange at all: the
// lane revises the NEXT row's south face as it finishes the current row
// (that row is loaded one iteration ahead) and carries that face and the
// north flux it makes into the next iteration as its south face and flux.
// No shared memory, no block barriers, and only 1/FM_UNI_H of a row of halo
// work in y.  (The round-1/2 kernel, 32 x 4 shared-memory tiles, revised
// 0.56 halo faces and solved 0.28 redundant fluxes per cell and waited on
// block barriers: 8.5 / 9.4 ms per stage at config 4 against 5.6 / 7.1 here,
// bit-identical.)  The next row's state and (stage 2) U's row are
// prefetched into L1 and loaded where used; HLL is inlined (the out-of-line
// call spilled the live state around it).
#ifndef FM_UNI_H
#define FM_UNI_H 64
#endif

#ifndef FM_UNI_MARCH_MINB
#define FM_UNI_MARCH_MINB 4
#endif
constexpr int kMarchCols = 30;

#ifndef FM_UNI_PREFETCH
#define FM_UNI_PREFETCH 1
#endif
__device__ __forceinline__ void prefetch_l1(const double* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

__device__ __forceinline__ Star shfl_star_down(const Star& a) {
  return Star{__shfl_down_sync(0xffffffffu, a.h, 1), __shfl_down_sync(0xffffffffu, a.qx, 1),
              __shfl_down_sync(0xffffffffu, a.qy, 1)};
}
__device__ __forceinline__ Flx shfl_flx_up(const Flx& a) {
  return Flx{__shfl_up_sync(0xffffffffu, a.m, 1), __shfl_up_sync(0xffffffffu, a.n, 1),
             __shfl_up_sync(0xffffffffu, a.t, 1)};
}

template <int STAGE, bool P2>
__global__ void __launch_bounds__(128, FM_UNI_MARCH_MINB) k_uni_march(UniView v, NuView nv,
                                                                     const DevClock* __restrict__ clk, DevRed* red,
                                                                     const double* __restrict__ in, const double* uold,
                                                                     double* out, int last, int manual, double mdt,
                                                                     int* err) {
  const DevClock* c = clk + 1;
  if (!manual && !c->active) return;
  const double dt = manual ? mdt : c->dt;
  const int lane = threadIdx.x & 31;
  const int wx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int cx0 = wx * kMarchCols;
  if (cx0 >= v.nx) return;  // whole warps only
  const int i = cx0 - 1 + lane;
  const bool colok = i >= 0 && i < v.nx;
  const bool own = colok && lane >= 1 && lane <= kMarchCols;
  const int ic = min(max(i, 0), v.nx - 1);
  const bool hasE = ic + 1 < v.nx, hasW = ic > 0;
  const int y0 = blockIdx.y * FM_UNI_H, y1 = min(y0 + FM_UNI_H, v.ny);
  const double inv = 1.0 / v.R;
  const bool dg2 = v.scheme == FM_DG2;
  // prologue: row y0's state and its south face, and the flux below row y0
  double s[9];
  load9v(in, (long long)cidx(v, ic, y0), s);
  P3 zc = ld3(v.z, cidx(v, ic, y0));
  const bool hasS0 = v.gy0 + y0 > 0;
  Star st_s;  // the current row's revised south face
  double zd_s;
  Flx fs;     // the flux through the current row's south face
  {
    const double zns = hasS0 ? face_val(ld3(v.z, cidx(v, ic, y0 - 1)), 0) : 0.0;
    const FaceRev rs = revise_face(s, zc, 2, zns, hasS0, v.hdry);
    st_s = rs.st;
    zd_s = rs.zd;
    Star l = st_s, r = st_s;
    if (hasS0) {
      double t[9];
      const size_t cs = cidx(v, ic, y0 - 1);
      load9v(in, (long long)cs, t);
      l = revise_face(t, ld3(v.z, cs), 0, face_val(zc, 2), true, v.hdry).st;
    } else if (v.bc[2] == FM_REFLECTIVE) {
      l.qy = -l.qy;
    }
    fs = hll_inl(l.h, l.qy, l.qx, r.h, r.qy, r.qx, v.g, v.hdry, err);
  }
  for (int j = y0; j < y1; ++j) {
    const int gj = v.gy0 + j;
    const bool hasN = gj + 1 < v.nyg;
    // the next row's topography now; its state and (stage 2) U's row of this
    // cell are prefetched into L1 here and loaded where they are used, so
    // they hold no registers through the face work
    const size_t cn = hasN ? cidx(v, ic, j + 1) : size_t(j) * v.nx + ic;
    P3 zn{0.0, 0.0, 0.0};
    if (hasN) zn = ld3(v.z, cn);
#if FM_UNI_PREFETCH
    prefetch_l1(in + 9 * cn);
    prefetch_l1(in + 9 * cn + 8);
    if (STAGE == 2) {
      prefetch_l1(uold + 9 * (size_t(j) * v.nx + ic));
      prefetch_l1(uold + 9 * (size_t(j) * v.nx + ic) + 8);
    }
#endif
    // east / west / north faces of this row
    const double fwv = face_val(zc, 3), fev = face_val(zc, 1);
    const double zwe = __shfl_down_sync(0xffffffffu, fwv, 1);  // the east neighbour's west face value
    const double zew = __shfl_up_sync(0xffffffffu, fev, 1);    // the west neighbour's east face value
    const FaceRev re = revise_face(s, zc, 1, zwe, hasE, v.hdry);
    const FaceRev rw = revise_face(s, zc, 3, zew, hasW, v.hdry);
    const FaceRev rn = revise_face(s, zc, 0, hasN ? face_val(zn, 2) : 0.0, hasN, v.hdry);
    // x fluxes: lane L solves the face between its column and the next;
    // lane 0 (column cx0 - 1 < 0 at the west edge) solves the west boundary
    Flx fe;
    {
      const Star wnext = shfl_star_down(rw.st);
      Star l = re.st, r = wnext;
      if (i == -1) {  // the domain's west boundary face, west of column 0
        l = wnext;
        if (v.bc[3] == FM_REFLECTIVE) l.qx = -l.qx;
      } else if (i == v.nx - 1) {  // the east boundary face
        r = re.st;
        if (v.bc[1] == FM_REFLECTIVE) r.qx = -r.qx;
      }
      fe = hll_inl(l.h, l.qx, l.qy, r.h, r.qx, r.qy, v.g, v.hdry, err);
    }
    const Flx fw = shfl_flx_up(fe);
    // the north face: the next row's south face, revised now and carried
    Flx fn;
    double sn[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    Star st_sn = rn.st;
    double zd_sn = 0.0;
    {
      Star l = rn.st, r = rn.st;
      if (hasN) {
        load9v(in, (long long)cn, sn);
        const FaceRev rs1 = revise_face(sn, zn, 2, face_val(zc, 0), true, v.hdry);
        st_sn = rs1.st;
        zd_sn = rs1.zd;
        r = st_sn;
      } else if (v.bc[0] == FM_REFLECTIVE) {
        r.qy = -r.qy;
      }
      fn = hll_inl(l.h, l.qy, l.qx, r.h, r.qy, r.qx, v.g, v.hdry, err);
    }
    // assemble + update
    double res[9];
    if (own) {
      const double k3 = kHalfInvS3;
      const DirMod X{0.5 * (re.st.h + rw.st.h),   (re.st.h - rw.st.h) * k3,   0.5 * (re.st.qx + rw.st.qx),
                     (re.st.qx - rw.st.qx) * k3, 0.5 * (re.st.qy + rw.st.qy), (re.st.qy - rw.st.qy) * k3,
                     (re.zd - rw.zd) * k3};
      const DirMod Y{0.5 * (rn.st.h + st_s.h),   (rn.st.h - st_s.h) * k3,   0.5 * (rn.st.qx + st_s.qx),
                     (rn.st.qx - st_s.qx) * k3, 0.5 * (rn.st.qy + st_s.qy), (rn.st.qy - st_s.qy) * k3,
                     (rn.zd - zd_s) * k3};
      double Lr[9];
      l_operator<P2>(fn, fe, fs, fw, X, Y, v.R, inv, v.g, v.hdry, dg2, Lr);
      if (STAGE == 1) {
#pragma unroll
        for (int q = 0; q < 9; ++q) res[q] = s[q] + Lr[q] * dt;
      } else {
        double u0[9];
        load9v(uold, (long long)(size_t(j) * v.nx + ic), u0);
#pragma unroll
        for (int q = 0; q < 9; ++q) {
          double a = s[q];
          a += Lr[q] * dt;
          a += u0[q];
          a *= 0.5;
          res[q] = a;
        }
      }
      positivity(res, v.hdry);
      if (last && !manual) {
        for (int f = 0; f < v.ninflow; ++f) {
          if (!c->on[f]) continue;
          if (i >= v.rect[4 * f] && gj >= v.rect[4 * f + 1] && i <= v.rect[4 * f + 2] && gj <= v.rect[4 * f + 3])
            res[0] += ddiv(c->per_cell[f] * 1, v.R * v.R);
        }
      }
      store9v(out, (long long)(size_t(j) * v.nx + i), res);
    } else {
#pragma unroll
      for (int q = 0; q < 9; ++q) res[q] = 0.0;
    }
    if (last && !manual) reduce_leaf(nv, red, *c, res, v.R, leaf_key(0, i, gj), own);
    // advance: the next row becomes the current one
#pragma unroll
    for (int q = 0; q < 9; ++q) s[q] = sn[q];
    zc = zn;
    st_s = st_sn;
    zd_s = zd_sn;
    fs = fn;
  }
}

// ---- ACC (solver_uniform.cpp:330-415) --------------------------------------
// x faces (nx+1)*ny then y faces nx*(ny+1), one thread per face; step head.
__global__ void __launch_bounds__(256) k_uni_acc_faces(UniView v, NuView nv, DevClock* clk, DevRed* red,
                                                      const Hydro* hy, const double* __restrict__ u,
                                                      double* __restrict__ qx, double* __restrict__ qy,
                                                      int manual, double mdt) {
  const long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int go;
  double dt;
  step_head(nv, clk, red, hy, manual, mdt, go, dt);
  const long long nfx = (long long)(v.nx + 1) * v.ny, nfy = (long long)v.nx * (v.ny + 1);
  if (!go || f >= nfx + nfy) return;
  const bool xf = f < nfx;
  const long long g = xf ? f : f - nfx;
  int i, j, side;
  size_t l = 0, r = 0, edge = 0;
  bool boundary;
  if (xf) {
    j = int(g / (v.nx + 1));
    i = int(g % (v.nx + 1));
    boundary = i == 0 || i == v.nx;
    side = i == 0 ? 3 : 1;
    edge = size_t(j) * v.nx + (i == 0 ? 0 : v.nx - 1);
    if (!boundary) {
      l = size_t(j) * v.nx + i - 1;
      r = l + 1;
    }
  } else {
    j = int(g / v.nx);  // local face row: between local rows j - 1 and j
    i = int(g % v.nx);
    const int gf = v.gy0 + j;
    boundary = gf == 0 || gf == v.nyg;
    side = gf == 0 ? 2 : 0;
    edge = size_t(gf == 0 ? 0 : v.ny - 1) * v.nx + i;
    if (!boundary) {
      l = cidx(v, i, j - 1);
      r = cidx(v, i, j);
    }
  }
  double* qp = xf ? qx + g : qy + g;
  double q = *qp;
  if (boundary) {
    if (v.bc[side] == FM_REFLECTIVE) {
      *qp = 0.0;
      return;
    }
    const double hf = u[9 * edge];
    if (hf <= v.hdry) {
      *qp = 0.0;
      return;
    }
    const double n = v.nman[edge];
    *qp = zdiv(q, 1.0 + zdiv(v.g * dt * n * n * fabs(q), pow73_m(hf, v.libm)));
    return;
  }
  const double zl = v.z[3 * l], zr = v.z[3 * r];
  const double el = u[9 * l] + zl, er = u[9 * r] + zr;
  const double hf = smax(el, er) - smax(zl, zr);
  if (hf <= v.hdry) {
    *qp = 0.0;
    return;
  }
  const double nf = 0.5 * (v.nman[l] + v.nman[r]);
  *qp = ddiv(q - ddiv(v.g * hf * dt * (er - el), v.R),
             1.0 + zdiv(v.g * dt * nf * nf * fabs(q), pow73_m(hf, v.libm)));
}

__global__ void __launch_bounds__(256) k_uni_acc_cells(UniView v, NuView nv, const DevClock* __restrict__ clk,
                                                      DevRed* red, double* __restrict__ u,
                                                      const double* __restrict__ qx,
                                                      const double* __restrict__ qy, int manual,
                                                      double mdt) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const DevClock* c = clk + 1;
  if (!manual && !c->active) return;
  const double dt = manual ? mdt : c->dt;
  const long long n = (long long)v.nx * v.ny;
  const bool valid = k < n;
  double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  int i = 0, j = 0;
  if (valid) {
    j = int(k / v.nx);
    i = int(k % v.nx);
    ld9(u, k, s);
    const double qw = qx[size_t(j) * (v.nx + 1) + i], qe = qx[size_t(j) * (v.nx + 1) + i + 1];
    const double qs = qy[size_t(j) * v.nx + i], qn = qy[size_t(j + 1) * v.nx + i];
    s[0] -= zdiv(dt * ((qe - qw) + (qn - qs)), v.R);
    s[3] = 0.5 * (qw + qe);
    s[6] = 0.5 * (qs + qn);
    const int gj = v.gy0 + j;
    if (!manual) {
      for (int f = 0; f < v.ninflow; ++f) {
        if (!c->on[f]) continue;
        if (i >= v.rect[4 * f] && gj >= v.rect[4 * f + 1] && i <= v.rect[4 * f + 2] && gj <= v.rect[4 * f + 3])
          s[0] += ddiv(c->per_cell[f] * 1, v.R * v.R);
      }
    }
    u[9 * k] = s[0];
    u[9 * k + 3] = s[3];
    u[9 * k + 6] = s[6];
  }
  if (!manual) reduce_leaf(nv, red, *c, s, v.R, leaf_key(0, i, v.gy0 + j), valid);
}

__global__ void k_uni_reduce_init(NuView nv, int nx, int gy0, const DevClock* clk, DevRed* red,
                                  const double* __restrict__ u) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool valid = k < nv.n;
  double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  int i = 0, j = 0;
  if (valid) {
    ld9(u, k, s);
    j = gy0 + int(k / nx);
    i = int(k % nx);
  }
  DevClock c = clk[1];
  reduce_leaf(nv, red, c, s, nv.R, leaf_key(0, i, j), valid);
}

// Setup kernels (make_uniform_sim, solver_uniform.cpp:522-601).
__global__ void k_uni_manning(int nx, int ny, const double* __restrict__ mr, int nc, int nr,
                              double uniform, double* __restrict__ out) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= (long long)nx * ny) return;
  const int j = int(k / nx), i = int(k % nx);
  if (!mr) {
    out[k] = uniform;
    return;
  }
  const int row = min(max(nr - 1 - j, 0), nr - 1);
  const int col = min(max(i, 0), nc - 1);
  out[k] = mr[size_t(row) * nc + col];
}

__global__ void k_uni_ic(long long n, const double* __restrict__ z, const double* __restrict__ hplanes,
                         int mode, double val, int pc, double hdry, double* __restrict__ zout,
                         double* __restrict__ u) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double f[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  const double c0 = z[3 * k], cx = z[3 * k + 1], cy = z[3 * k + 2];
  if (hplanes) {
    f[0] = hplanes[3 * k];
    f[1] = hplanes[3 * k + 1];
    f[2] = hplanes[3 * k + 2];
  } else if (mode == 1) {  // flow_from_surface (solver_uniform.cpp:60-71)
    const double span = kS3 * (fabs(cx) + fabs(cy));
    if (c0 + span < val) {
      f[0] = val - c0;
      f[1] = -cx;
      f[2] = -cy;
    } else if (c0 - span >= val) {
    } else {
      f[0] = smax(0.0, val - c0);
    }
  } else if (mode == 2) {
    f[0] = val;
  }
  if (pc) {
    zout[3 * k + 1] = 0.0;
    zout[3 * k + 2] = 0.0;
    f[1] = f[2] = 0.0;
    for (int q = 3; q < 9; ++q) f[q] = 0.0;
  }
  positivity(f, hdry);
  for (int q = 0; q < 9; ++q) u[9 * k + q] = f[q];
}

__global__ void k_uni_ij(int nx, long long n, int32_t* li, int32_t* lj) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  li[k] = int32_t(k % nx);
  lj[k] = int32_t(k / nx);
}

// apply_inflows for the host API path (solver_uniform.cpp:444-455)
__global__ void k_uni_inflow_add(UniView v, const double* __restrict__ per_cell, double* u) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= (long long)v.nx * v.ny) return;
  const int j = v.gy0 + int(k / v.nx), i = int(k % v.nx);
  double h = u[9 * k];
  for (int f = 0; f < v.ninflow; ++f) {
    if (per_cell[f] == 0.0) continue;
    if (i >= v.rect[4 * f] && j >= v.rect[4 * f + 1] && i <= v.rect[4 * f + 2] && j <= v.rect[4 * f + 3])
      h += ddiv(per_cell[f] * 1, v.R * v.R);
  }
  u[9 * k] = h;
}

inline unsigned nblk(long long n, int t) { return unsigned((n + t - 1) / t); }

UniView uview(const Sim& s) {
  UniView v{};
  v.nx = s.nx;
  v.ny = s.ny;
  v.gy0 = s.gy0;
  v.nyg = s.nyg ? s.nyg : s.ny;
  v.hs = s.ghost_s;
  v.hn = s.ghost_n;
  v.scheme = s.scheme;
  v.ninflow = s.ninflow;
  v.libm = s.libm;
  v.R = s.R;
  v.x0 = s.x0;
  v.y0 = s.y0;
  v.g = s.g;
  v.hdry = s.hdry;
  v.courant = s.courant;
  for (int q = 0; q < 4; ++q) v.bc[q] = s.bc[q];
  v.z = s.z.p;
  v.nman = s.nman.p;
  for (int q = 0; q < 4 * s.ninflow; ++q) v.rect[q] = s.rect[q];
  return v;
}

}  // namespace

bool geometry_is_p2(double R, double x0, double y0, int L, int M, int N);

void uniform_init(Sim& s, const fm_sim_desc* d, const fm_raster* dem) {
  cudaStream_t st = stream();
  if (d->solver == FM_MWDG2 || d->solver == FM_HWFV1)
    throw Error(FM_ERR_CONFIG, "uniform solver cannot run adaptive kinds");
  if (dem->ncols < 2 || dem->nrows < 2)
    throw Error(FM_ERR_CONFIG, "DEM must have at least 2x2 samples to define elements");
  s.nx = dem->ncols - 1;
  s.ny = dem->nrows - 1;
  s.R = dem->cellsize;
  s.x0 = dem->xll;
  s.y0 = dem->yll;
  s.L = 0;
  s.M = s.nx;
  s.N = s.ny;
  s.n = int64_t(s.nx) * s.ny;
  // power-of-two cell size: the raster has no offsets, only /R divisions
  {
    int e = 0;
    s.p2 = std::frexp(s.R, &e) == 0.5;
  }
  const long long n = s.n;
  project_planes_rowmajor(dem, s.z);
  s.nman.alloc(n);
  k_uni_manning<<<nblk(n, 256), 256, 0, st>>>(s.nx, s.ny, s.has_mr ? s.mr.p : nullptr, s.mr_ncols,
                                               s.mr_nrows, s.manning, s.nman.p);
  FM_LAUNCHED();
  s.u.alloc(9 * n);
  s.us.alloc(9 * n);
  DBuf<double> hp;
  int mode = 0;
  double val = 0.0;
  if (d->initial_depth_raster) {
    const fm_raster* hr = d->initial_depth_raster;
    if (hr->ncols != dem->ncols || hr->nrows != dem->nrows)
      throw Error(FM_ERR_CONFIG, "initial_depth_raster geometry must match the DEM");
    project_planes_rowmajor(hr, hp);
  } else if (d->has_initial_surface) {
    mode = 1;
    val = d->initial_surface;
  } else if (d->initial_depth > 0.0) {
    mode = 2;
    val = d->initial_depth;
  }
  k_uni_ic<<<nblk(n, 256), 256, 0, st>>>(n, s.z.p, hp.n ? hp.p : nullptr, mode, val,
                                          s.scheme != FM_DG2, s.hdry, s.z.p, s.u.p);
  FM_LAUNCHED();
  // inflows: the rectangle itself is the target set (one cell each)
  for (int f = 0; f < s.ninflow; ++f) {
    const int* r = &s.rect[4 * f];
    if (r[0] < 0 || r[1] < 0 || r[2] >= s.nx || r[3] >= s.ny)
      throw Error(FM_ERR_CONFIG, "inflow region outside the domain");
    if (!dem->on_device) {  // element_nodata_mask (sim_common.cpp:118-131)
      bool any = false;
      for (int j = r[1]; j <= r[3] && !any; ++j)
        for (int i = r[0]; i <= r[2] && !any; ++i) {
          const int rs = dem->nrows - 1 - j;
          auto nd = [&](int row, int col) { return dem->values[size_t(row) * dem->ncols + col] == dem->nodata; };
          if (!(nd(rs, i) || nd(rs, i + 1) || nd(rs - 1, i) || nd(rs - 1, i + 1))) any = true;
        }
      if (!any) throw Error(FM_ERR_CONFIG, "inflow region lies entirely on nodata cells");
    }
  }
  s.li.alloc(n);
  s.lj.alloc(n);
  k_uni_ij<<<nblk(n, 256), 256, 0, st>>>(s.nx, n, s.li.p, s.lj.p);
  FM_LAUNCHED();
  if (s.scheme == FM_ACC) {
    s.aqx.alloc(size_t(s.nx + 1) * s.ny);
    s.aqy.alloc(size_t(s.nx) * (s.ny + 1));
    s.aqx.zero();
    s.aqy.zero();
  }
  s.nseg = int64_t(s.nx + 1) * s.ny + int64_t(s.nx) * (s.ny + 1);
}

// The device phases of a uniform-raster step (the op sequence of nu_step_ops;
// exchanges and reductions of a sharded band are the shard layer's).
void un_step_op(Sim& s, int op, bool manual, double mdt, int* err) {
  cudaStream_t st = stream();
  const UniView v = uview(s);
  const NuView nv = s.view();
  const int nwx = (s.nx + kMarchCols - 1) / kMarchCols;
  const dim3 mgrid((nwx + 3) / 4, (s.ny + FM_UNI_H - 1) / FM_UNI_H);
  const bool fv1 = s.scheme == FM_FV1;
  if (s.shard && (op == OP_ACC || op == OP_STAGE1 || op == OP_STAGE2)) shard_finish(s);
  switch (op) {
    case OP_ACC: {
      if (!manual) launch_decide(s);  // the step decision, once (step_common.cuh)
      const long long nf = int64_t(s.nx + 1) * s.ny + int64_t(s.nx) * (s.ny + 1);
      kt_begin(KF_ACC_FACES);
      k_uni_acc_faces<<<nblk(nf, 256), 256, 0, st>>>(v, nv, s.clk.p, s.red.p, s.hydro.p, s.u.p, s.aqx.p,
                                                      s.aqy.p, manual, mdt);
      FM_LAUNCHED();
      kt_end();
      kt_begin(KF_ACC_LEAVES);
      k_uni_acc_cells<<<nblk(s.n, 256), 256, 0, st>>>(v, nv, s.clk.p, s.red.p, s.u.p, s.aqx.p, s.aqy.p,
                                                       manual, mdt);
      FM_LAUNCHED();
      kt_end();
      break;
    }
    case OP_HEAD:
      if (!manual) launch_decide(s);
      launch_head_friction(s, fv1 ? s.us.p : s.u.p, s.u.p, manual, mdt);
      break;
    case OP_STAGE1:
      kt_begin(KF_UNI_STAGE1);
      (s.p2 ? k_uni_march<1, true> : k_uni_march<1, false>)<<<mgrid, 128, 0, st>>>(
          v, nv, s.clk.p, s.red.p, s.u.p, nullptr, s.us.p, fv1 ? 1 : 0, manual, mdt, err);
      FM_LAUNCHED();
      kt_end();
      break;
    case OP_STAGE2:
      kt_begin(KF_UNI_STAGE2);
      (s.p2 ? k_uni_march<2, true> : k_uni_march<2, false>)<<<mgrid, 128, 0, st>>>(
          v, nv, s.clk.p, s.red.p, s.us.p, s.u.p, s.u.p, 1, manual, mdt, err);
      FM_LAUNCHED();
      kt_end();
      break;
    default:
      break;
  }
}

void un_launch_step(Sim& s, bool manual, double mdt, int* err) {
  for (int op : nu_step_ops(s, manual)) {
    if (op == OP_EXCH_U || op == OP_EXCH_US || op == OP_REDUCE) {
      if (s.shard) shard_op(s, op);
    } else {
      un_step_op(s, op, manual, mdt, err);
    }
  }
}

void un_launch_inflow_add(Sim& s, const double* per_cell_dev) {
  k_uni_inflow_add<<<nblk(s.n, 256), 256, 0, stream()>>>(uview(s), per_cell_dev, s.u.p);
  FM_LAUNCHED();
}

void un_launch_reduce_init(Sim& s) {
  // FV1 between steps keeps its state in U* (fv1_in_star): reduce over that
  const double* st = s.fv1_in_star ? s.us.p : s.u.p;
  k_uni_reduce_init<<<nblk(s.n, 256), 256, 0, stream()>>>(s.view(), s.nx, s.gy0, s.clk.p, s.red.p, st);
  FM_LAUNCHED();
}

}  // namespace fmh
