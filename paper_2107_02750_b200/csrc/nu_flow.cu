// Per-timestep flow updates on the non-uniform leaf set (sm_100a, fp64).
//
// Replaces NonUniformSim::step_rk / step_acc / compute_dt / apply_inflows /
// finite_state (solver_nonuniform.cpp:306-487) and the drive-loop body
// (run.cpp:80-111).  Leaves in Morton order; per DG2 step:
//
//   k_decide         the step decision (compute_dt :427-449 + EventClock::clip
//                    from the previous step's reduction), one thread.
//   k_head_friction  Manning friction (sim_common.cpp:30-46) in place.
//   k_seg            one thread per interior segment: segment_states
//                    (:91-115), the HLL flux of every face solved once.
//   k_stage<1>       one thread per leaf: side-effective states from the
//                    segment states, assemble, L operator, Euler update,
//                    positivity (:117-304).
//   k_seg, k_stage<2>  the same on U*, RK2 average, then (fused epilogue) the
//                    inflow sources, the non-finite guard and the CFL
//                    reduction for the next step.
//   k_acc_faces / k_acc_leaves   ACC (step_acc :350-418).
//
// All sums are gathers in the reference's order (sides N,E,S,W; sub-faces
// south-to-north / west-to-east), never floating-point atomics, so results
// do not depend on scheduling.
#include "fm_device.cuh"
#include "fm_sim.hpp"
#include "step_common.cuh"

// minimum resident CTAs per SM (register caps; tuned on B200 with
// scripts/ab_profile.py)
// 1: the segment and stage kernels have no early exit on inactive steps (A/B
// on B200: 0.799 -> 0.792 ms/step; the row loads issue ahead of the clock load)
#ifndef FM_NO_EXIT
#define FM_NO_EXIT 1
#endif
// compact FV1 rows (W = 3): 6 CTAs per SM (0.105 -> 0.101 ms, profiles/r2d_ab_seg_minb.txt)
#ifndef FM_SEG_MINB3
#define FM_SEG_MINB3 6
#endif
#ifndef FM_SEG_MINB
#define FM_SEG_MINB 5  // 51 registers: 5 CTAs of 256 threads per SM (4: 0.135, 5: 0.132, 6: 0.155 ms after the static z limits)
#endif

using namespace fmd;

namespace fmh {

namespace {

// ---- the step decision (one thread) -------------------------------------
__global__ void k_decide(NuView v, DevClock* clk, DevRed* red, const Hydro* hy) {
  decide_publish(v, clk, red, hy);
}

// ---- step head: clock + friction (DG2/FV1) ------------------------------
// src == dst for DG2; FV1 keeps its post-step state in U* (see k_stage) and
// the head moves it back into U while applying friction.
template <int W>
__global__ void __launch_bounds__(256) k_head_friction(NuView v, DevClock* clk, DevRed* red,
                                                      const Hydro* hy, const double* src,
                                                      double* dst, int manual, double mdt) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int go;
  double dt;
  step_head(v, clk, red, hy, manual, mdt, go, dt);
  if (!go || k >= v.n) return;
  if (src == dst) {
    // in place (DG2): friction reads h.c0, qx.c0, qy.c0 and writes q.c0 (wet)
    // or zeroes both discharges (dry); the other coefficients stay in HBM
    double* o = dst + 9 * k;
    const double h0 = o[0];
    if (h0 <= v.hdry) {
#pragma unroll
      for (int q = 3; q < 9; ++q) o[q] = 0.0;
      return;
    }
    double s[9];
    s[0] = h0;
    s[3] = o[3];
    s[6] = o[6];
    const double q3 = s[3], q6 = s[6];
    friction(s, v.nman[k], v.g, v.hdry, dt, v.libm);
    if (s[3] != q3 || s[6] != q6) {  // bit-level: friction changed them
      o[3] = s[3];
      o[6] = s[6];
    }
    return;
  }
  double s[9];
  if constexpr (W == 9) {
    load9(src, k, s);
  } else {
    load_row<W>(src, k, s);
  }
  friction(s, v.nman[k], v.g, v.hdry, dt, v.libm);
  if constexpr (W == 9) {
    double* o = dst + 9 * k;
#pragma unroll
    for (int q = 0; q < 9; ++q) o[q] = s[q];
  } else {
    store_row<W>(dst, k, s);
  }
}

// The DG2 head in place with FM_HEAD_LPT leaves per thread (strided by the
// block size, so the loads stay coalesced), every row's three values and
// Manning n loaded before the friction chains (A/B on B200, config 4: the
// former head 0.062 ms; this kernel 0.053 / 0.055 / 0.056 ms at 1 / 2 / 4
// leaves per thread).
#ifndef FM_HEAD_LPT
#define FM_HEAD_LPT 1
#endif
__global__ void __launch_bounds__(256) k_head_fric_ip(NuView v, DevClock* clk, DevRed* red, const Hydro* hy,
                                                     double* __restrict__ u, int manual, double mdt) {
  constexpr int P = FM_HEAD_LPT;
  const long long k0 = blockIdx.x * (long long)(P * blockDim.x) + threadIdx.x;
  int go;
  double dt;
  step_head(v, clk, red, hy, manual, mdt, go, dt);
  if (!go) return;
  double h[P], a[P], b[P], nm[P];
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const long long k = k0 + j * (long long)blockDim.x;
    const long long kc = k < v.n ? k : v.n - 1;
    h[j] = u[9 * kc];
    a[j] = u[9 * kc + 3];
    b[j] = u[9 * kc + 6];
    nm[j] = v.nman[kc];
  }
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const long long k = k0 + j * (long long)blockDim.x;
    if (k >= v.n) continue;
    double* o = u + 9 * k;
    if (h[j] <= v.hdry) {
#pragma unroll
      for (int q = 3; q < 9; ++q) o[q] = 0.0;
      continue;
    }
    double s[9];
    s[0] = h[j];
    s[3] = a[j];
    s[6] = b[j];
    friction(s, nm[j], v.g, v.hdry, dt, v.libm);
    if (s[3] != a[j] || s[6] != b[j]) {  // bit-level: friction changed them
      o[3] = s[3];
      o[6] = s[6];
    }
  }
}

// ---- segment states ------------------------------------------------------
// One thread per interior segment (segment_states, solver_nonuniform.cpp:91-115):
// both leaves' limits at the segment centre, z* = max(zL, zR), the starred
// depths and the HLL flux, stored as {m, n, t, z*, h*L, h*R}.  Every segment
// runs the same code path (one HLL), unlike a per-leaf-side formulation where
// lanes of a warp face 0, 1 or 2 sub-faces and every face is solved twice.
template <bool P2, int W>
__global__ void __launch_bounds__(256, W == 3 ? FM_SEG_MINB3 : FM_SEG_MINB) k_seg(NuView v, const DevClock* __restrict__ clk,
                                             const double* __restrict__ in, double* __restrict__ out,
                                             int manual, int* err, long long q0, long long q1) {
  const long long q = q0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= q1 || (v.nseg_dev && q >= *v.nseg_dev)) return;  // adaptive: q1 is an upper bound
  const int a = v.seg_l[q], b = v.seg_r[q];  // W/S and E/N leaf (loaded before the active check)
#if FM_NO_EXIT
  const bool act = manual || clk[1].active;
  if (!act) err = nullptr;
#else
  if (!manual && !clk[1].active) return;
  const bool act = true;
#endif
  double sa[9], sb[9];
  load_row<W>(in, a, sa);
  load_row<W>(in, b, sb);
  // P2: the static topography limits at the segment centre (k_seg_z) in one
  // 16 B load instead of both leaves' z rows and two plane evaluations
  const double2 zz = P2 ? v.segz[q] : make_double2(0.0, 0.0);
  const P3 za = P2 ? P3{0.0, 0.0, 0.0} : load3v(v.z, a), zb = P2 ? P3{0.0, 0.0, 0.0} : load3v(v.z, b);
  Pt A, B;
  bool xn;
  if (P2) {
    // enumerate_faces geometry (quadgrid.cpp:222-245) as exact offsets: the
    // centre lies on the face, at the finer (or either) leaf's centre along
    // it.  Static per segment, precomputed (k_seg_geo): no gathers of the
    // leaves' keys on this kernel's critical path.
    const int gc = v.seg_geo[q];
    xn = gc & 1;
    const int ca = (gc >> 1) & 3, cb = (gc >> 3) & 3;
    const double ta = ca == 0 ? 0.0 : ca == 2 ? 0.25 : -0.25;
    const double tb = cb == 0 ? 0.0 : cb == 2 ? 0.25 : -0.25;
    // one evaluation path for the x- and y-normal segments that interleave in
    // a warp: select the offsets, not the call
    A = limit_rel_z(sa, zz.x, xn ? 0.5 : ta, xn ? ta : 0.5, v.hdry);
    B = limit_rel_z(sb, zz.y, xn ? -0.5 : tb, xn ? tb : -0.5, v.hdry);
  } else {
    const int la = v.lvl[a], lb = v.lvl[b];
    const int ia = v.li[a], ja = v.lj[a], ib = v.li[b], jb = v.lj[b];
    // x-normal iff b starts where a ends along x (fine-cell units)
    xn = (ib << (v.L - lb)) == ((ia + 1) << (v.L - la));
    const double sza = lsize(v, la), szb = lsize(v, lb);
    const double cxa = lcen(v.x0, v, la, ia), cya = lcen(v.y0, v, la, ja);
    const double cxb = lcen(v.x0, v, lb, ib), cyb = lcen(v.y0, v, lb, jb);
    // owner: the coarser leaf, or the W/S leaf at equal level; it fixes the
    // normal coordinate from its face, the other leaf the tangential one
    const bool own_a = la <= lb;
    double x, y;
    if (xn) {
      x = own_a ? cxa + sza / 2 : cxb - szb / 2;
      y = own_a ? cyb : cya;
    } else {
      y = own_a ? cya + sza / 2 : cyb - szb / 2;
      x = own_a ? cxb : cxa;
    }
    A = limit(sa, za, cxa, cya, sza, x, y, v.hdry);
    B = limit(sb, zb, cxb, cyb, szb, x, y, v.hdry);
  }
  const double zs = smax(A.z, B.z);
  const double hl = smax(0.0, A.eta - zs), hr = smax(0.0, B.eta - zs);
  // rotate to the face normal (x-normal: n = x; y-normal: n = y)
  const double unA = xn ? A.u : A.v, utA = xn ? A.v : A.u;
  const double unB = xn ? B.u : B.v, utB = xn ? B.v : B.u;
  const Flx f = hll_inl(hl, hl * unA, hl * utA, hr, hr * unB, hr * utB, v.g, v.hdry, err);
  if (!act) return;
  double2* o = reinterpret_cast<double2*>(out + 6 * q);  // 16 B aligned
  o[0] = make_double2(f.m, f.n);
  o[1] = make_double2(f.t, zs);
  o[2] = make_double2(hl, hr);
}

// ---- one RK stage over all leaves ---------------------------------------
// STAGE 1: out = positivity(U + dt L(U))               -> U*  (FV1: the full step)
// STAGE 2: out = positivity(((U* + dt L(U*)) + U) / 2) -> U (in place)
//
// One thread per leaf takes its four sides in turn (E, W, then N, S): the
// side's face limit (limit_at, solver_nonuniform.cpp:52-66), the
// side-effective starred state from the side's segment states
// (side_effective :117-178), the side's flux sum with the pressure correction
// (assemble :190-226); then the Gauss-point physical fluxes, the L operator,
// the update and positivity.  (A four-threads-per-leaf layout with the sides
// meeting in shared memory measured 1.6x slower on B200: the per-lane
// redundant update and the exchange cost more than the parallel sides gain.)
struct SideOut {
  double h, qx, qy, zd, fm, fn, ft;
};

// 1: the stage kernels keep the leaf's own row (9 + 3 doubles) in a per-thread
// shared-memory slot and reload it where it is used (each side's face limit,
// the update) instead of holding it in registers across the kernel: no spills
// at 102 registers, 10 CTAs per SM (A/B on B200: 0.796 -> 0.775 ms/step,
// bit-identical)
#ifndef FM_STAGE_SROW
#define FM_STAGE_SROW 1
#endif
#ifndef FM_SID_ROW
#define FM_SID_ROW 1
#endif
#ifndef FM_FV1_CONST
#define FM_FV1_CONST 1
#endif
template <bool P2, int W = 9>
__device__ __forceinline__ SideOut side_eval(const NuView& v, const double s[9], const P3& zc,
                                             long long kk, int sd, int kind, double cx, double cy,
                                             double sz, int* err, int2 ids,
                                             const volatile double* lrow) {
  const bool xn = sd == 1 || sd == 3;
  const bool mine_left = sd == 0 || sd == 1;
  const int nseg = kind == 0 ? 0 : kind == 3 ? 2 : 1;
  double sg[2][6];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    if (t < nseg) {
      // 48 B state, 16 B aligned: three 16 B loads
#if FM_SID_ROW
      const int id = t == 0 ? ids.x : ids.y;
#else
      const int id = v.sid[8 * kk + 2 * sd + t];
#endif
      const double2* q = reinterpret_cast<const double2*>(v.segst + 6 * (long long)id);
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        const double2 w2 = q[e];
        sg[t][2 * e] = w2.x;
        sg[t][2 * e + 1] = w2.y;
      }
    }
  }
  const double ox = sd == 1 ? 0.5 : sd == 3 ? -0.5 : 0.0;
  const double oy = sd == 0 ? 0.5 : sd == 2 ? -0.5 : 0.0;
  const double fx = P2 ? 0.0 : cx + (sd == 1 ? sz / 2 : sd == 3 ? -sz / 2 : 0.0);
  const double fy = P2 ? 0.0 : cy + (sd == 0 ? sz / 2 : sd == 2 ? -sz / 2 : 0.0);
#if FM_STAGE_SROW
  // the leaf's row from its shared-memory copy, read where it is used
  double sl[9];
#pragma unroll
  // W = 3 (compact FV1 rows): the slopes are +0 by construction (load_row),
  // so they are literals here rather than opaque shared-memory reads
  // (FM_FV1_CONST 2: the three means stay in registers too, so the four
  // sides' identical limit values -- their two divisions -- are formed once)
  for (int q = 0; q < 9; ++q)
    sl[q] = (FM_FV1_CONST && W == 3 && q % 3 != 0) ? 0.0 : (FM_FV1_CONST == 2 && W == 3) ? s[q] : lrow[q];
  // P2: the leaf's static topography limit on this side (k_seg_z's zside,
  // in lrow[9 + sd]) instead of its z plane evaluated here
  const P3 zl{lrow[9], lrow[10], lrow[11]};
  const Pt me = P2 ? limit_rel_z(sl, lrow[9 + sd], ox, oy, v.hdry) : limit(sl, zl, cx, cy, sz, fx, fy, v.hdry);
#else
  const Pt me = P2 ? limit_rel_z(s, v.zside[4 * kk + sd], ox, oy, v.hdry) : limit(s, zc, cx, cy, sz, fx, fy, v.hdry);
#endif
  const double w = kind == 3 ? 0.5 : 1.0;
  double zstar;
  if (kind == 0) {
    zstar = me.z;
  } else if (nseg == 1) {
    zstar = sg[0][3];
  } else if (v.zpair) {
    zstar = smax(me.z, v.zpair[4 * kk + sd]);
  } else {
    double acc = 0.0;
    acc += w * sg[0][3];
    acc += w * sg[1][3];
    zstar = acc;
  }
  SideOut o;
  const double h = smax(0.0, me.eta - zstar);
  o.h = h;
  o.qx = h * me.u;
  o.qy = h * me.v;
  o.zd = zstar - smax(0.0, zstar - me.eta);
  Flx acc{0.0, 0.0, 0.0};
  if (kind == 0) {
    const double qn = xn ? o.qx : o.qy, qt = xn ? o.qy : o.qx;
    const double qg = v.bc[sd] == FM_REFLECTIVE ? -qn : qn;
    const Flx f = mine_left ? hll(h, qn, qt, h, qg, qt, v.g, v.hdry, err)
                            : hll(h, qg, qt, h, qn, qt, v.g, v.hdry, err);
    acc.m += f.m;
    acc.n += f.n;
    acc.t += f.t;
  } else {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (t < nseg) {
        const double hme = mine_left ? sg[t][4] : sg[t][5];
        const double corr = 0.5 * v.g * (h * h - hme * hme);
        acc.m += w * sg[t][0];
        acc.n += w * (sg[t][1] + corr);
        acc.t += w * sg[t][2];
      }
    }
  }
  o.fm = acc.m;
  o.fn = acc.n;
  o.ft = acc.t;
  return o;
}

// 64-thread CTAs, >= 10 resident per SM (a 102-register cap, with the row in
// shared memory; 8 / 9 / 11 / 12 and 128-thread CTAs measured slower): tuned
// by A/B on B200 (scripts/ab_profile.py)
#ifndef FM_STAGE_THREADS
#define FM_STAGE_THREADS 64
#endif
#ifndef FM_STAGE_MINB
#define FM_STAGE_MINB 10
#endif
// the compact FV1 stage (W = 3) keeps far fewer values live: its own cap
#ifndef FM_STAGE_MINB3
#define FM_STAGE_MINB3 FM_STAGE_MINB
#endif

// LIST: the leaves are list[0..cnt) (a shard's stage split) instead of 0..n-1
template <int STAGE, bool P2, int W = 9, bool LIST = false>
__global__ void __launch_bounds__(FM_STAGE_THREADS, W == 3 ? FM_STAGE_MINB3 : FM_STAGE_MINB) k_stage(
    NuView v, const DevClock* __restrict__ clk, DevRed* red, const double* __restrict__ in,
    const double* uold, double* out, int last, int manual, double mdt, int* err,
    const int32_t* __restrict__ list, long long cnt) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool valid = LIST ? t < cnt : t < v.n;
  const long long kk = LIST ? (long long)list[valid ? t : cnt - 1] : (valid ? t : v.n - 1);
  // the leaf's rows are loaded before the step-active check: they do not
  // depend on it, and the check's clock load would otherwise put a second
  // round trip in front of the first gathers
  const int l = v.lvl[kk], i = v.li[kk], j = v.lj[kk];
  double s[9];
  load_row<W>(in, kk, s);
  // P2: the four static side limits of the topography (N E S W, k_seg_z);
  // otherwise the z plane
  P3 zc{0.0, 0.0, 0.0};
  double2 zs01 = make_double2(0.0, 0.0), zs23 = make_double2(0.0, 0.0);
  if (P2) {
    const double2* zp = reinterpret_cast<const double2*>(v.zside + 4 * kk);
    zs01 = zp[0];
    zs23 = zp[1];
  } else {
    zc = load3v(v.z, kk);
  }
  const int code = v.sk[kk];
#if FM_STAGE_SROW
  __shared__ double srow_all[FM_STAGE_THREADS * 13];  // 13-double stride: conflict-free
  volatile double* lrow = srow_all + 13 * threadIdx.x;
#pragma unroll
  for (int q = 0; q < 9; ++q)
    if (!(FM_FV1_CONST && W == 3 && q % 3 != 0)) lrow[q] = s[q];
  if (P2) {
    lrow[9] = zs01.x;
    lrow[10] = zs01.y;
    lrow[11] = zs23.x;
    lrow[12] = zs23.y;
  } else {
    lrow[9] = zc.c0;
    lrow[10] = zc.cx;
    lrow[11] = zc.cy;
  }
#else
  const volatile double* lrow = nullptr;
#endif
  // the leaf's segment ids, 2 per side (N E S W), as two 16 B loads
#if FM_SID_ROW
  const int4* srow = reinterpret_cast<const int4*>(v.sid + 8 * kk);
  const int4 s03 = srow[0], s47 = srow[1];
  const int2 idn{s03.x, s03.y}, ide{s03.z, s03.w}, ids_{s47.x, s47.y}, idw{s47.z, s47.w};
#else
  const int2 idn{0, 0}, ide{0, 0}, ids_{0, 0}, idw{0, 0};
#endif
  const DevClock* c = clk + 1;
#if FM_NO_EXIT
  // no early exit: an inactive step (rare: the tail of a graph batch after an
  // event) computes on a stale dt with every side effect predicated off, so
  // the compiler keeps all the row loads ahead of the clock load
  const bool act = manual || c->active;
  if (!act) err = nullptr;
#else
  if (!manual && !c->active) return;
  const bool act = true;
#endif
  const double dt = manual ? mdt : c->dt;
  const double sz = lsize(v, l);
  const double inv = v.linv[l];
  const double cx = P2 ? 0.0 : lcen(v.x0, v, l, i), cy = P2 ? 0.0 : lcen(v.y0, v, l, j);
  const bool dg2 = (FM_FV1_CONST && W == 3) ? false : v.scheme == FM_DG2;
  const bool epi = last && !manual;
  // the first inflow's count for this leaf, loaded early: its latency
  // otherwise sits at the end of the leaf's critical path
  const int cnt0 = (epi && v.ninflow > 0) ? v.infc[kk] : 0;
  // x direction: E and W sides, then the Gauss-point fluxes along x
  const SideOut ee = side_eval<P2, W>(v, s, zc, kk, 1, (code >> 2) & 3, cx, cy, sz, err, ide, lrow);
  const SideOut ew = side_eval<P2, W>(v, s, zc, kk, 3, (code >> 6) & 3, cx, cy, sz, err, idw, lrow);
  const DirMod X{0.5 * (ee.h + ew.h),   (ee.h - ew.h) * kHalfInvS3,   0.5 * (ee.qx + ew.qx),
                 (ee.qx - ew.qx) * kHalfInvS3, 0.5 * (ee.qy + ew.qy), (ee.qy - ew.qy) * kHalfInvS3,
                 (ee.zd - ew.zd) * kHalfInvS3};
  double xp[3] = {0, 0, 0}, xm[3] = {0, 0, 0};
  if (dg2) {
    phys_x(X.h0 + X.h1, X.qx0 + X.qx1, X.qy0 + X.qy1, v.g, v.hdry, xp[0], xp[1], xp[2]);
    phys_x(X.h0 - X.h1, X.qx0 - X.qx1, X.qy0 - X.qy1, v.g, v.hdry, xm[0], xm[1], xm[2]);
  }
  const Flx fe{ee.fm, ee.fn, ee.ft}, fw{ew.fm, ew.fn, ew.ft};
  // the x direction's share of the L operator (solver_nonuniform.cpp:228-271)
  // now, so only seven doubles (three slopes, three flux differences, the x
  // bed-slope source) stay live through the y direction instead of X, the
  // fluxes and the Gauss-point fluxes; the same operations on the same
  // operands (A/B on B200: step 0.778 -> 0.758 ms, bit-identical)
  double Lr[9];
  const double kk3 = P2 ? kS3 * inv : kS3 / sz;
  if (dg2) {
    Lr[1] = -kk3 * (fe.m + fw.m - xp[0] - xm[0]);
    Lr[4] = -kk3 * (fe.n + fw.n - xp[1] - xm[1]) - div_sz<P2>(v.g * X.h1 * (2.0 * kS3 * X.z1), sz, inv);
    Lr[7] = -kk3 * (fe.t + fw.t - xp[2] - xm[2]);
  }
  const double dxm = fe.m - fw.m, dxn = fe.n - fw.n, dxt = fe.t - fw.t;
  const double srcx = div_sz<P2>(v.g * X.h0 * (2.0 * kS3 * X.z1), sz, inv);
  // y direction
  const SideOut en = side_eval<P2, W>(v, s, zc, kk, 0, code & 3, cx, cy, sz, err, idn, lrow);
  const SideOut es = side_eval<P2, W>(v, s, zc, kk, 2, (code >> 4) & 3, cx, cy, sz, err, ids_, lrow);
  const DirMod Y{0.5 * (en.h + es.h),   (en.h - es.h) * kHalfInvS3,   0.5 * (en.qx + es.qx),
                 (en.qx - es.qx) * kHalfInvS3, 0.5 * (en.qy + es.qy), (en.qy - es.qy) * kHalfInvS3,
                 (en.zd - es.zd) * kHalfInvS3};
  double yp[3] = {0, 0, 0}, ym[3] = {0, 0, 0};
  if (dg2) {
    phys_y(Y.h0 + Y.h1, Y.qx0 + Y.qx1, Y.qy0 + Y.qy1, v.g, v.hdry, yp[0], yp[1], yp[2]);
    phys_y(Y.h0 - Y.h1, Y.qx0 - Y.qx1, Y.qy0 - Y.qy1, v.g, v.hdry, ym[0], ym[1], ym[2]);
  }
  const Flx fn{en.fm, en.fn, en.ft}, fs{es.fm, es.fn, es.ft};
  // the y direction's share and the means
  Lr[0] = div_sz<P2>(-(dxm + (fn.m - fs.m)), sz, inv);
  Lr[3] = div_sz<P2>(-(dxn + (fn.t - fs.t)), sz, inv) - srcx;
  Lr[6] = div_sz<P2>(-(dxt + (fn.n - fs.n)), sz, inv) -
          div_sz<P2>(v.g * Y.h0 * (2.0 * kS3 * Y.z1), sz, inv);
  if (dg2) {
    Lr[2] = -kk3 * (fn.m + fs.m - yp[0] - ym[0]);
    Lr[5] = -kk3 * (fn.t + fs.t - yp[1] - ym[1]);
    Lr[8] = -kk3 * (fn.n + fs.n - yp[2] - ym[2]) - div_sz<P2>(v.g * Y.h1 * (2.0 * kS3 * Y.z1), sz, inv);
  } else {
    Lr[1] = Lr[2] = Lr[4] = Lr[5] = Lr[7] = Lr[8] = 0.0;
  }
  double res[9];
#if FM_STAGE_SROW
#pragma unroll
  for (int q = 0; q < 9; ++q)
    s[q] = (FM_FV1_CONST && W == 3 && q % 3 != 0) ? 0.0 : (FM_FV1_CONST == 2 && W == 3) ? s[q] : lrow[q];
#endif
  if (STAGE == 1) {
#pragma unroll
    for (int q = 0; q < 9; ++q) res[q] = s[q] + Lr[q] * dt;
  } else {
    double u0[9];
    load_row<W>(uold, kk, u0);
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
  if (epi && valid) {
    // apply_inflows (solver_nonuniform.cpp:451-465), inflow order.  P2: the
    // leaf area is a power of two, so / (sz sz) is exactly * (inv inv)
    for (int f = 0; f < v.ninflow; ++f) {
      if (!c->on[f]) continue;
      const int cnt = f == 0 ? cnt0 : v.infc[f * v.n + kk];
      if (cnt) {
        const double num = c->per_cell[f] * cnt;
        res[0] += P2 ? num * (inv * inv) : ddiv(num, sz * sz);
      }
    }
  }
  if (valid && act) store_row<W>(out, kk, res);
  if (epi && act) reduce_leaf(v, red, *c, res, sz, leaf_key(l, i, j), valid);
}

// ---- ACC ------------------------------------------------------------------
// ACC's state is h.c0, qx.c0, qy.c0 (the slopes are zero and never change,
// solver_nonuniform.cpp:600-607), so while the device loop runs it lives in
// three compact arrays (SoA) instead of the 72 B rows: the face kernel's
// leaf gathers (h, z.c0, n, level: 25 B per leaf, ~60 MB at config 4) stay
// L2-resident, and the leaf kernel writes 24 B per leaf instead of three
// partial sectors of a row.  acc_to_soa / acc_to_aos (sim.cu) convert at the
// API boundary.  The arithmetic is the reference's, operand for operand.

// Per interior segment (solver_nonuniform.cpp:354-371).  Also the step head.
// FM_ACC_SPT segments per thread (strided by the block size, so every load
// stays coalesced): the independent gather chains (segment ids -> leaf
// depth / level / Manning) of several segments are in flight together.
#ifndef FM_ACC_SPT
#define FM_ACC_SPT 2
#endif
#ifndef FM_ACC_FACE_THREADS
#define FM_ACC_FACE_THREADS 128
#endif
template <bool P2>
__global__ void __launch_bounds__(FM_ACC_FACE_THREADS) k_acc_faces(NuView v, DevClock* clk, DevRed* red,
                                                  const Hydro* hy, const double* __restrict__ ch,
                                                  const double* __restrict__ czc,
                                                  double* __restrict__ q, int manual, double mdt) {
  constexpr int S = FM_ACC_SPT;
  // blocks in reverse order (FM_ACC_REV): the leaf kernel that follows walks
  // the leaves forward, so the discharges written last -- the low segments,
  // owned by the low leaves -- are the first it gathers, still in L2; and this
  // kernel gathers the depths the previous leaf kernel wrote last first
#ifndef FM_ACC_REV
#define FM_ACC_REV 1
#endif
  const long long blk = FM_ACC_REV ? (long long)gridDim.x - 1 - blockIdx.x : (long long)blockIdx.x;
  const long long s0 = blk * (long long)(S * blockDim.x) + threadIdx.x;
  int go;
  double dt;
  step_head(v, clk, red, hy, manual, mdt, go, dt);
  if (!go) return;
  int l[S], r[S];
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const long long sj = s0 + j * (long long)blockDim.x;
    const long long sc = sj < v.nseg ? sj : v.nseg - 1;
    l[j] = v.seg_l[sc];
    r[j] = v.seg_r[sc];
  }
  double zl[S], zr[S], hl[S], hr[S], Qo[S], nl[S], nr[S];
  int al[S], ar[S];
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const long long sj = s0 + j * (long long)blockDim.x;
    const long long sc = sj < v.nseg ? sj : v.nseg - 1;
    zl[j] = czc[l[j]];
    zr[j] = czc[r[j]];
    hl[j] = ch[l[j]];
    hr[j] = ch[r[j]];
    Qo[j] = q[sc];
    al[j] = v.lvl[l[j]];
    ar[j] = v.lvl[r[j]];
    nl[j] = v.nman[l[j]];
    nr[j] = v.nman[r[j]];
  }
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const long long sj = s0 + j * (long long)blockDim.x;
    if (sj >= v.nseg) break;
    const double el = hl[j] + zl[j], er = hr[j] + zr[j];
    const double hf = smax(el, er) - smax(zl[j], zr[j]);
    double Q = Qo[j];
    if (hf <= v.hdry) {
      q[sj] = 0.0;
      continue;
    }
    const double dist = 0.5 * (lsize(v, al[j]) + lsize(v, ar[j]));
    const double nf = 0.5 * (nl[j] + nr[j]);
    // P2, equal levels: dist is the (power-of-two) leaf size and / dist is
    // exactly * 1/size
    const double grad = (P2 && al[j] == ar[j]) ? (v.g * hf * dt * (er - el)) * v.linv[al[j]]
                                               : ddiv(v.g * hf * dt * (er - el), dist);
    Q = ddiv(Q - grad, 1.0 + zdiv(v.g * dt * nf * nf * fabs(Q), pow73_m(hf, v.libm)));
    q[sj] = Q;
  }
}

// The next step's ACC reductions (compute_dt :429-437, finite_state :479-487)
// of a block: the minimum wet leaf size, the maximum wet depth and the minimum
// key of a leaf with a non-finite coefficient, warp then block reduced, one
// atomic per block and field (one per warp put ~150 k same-address atomics
// in every step's tail).
template <int NT>
__device__ __forceinline__ void reduce_acc(DevRed* red, const DevClock& c, double h, double sz,
                                           double hdry, unsigned long long bad, bool valid) {
  double dtc = INFINITY, hm = 0.0;
  if (valid && h > hdry) {
    hm = h;
    dtc = sz;
  }
  unsigned long long db = dbits(dtc);
  const unsigned hi = __reduce_min_sync(0xffffffffu, unsigned(db >> 32));
  const unsigned lo = __reduce_min_sync(0xffffffffu, unsigned(db >> 32) == hi ? unsigned(db) : 0xffffffffu);
  db = (static_cast<unsigned long long>(hi) << 32) | lo;
  for (int o = 16; o; o >>= 1) hm = smax(hm, __shfl_xor_sync(0xffffffffu, hm, o));
  if (__any_sync(0xffffffffu, bad != ~0ull)) {
    for (int o = 16; o; o >>= 1) {
      const unsigned long long b2 = __shfl_xor_sync(0xffffffffu, bad, o);
      bad = b2 < bad ? b2 : bad;
    }
  }
  constexpr int W = NT / 32;
  __shared__ unsigned long long s_d[W], s_b[W];
  __shared__ double s_h[W];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_d[w] = db;
    s_h[w] = hm;
    s_b[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 1; k < W; ++k) {
      db = s_d[k] < db ? s_d[k] : db;
      hm = smax(hm, s_h[k]);
      bad = s_b[k] < bad ? s_b[k] : bad;
    }
    DevRed& r = red[(c.steps) & 1];
    if (db < dbits(INFINITY)) atomicMin(&r.dtmin, db);
    if (hm > 0.0) atomicMin(&r.hmaxc, ~dbits(hm));
    if (bad != ~0ull) atomicMin(&r.badkey, bad);
  }
}

// Per leaf: boundary discharges (:372-386), volume update and diagnostic
// discharges (:387-417), then the fused inflow / finite / CFL epilogue.
// A side's sub-face length needs no neighbour lookup: on a graded grid it is
// the leaf's size, or half of it when the side has two (finer) neighbours
// (kind 3) -- the same IEEE value as min(size_l, size_r).
#ifndef FM_ACC_LEAF_THREADS
#define FM_ACC_LEAF_THREADS 128
#endif
#ifndef FM_ACC_HOIST
#define FM_ACC_HOIST 1
#endif
constexpr int kAccLeafThreads = FM_ACC_LEAF_THREADS;
template <bool P2>
__global__ void __launch_bounds__(kAccLeafThreads) k_acc_leaves(
    NuView v, const DevClock* __restrict__ clk, DevRed* red, double* __restrict__ ch,
    double* __restrict__ cqx, double* __restrict__ cqy, const double* __restrict__ q,
    double* __restrict__ qb, const unsigned long long* __restrict__ slope_bad, int manual, double mdt) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const DevClock* c = clk + 1;
  if (!manual && !c->active) return;
  const double dt = manual ? mdt : c->dt;
  const bool valid = k < v.n;
  double h = 0.0, sz = 0.0;
  unsigned long long bad = ~0ull;
  if (valid) {
    const int l = v.lvl[k];
    sz = lsize(v, l);
    const double inv = v.linv[l];  // P2: 1 / sz exactly
    h = ch[k];
    const uint8_t code = v.sk[k];
    const int4* srow = reinterpret_cast<const int4*>(v.sid + 8 * k);
    const int4 s03 = srow[0], s47 = srow[1];
    const int ids[8] = {s03.x, s03.y, s03.z, s03.w, s47.x, s47.y, s47.z, s47.w};
    const double area = sz * sz;
    double net = 0.0, sx = 0.0, sy = 0.0;
#if FM_ACC_HOIST
    // every side's discharge gathers issued together, ahead of the side
    // loop's branches (an unused slot holds -1 and loads nothing)
    double Qs[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) Qs[t] = ids[t] >= 0 ? q[ids[t]] : 0.0;
#endif
#pragma unroll
    for (int sd = 0; sd < 4; ++sd) {
      const int kind = (code >> (2 * sd)) & 3;
      const double sign = (sd == 1 || sd == 0) ? -1.0 : 1.0;
      if (kind == 0) {
        double b = qb[4 * k + sd];
        if (v.bc[sd] == FM_REFLECTIVE) {
          b = 0.0;
        } else {
          const double hf = h;
          if (hf <= v.hdry) {
            b = 0.0;
          } else {
            const double nf = v.nman[k];
            b = zdiv(b, 1.0 + zdiv(v.g * dt * nf * nf * fabs(b), pow73_m(hf, v.libm)));
          }
        }
        qb[4 * k + sd] = b;
        net += sign * b * sz;
        if (sd == 1 || sd == 3)
          sx += b * sz;
        else
          sy += b * sz;
      } else {
        const double len = kind == 3 ? 0.5 * sz : sz;
        const int nseg = kind == 3 ? 2 : 1;
        for (int t = 0; t < nseg; ++t) {
#if FM_ACC_HOIST
          const double Q = t ? Qs[2 * sd + 1] : Qs[2 * sd];
#else
          const double Q = q[ids[2 * sd + t]];
#endif
          net += sign * Q * len;
          if (sd == 1 || sd == 3)
            sx += Q * len;
          else
            sy += Q * len;
        }
      }
    }
    // P2: the leaf size and area are powers of two, so the divisions are
    // exact reciprocal multiplies (bit-identical)
    h += P2 ? (dt * net) * (inv * inv) : zdiv(dt * net, area);
    const double qx = div_sz<P2>(0.5 * sx, sz, inv);
    const double qy = div_sz<P2>(0.5 * sy, sz, inv);
    if (!manual) {
      for (int f = 0; f < v.ninflow; ++f) {
        if (!c->on[f]) continue;
        const int cnt = v.infc[f * v.n + k];
        if (cnt) {
          const double num = c->per_cell[f] * cnt;
          h += P2 ? num * (inv * inv) : ddiv(num, area);
        }
      }
    }
    ch[k] = h;
    cqx[k] = qx;
    cqy[k] = qy;
    if (!(isfinite(h) && isfinite(qx) && isfinite(qy))) bad = leaf_key(l, v.li[k], v.lj[k]);
  }
  if (!manual) {
    // the slopes never change under ACC: their non-finite key (if any) was
    // found when the state entered the compact layout
    if (k == 0 && *slope_bad != ~0ull) bad = min(bad, *slope_bad);
    reduce_acc<kAccLeafThreads>(red, *c, h, sz, v.hdry, bad, valid);
  }
}

// Layout changes of the ACC state.  To SoA: h, qx, qy from the rows, z.c0 of
// every local leaf (owned + halo) and the minimum key of a leaf with a
// non-finite slope.  To the rows: c0 of h, qx, qy (the slopes are untouched).
__global__ void k_acc_to_soa(long long n, long long ntot, const int8_t* __restrict__ lvl,
                             const int32_t* __restrict__ li, const int32_t* __restrict__ lj,
                             const double* __restrict__ u, const double* __restrict__ z,
                             double* __restrict__ ch, double* __restrict__ cqx, double* __restrict__ cqy,
                             double* __restrict__ czc, unsigned long long* __restrict__ slope_bad) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= ntot) return;
  czc[k] = z[3 * k];
  ch[k] = u[9 * k];
  if (k >= n) return;
  cqx[k] = u[9 * k + 3];
  cqy[k] = u[9 * k + 6];
  const double* r = u + 9 * k;
  if (!(isfinite(r[1]) && isfinite(r[2]) && isfinite(r[4]) && isfinite(r[5]) && isfinite(r[7]) &&
        isfinite(r[8])))
    atomicMin(slope_bad, leaf_key(lvl[k], li[k], lj[k]));
}

__global__ void k_acc_to_aos(long long n, const double* __restrict__ ch, const double* __restrict__ cqx,
                             const double* __restrict__ cqy, double* __restrict__ u) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  u[9 * k] = ch[k];
  u[9 * k + 3] = cqx[k];
  u[9 * k + 6] = cqy[k];
}

// Initial reduction (before the first step of a run) into slot steps&1.
// ACC in the compact layout: c0 of h, qx, qy from the compact arrays (the
// slopes in U are current: ACC never changes them).
__global__ void k_reduce_init(NuView v, const DevClock* clk, DevRed* red, const double* __restrict__ u,
                              const double* __restrict__ ch, const double* __restrict__ cqx,
                              const double* __restrict__ cqy, int cst) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool valid = k < v.n;
  double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double sz = 0.0;
  unsigned long long key = 0;
  if (valid) {
    const int l = v.lvl[k];
    sz = lsize(v, l);
    key = leaf_key(l, v.li[k], v.lj[k]);
    load9(u, k, s);
    if (ch) {
      s[0] = ch[cst * k];
      s[3] = cqx[cst * k];
      s[6] = cqy[cst * k];
    }
  }
  DevClock c = clk[1];
  reduce_leaf(v, red, c, s, sz, key, valid);
}

// Close the last step of a run: the non-finite guard and event counters of
// decide_step without starting a new step.
__global__ void k_close(DevClock* clk, DevRed* red, const Hydro* hy, NuView v) {
  DevClock c0 = clk[1];
  c0.max_steps = c0.steps;  // forbid a new step
  DevClock c;
  decide_step(c0, red[c0.steps & 1], hy, v.scheme, v.courant, v.g, v.hdry, v.ninflow, c);
  c.max_steps = clk[1].max_steps;
  clk[1] = c;
}


// apply_inflows for the host API path.
__global__ void k_inflow_add(NuView v, const double* per_cell, double* u) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= v.n) return;
  const double sz = lsize(v, v.lvl[k]);
  double h = u[9 * k];
  for (int f = 0; f < v.ninflow; ++f) {
    const double pc = per_cell[f];
    if (pc == 0.0) continue;
    const int cnt = v.infc[f * v.n + k];
    if (cnt) h += pc * cnt / (sz * sz);
  }
  u[9 * k] = h;
}

inline unsigned nblk(long long n, int t) { return unsigned((n + t - 1) / t); }

}  // namespace

void launch_decide(Sim& s);

// ---- launch helpers used by sim.cu --------------------------------------------
// A step is a fixed sequence of operations (StepOp): device phases plus, for a
// sharded sim, the halo exchanges of the state a phase is about to gather and
// the cross-rank reduction of the next-step CFL / non-finite slot.
//   DG2: HEAD  X(U)  STAGE1  X(U*)  STAGE2  REDUCE
//   FV1: HEAD  X(U)  STAGE1  REDUCE
//   ACC: X(U)  ACC  REDUCE
// (manual host-API steps have no REDUCE).  HEAD and ACC start with the
// one-thread step decision (k_decide).
std::vector<int> nu_step_ops(const Sim& s, bool manual) {
  std::vector<int> ops;
  if (s.scheme == FM_ACC) {
    ops = {OP_EXCH_U, OP_ACC};
  } else if (s.scheme == FM_FV1) {
    ops = {OP_HEAD, OP_EXCH_U, OP_STAGE1};
  } else {
    ops = {OP_HEAD, OP_EXCH_U, OP_STAGE1, OP_EXCH_US, OP_STAGE2};
  }
  if (!manual) ops.push_back(OP_REDUCE);
  return ops;
}

// The device phases of a step (exchange / reduce ops are the shard layer's).
void nu_step_op(Sim& s, int op, bool manual, double mdt, int* err) {
  cudaStream_t st = stream();
  const NuView v = s.view();
  DevClock* clk = s.clk.p;
  DevRed* red = s.red.p;
  const long long n = s.n;
  const long long ns = std::max<long long>(s.nseg, 1);
  const bool fv1 = s.scheme == FM_FV1;
  // Segment states over [q0, q1).  A sharded sim orders its segments with
  // the ones that touch only owned leaves first: those run while the halo
  // exchange is in flight on the shard's side stream, the rest after it.
  // FV1 in the compact layout (s.fv1c): rows of 3 (h, qx, qy means) in
  // s.cu3 (U) and s.cs3 (U*) instead of the 72 B rows of U and U*
  const bool c3 = s.fv1c;
  auto seg_range = [&](const double* in, long long q0, long long q1) {
    if (q1 <= q0) return;
    auto kern = s.p2 ? (c3 ? k_seg<true, 3> : k_seg<true, 9>) : (c3 ? k_seg<false, 3> : k_seg<false, 9>);
    launch_k(kern, nblk(q1 - q0, 256), 256, st, v, (const DevClock*)clk, in, s.segst.p, (int)manual, err, q0, q1);
    FM_LAUNCHED();
  };
  auto seg = [&](int fam, const double* in) {
    kt_begin(fam);
    const long long inner = s.shard ? std::min<long long>(s.nseg_inner, ns) : ns;
    seg_range(in, 0, inner);
    if (s.shard) shard_finish(s);  // the halo has landed
    seg_range(in, inner, ns);
    kt_end();
  };
  switch (op) {
    case OP_ACC:
      if (s.shard) shard_finish(s);
      if (!manual) launch_decide(s);
      kt_begin(KF_ACC_FACES);
      (s.p2 ? k_acc_faces<true> : k_acc_faces<false>)<<<nblk(ns, FM_ACC_FACE_THREADS * FM_ACC_SPT), FM_ACC_FACE_THREADS, 0, st>>>(
          v, clk, red, s.hydro.p, s.ch.p, s.czc.p, s.accq.p, manual, mdt);
      FM_LAUNCHED();
      kt_end();
      kt_begin(KF_ACC_LEAVES);
      (s.p2 ? k_acc_leaves<true> : k_acc_leaves<false>)<<<nblk(n, kAccLeafThreads), kAccLeafThreads, 0, st>>>(
          v, clk, red, s.ch.p, s.cqx.p, s.cqy.p, s.accq.p, s.accqb.p, s.cbad.p, manual, mdt);
      FM_LAUNCHED();
      kt_end();
      break;
    case OP_HEAD:
      if (!manual) launch_decide(s);
      // FV1 keeps its state in U* between steps; the head moves it to U with friction
      kt_begin(KF_HEAD);
      if (c3)
        launch_k(k_head_friction<3>, nblk(n, 256), 256, st, v, clk, red, (const Hydro*)s.hydro.p,
                 (const double*)s.cs3.p, s.cu3.p, (int)manual, mdt);
      else if (!fv1)  // DG2: in place
        launch_k(k_head_fric_ip, nblk(n, 256 * FM_HEAD_LPT), 256, st, v, clk, red, (const Hydro*)s.hydro.p, s.u.p,
                 (int)manual, mdt);
      else
        launch_k(k_head_friction<9>, nblk(n, 256), 256, st, v, clk, red, (const Hydro*)s.hydro.p,
                 (const double*)s.us.p, s.u.p, (int)manual, mdt);
      FM_LAUNCHED();
      kt_end();
      break;
    case OP_STAGE1: {
      const double* in = c3 ? s.cu3.p : s.u.p;
      double* out = c3 ? s.cs3.p : s.us.p;
      seg(KF_SEG1, in);
      kt_begin(KF_STAGE1);
      const int last1 = fv1 ? 1 : 0;
      if (s.shard && !fv1) {
        // the stage split: the leaves a peer needs first, then (NCCL) their
        // U* exchange starts on the side stream while the rest run
        Shard& sh = *s.shard;
        auto lk = s.p2 ? k_stage<1, true, 9, true> : k_stage<1, false, 9, true>;
        if (sh.n_first) {
          launch_k(lk, nblk(sh.n_first, FM_STAGE_THREADS), FM_STAGE_THREADS, st, v, (const DevClock*)clk, red, in,
                   (const double*)nullptr, out, last1, (int)manual, mdt, err, (const int32_t*)sh.stage_first.p,
                   (long long)sh.n_first);
          FM_LAUNCHED();
        }
        if (shard_nccl(s)) {
          shard_op(s, OP_EXCH_US);
          sh.us_started = true;
        }
        if (sh.n_rest) {
          launch_k(lk, nblk(sh.n_rest, FM_STAGE_THREADS), FM_STAGE_THREADS, st, v, (const DevClock*)clk, red, in,
                   (const double*)nullptr, out, last1, (int)manual, mdt, err, (const int32_t*)sh.stage_rest.p,
                   (long long)sh.n_rest);
          FM_LAUNCHED();
        }
        kt_end();
        break;
      }
      auto kern = s.p2 ? (c3 ? k_stage<1, true, 3> : k_stage<1, true, 9>)
                       : (c3 ? k_stage<1, false, 3> : k_stage<1, false, 9>);
      launch_k(kern, nblk(n, FM_STAGE_THREADS), FM_STAGE_THREADS, st, v, (const DevClock*)clk, red, in,
               (const double*)nullptr, out, last1, (int)manual, mdt, err, (const int32_t*)nullptr, 0ll);
      FM_LAUNCHED();
      kt_end();
      break;
    }
    case OP_STAGE2:
      seg(KF_SEG2, s.us.p);
      kt_begin(KF_STAGE2);
      if (s.p2)
        launch_k(k_stage<2, true, 9>, nblk(n, FM_STAGE_THREADS), FM_STAGE_THREADS, st, v, (const DevClock*)clk, red, (const double*)s.us.p, (const double*)s.u.p, s.u.p, 1, (int)manual, mdt, err, (const int32_t*)nullptr, 0ll);
      else
        launch_k(k_stage<2, false, 9>, nblk(n, FM_STAGE_THREADS), FM_STAGE_THREADS, st, v, (const DevClock*)clk, red, (const double*)s.us.p, (const double*)s.u.p, s.u.p, 1, (int)manual, mdt, err, (const int32_t*)nullptr, 0ll);
      FM_LAUNCHED();
      kt_end();
      break;
    default:
      break;
  }
}

void nu_launch_step(Sim& s, bool manual, double mdt, int* err) {
  for (int op : nu_step_ops(s, manual)) {
    if (op == OP_EXCH_US && s.shard && s.shard->us_started) {
      s.shard->us_started = false;  // already in flight (the stage split)
      continue;
    }
    if (op == OP_EXCH_U || op == OP_EXCH_US || op == OP_REDUCE) {
      if (s.shard) shard_op(s, op);
    } else {
      nu_step_op(s, op, manual, mdt, err);
    }
  }
}

void launch_decide(Sim& s) {
  kt_begin(KF_DECIDE);
  launch_k(k_decide, 1, 1, stream(), s.view(), s.clk.p, s.red.p, (const Hydro*)s.hydro.p);
  FM_LAUNCHED();
  kt_end();
}

void launch_head_friction(Sim& s, const double* src, double* dst, bool manual, double mdt) {
  kt_begin(s.uniform ? KF_UNI_HEAD : KF_HEAD);
  if (src == dst)  // DG2: in place
    k_head_fric_ip<<<nblk(s.n, 256 * FM_HEAD_LPT), 256, 0, stream()>>>(s.view(), s.clk.p, s.red.p, s.hydro.p, dst,
                                                                       manual, mdt);
  else
    k_head_friction<9><<<nblk(s.n, 256), 256, 0, stream()>>>(s.view(), s.clk.p, s.red.p, s.hydro.p, src,
                                                              dst, manual, mdt);
  FM_LAUNCHED();
  kt_end();
}


void nu_launch_reduce_init(Sim& s) {
  // the compact layouts hold the means (ACC: three arrays; FV1: rows of 3 in U*)
  const double* ch = s.acc_soa ? s.ch.p : s.fv1c ? s.cs3.p : nullptr;
  const double* cqx = s.acc_soa ? s.cqx.p : s.fv1c ? s.cs3.p + 1 : nullptr;
  const double* cqy = s.acc_soa ? s.cqy.p : s.fv1c ? s.cs3.p + 2 : nullptr;
  // FV1 on 72 B rows between steps keeps its state in U* (fv1_in_star)
  const double* st = s.fv1_in_star ? s.us.p : s.u.p;
  k_reduce_init<<<nblk(s.n, 256), 256, 0, stream()>>>(s.view(), s.clk.p, s.red.p, st, ch, cqx, cqy,
                                                       s.fv1c ? 3 : 1);
  FM_LAUNCHED();
}

void nu_launch_close(Sim& s) {
  k_close<<<1, 1, 0, stream()>>>(s.clk.p, s.red.p, s.hydro.p, s.view());
  FM_LAUNCHED();
}

void nu_launch_acc_to_soa(Sim& s, long long ntot) {
  s.ch.alloc(size_t(ntot));
  s.czc.alloc(size_t(ntot));
  s.cqx.alloc(size_t(s.n));
  s.cqy.alloc(size_t(s.n));
  s.cbad.alloc(1);
  s.cbad.fill_bytes(0xff);
  k_acc_to_soa<<<nblk(ntot, 256), 256, 0, stream()>>>(s.n, ntot, s.lvl.p, s.li.p, s.lj.p, s.u.p, s.z.p, s.ch.p,
                                                       s.cqx.p, s.cqy.p, s.czc.p, s.cbad.p);
  FM_LAUNCHED();
}

void nu_launch_acc_to_aos(Sim& s) {
  k_acc_to_aos<<<nblk(s.n, 256), 256, 0, stream()>>>(s.n, s.ch.p, s.cqx.p, s.cqy.p, s.u.p);
  FM_LAUNCHED();
}

namespace {
// FV1 into the compact layout: the means of U's rows into U* compact (the
// next step's head moves them to U compact with friction); `nz` counts owned
// leaves with a slope that is not +0 exactly (then the compact path is off)
__global__ void k_fv1_to_c(long long n, const double* __restrict__ u, double* __restrict__ cs3,
                           unsigned long long* __restrict__ nz) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double* r = u + 9 * k;
  store3v(cs3, k, r[0], r[3], r[6]);
  const unsigned long long o = dbits(r[1]) | dbits(r[2]) | dbits(r[4]) | dbits(r[5]) | dbits(r[7]) | dbits(r[8]);
  if (o) atomicAdd(nz, 1ull);
}
__global__ void k_c3_to_u(long long n, const double* __restrict__ cs3, double* __restrict__ u) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const P3 p = load3v(cs3, k);
  u[9 * k] = p.c0;
  u[9 * k + 3] = p.cx;
  u[9 * k + 6] = p.cy;
}
}  // namespace

// Returns whether the compact FV1 layout is in use (every slope +0).
bool nu_fv1_to_compact(Sim& s, long long ntot) {
  s.cu3.alloc(size_t(3 * ntot));
  s.cs3.alloc(size_t(3 * s.n));
  DBuf<unsigned long long> nz(1);
  nz.zero();
  k_fv1_to_c<<<nblk(s.n, 256), 256, 0, stream()>>>(s.n, s.u.p, s.cs3.p, nz.p);
  FM_LAUNCHED();
  unsigned long long h = 0;
  nz.download(&h, 1);
  FM_CUDA(cudaStreamSynchronize(stream()));
  return h == 0;
}

void nu_c3_to_u(Sim& s) {
  k_c3_to_u<<<nblk(s.n, 256), 256, 0, stream()>>>(s.n, s.cs3.p, s.u.p);
  FM_LAUNCHED();
}

void nu_launch_inflow_add(Sim& s, const double* per_cell_dev) {
  k_inflow_add<<<nblk(s.n, 256), 256, 0, stream()>>>(s.view(), per_cell_dev, s.u.p);
  FM_LAUNCHED();
}

}  // namespace fmh
