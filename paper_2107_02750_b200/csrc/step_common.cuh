// Device pieces shared by the non-uniform (nu_flow.cu) and uniform-raster
// (uniform.cu) step kernels: point states, the device drive-loop clock
// (run.cpp:80-111 + EventClock, sim_common.cpp:48-82) and the fused
// next-step reductions.
#pragma once

#include "fm_device.cuh"
#include "fm_sim.hpp"

namespace fmh {
namespace {

using namespace fmd;

struct Pt {
  double h, qx, qy, z, eta, u, v;
};

__device__ __forceinline__ double lsize(const NuView& v, int l) { return v.lsz[l]; }
__device__ __forceinline__ double lcen(double o, const NuView& v, int l, int i) {
  return o + (i + 0.5) * v.R * double(1 << (v.L - l));
}

// limit_at (solver_nonuniform.cpp:52-66)
__device__ __forceinline__ Pt limit(const double s[9], const P3& zc, double cx, double cy,
                                    double sz, double x, double y, double hdry) {
  Pt p;
  p.h = smax(0.0, eval_plane(P3{s[0], s[1], s[2]}, cx, cy, sz, x, y));
  p.qx = eval_plane(P3{s[3], s[4], s[5]}, cx, cy, sz, x, y);
  p.qy = eval_plane(P3{s[6], s[7], s[8]}, cx, cy, sz, x, y);
  p.z = eval_plane(zc, cx, cy, sz, x, y);
  p.eta = p.h + p.z;
  vel2(p.h, p.qx, p.qy, hdry, p.u, p.v);
  return p;
}

// P2 geometry (power-of-two element sizes, every coordinate exactly
// representable; checked on the host, Sim::p2): a point at offset (rx, ry)
// from the element centre in units of its size, rx, ry in {0, +-1/4, +-1/2}.
// There (x - xc) = rx R exactly and ((A (rx R)) / R) == A rx bit-for-bit, so
// evaluate (field.cpp:21-24) needs no division.
__device__ __forceinline__ double eval_rel(double c0, double cx, double cy, double rx, double ry) {
  return c0 + cx * 2.0 * kS3 * rx + cy * 2.0 * kS3 * ry;
}
// limit_rel with the topography's value at the point already known (static)
__device__ __forceinline__ Pt limit_rel_z(const double s[9], double z, double rx, double ry, double hdry) {
  Pt p;
  p.h = smax(0.0, eval_rel(s[0], s[1], s[2], rx, ry));
  p.qx = eval_rel(s[3], s[4], s[5], rx, ry);
  p.qy = eval_rel(s[6], s[7], s[8], rx, ry);
  p.z = z;
  p.eta = p.h + p.z;
  vel2(p.h, p.qx, p.qy, hdry, p.u, p.v);
  return p;
}
__device__ __forceinline__ Pt limit_rel(const double s[9], const P3& zc, double rx, double ry,
                                        double hdry) {
  Pt p;
  p.h = smax(0.0, eval_rel(s[0], s[1], s[2], rx, ry));
  p.qx = eval_rel(s[3], s[4], s[5], rx, ry);
  p.qy = eval_rel(s[6], s[7], s[8], rx, ry);
  p.z = eval_rel(zc.c0, zc.cx, zc.cy, rx, ry);
  p.eta = p.h + p.z;
  vel2(p.h, p.qx, p.qy, hdry, p.u, p.v);
  return p;
}

__device__ __forceinline__ void load9(const double* __restrict__ a, long long k, double s[9]) {
  const double* p = a + 9 * k;
#pragma unroll
  for (int q = 0; q < 9; ++q) s[q] = p[q];
}
__device__ __forceinline__ P3 load3(const double* __restrict__ a, long long k) {
  const double* p = a + 3 * k;
  return P3{p[0], p[1], p[2]};
}

// Vector forms for rows of 9 (72 B) and 3 (24 B) doubles in a 16 B aligned
// array: row k is 16 B aligned iff k is even, so one instruction sequence
// serves both parities — the 16 B part starts one double later for odd rows
// and the single double sits at the other end — and selects put the values
// back in order.  5 (2) memory instructions per row instead of 9 (3): the
// warp-wide 72 B-strided accesses touch half as many sector wavefronts.
__device__ __forceinline__ void load9v(const double* __restrict__ a, long long k, double s[9]) {
  const bool odd = k & 1;
  const double* p = a + 9 * k;
  const double2* pv = reinterpret_cast<const double2*>(p + (odd ? 1 : 0));
  double w[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double2 t = pv[i];
    w[2 * i] = t.x;
    w[2 * i + 1] = t.y;
  }
  const double x = p[odd ? 0 : 8];
  s[0] = odd ? x : w[0];
#pragma unroll
  for (int q = 1; q < 8; ++q) s[q] = odd ? w[q - 1] : w[q];
  s[8] = odd ? w[7] : x;
}
__device__ __forceinline__ void store9v(double* __restrict__ a, long long k, const double s[9]) {
  const bool odd = k & 1;
  double* p = a + 9 * k;
  double2* pv = reinterpret_cast<double2*>(p + (odd ? 1 : 0));
#pragma unroll
  for (int i = 0; i < 4; ++i)
    pv[i] = make_double2(odd ? s[2 * i + 1] : s[2 * i], odd ? s[2 * i + 2] : s[2 * i + 1]);
  p[odd ? 0 : 8] = odd ? s[0] : s[8];
}
__device__ __forceinline__ P3 load3v(const double* __restrict__ a, long long k) {
  const bool odd = k & 1;
  const double* p = a + 3 * k;
  const double2 t = *reinterpret_cast<const double2*>(p + (odd ? 1 : 0));
  const double x = p[odd ? 0 : 2];
  return odd ? P3{x, t.x, t.y} : P3{t.x, t.y, x};
}

__device__ __forceinline__ void store3v(double* __restrict__ a, long long k, double x0, double x1, double x2) {
  const bool odd = k & 1;
  double* p = a + 3 * k;
  *reinterpret_cast<double2*>(p + (odd ? 1 : 0)) = odd ? make_double2(x1, x2) : make_double2(x0, x1);
  p[odd ? 0 : 2] = odd ? x0 : x2;
}
// A flow row of width W: the 72 B rows of U (W = 9), or FV1's compact rows
// (W = 3: h, qx, qy means; the slopes are +0 exactly and read as +0)
template <int W>
__device__ __forceinline__ void load_row(const double* __restrict__ a, long long k, double s[9]) {
  if constexpr (W == 9) {
    load9v(a, k, s);
  } else {
    const P3 p = load3v(a, k);
    s[0] = p.c0, s[1] = 0.0, s[2] = 0.0;
    s[3] = p.cx, s[4] = 0.0, s[5] = 0.0;
    s[6] = p.cy, s[7] = 0.0, s[8] = 0.0;
  }
}
template <int W>
__device__ __forceinline__ void store_row(double* __restrict__ a, long long k, const double s[9]) {
  if constexpr (W == 9)
    store9v(a, k, s);
  else
    store3v(a, k, s[0], s[3], s[6]);
}

__device__ __forceinline__ unsigned long long leaf_key(int l, int i, int j) {
  return (static_cast<unsigned long long>(l) << 58) | (static_cast<unsigned long long>(j) << 29) |
         static_cast<unsigned long long>(i);
}

// hydrograph_at (hydrograph.cpp:38-49)
__device__ double hydro_at(const Hydro& h, int f, double t) {
  const int a = h.off[f], b = h.off[f + 1];
  if (t <= h.t[a]) return h.q[a];
  if (t >= h.t[b - 1]) return h.q[b - 1];
  int hi = a;
  while (hi < b && !(t < h.t[hi])) ++hi;
  const int lo = hi - 1;
  if (t == h.t[lo]) return h.q[lo];
  const double w = (t - h.t[lo]) / (h.t[hi] - h.t[lo]);
  return h.q[lo] + w * (h.q[hi] - h.q[lo]);
}

__device__ __forceinline__ bool reached(double now, double target) {
  return now >= target - 1e-9 * smax(1.0, target);
}

// The drive-loop bookkeeping for one step (run.cpp:80-111 with EventClock,
// sim_common.cpp:48-82).  Pure function of the step-start clock and the
// previous step's reductions, so every block derives the same decision; block
// 0 publishes it as clk[1].  It first closes the previous step (non-finite
// guard, then the gauge/output event counters, in the reference's order),
// then decides whether to run this step, computes dt = clip(compute_dt) and
// advances the clock and the inflow sources (apply_inflows uses the
// step-start time, run.cpp:84).
__device__ bool decide_step(const DevClock& c0, const DevRed& r, const Hydro* hy, int scheme,
                            double courant, double g, double hdry, int ninflow, DevClock& c) {
  c = c0;
  if (c.active && c.had_step) {
    if (r.badkey != ~0ull) {
      c.blew_up = 1;
      c.blow_t = c.now;
      c.bad_key = r.badkey;
      c.active = 0;
    } else {
      bool ev = false;
      if (c.gauge_int > 0.0 && reached(c.now, c.next_gauge * c.gauge_int)) {
        ++c.next_gauge;
        ev = true;
      }
      if (c.out_int > 0.0 && reached(c.now, c.next_out * c.out_int)) {
        ++c.next_out;
        ev = true;
      }
      if (ev && c.stop_at_events) {
        c.event_due = 1;
        c.active = 0;
      }
    }
  }
  c.had_step = 0;
  if (c.active && (c.now >= c.end_time || c.steps >= c.max_steps)) c.active = 0;
  c.finished = c.now >= c.end_time;
  if (!c.active) return false;
  double raw;
  if (scheme == FM_ACC) {
    const double hmax = bitsd(~r.hmaxc);
    raw = hmax <= hdry ? INFINITY : courant * bitsd(r.dtmin) / sqrt(g * hmax);
  } else {
    raw = bitsd(r.dtmin) * courant;
  }
  double e = c.end_time;
  if (c.out_int > 0.0) e = smin(e, c.next_out * c.out_int);
  if (c.gauge_int > 0.0) e = smin(e, c.next_gauge * c.gauge_int);
  const double gap = smax(e - c.now, 0.0);
  double dt = smin(raw, gap);
  if (!(dt > 0.0)) dt = smin(c.end_time, gap);
  c.dt = dt;
  c.t0 = c.now;
  double added = 0.0;
  for (int f = 0; f < ninflow; ++f) {
    const double q = hydro_at(*hy, f, c.now);
    if (q <= 0.0) {
      c.on[f] = 0;
      c.per_cell[f] = 0.0;
      continue;
    }
    const double vol = q * dt;
    c.on[f] = 1;
    c.per_cell[f] = vol / double(hy->region[f]);
    added += vol;
  }
  c.vol_in += added;
  c.now += dt;
  c.steps += 1;
  c.dt_min = smin(c.dt_min, dt);
  c.dt_max = smax(c.dt_max, dt);
  c.had_step = 1;
  c.finished = c.now >= c.end_time;
  return true;
}

// The step decision, once per step by a single thread (k_decide): evaluate
// decide_step on the step-start clock and the previous step's reductions,
// publish the in-flight clock clk[1] and clear the reduction slot this step
// accumulates into.  The step's kernels then only read clk[1].
__device__ __forceinline__ void decide_publish(const NuView& v, DevClock* clk, DevRed* red,
                                               const Hydro* hy) {
  const DevClock c0 = clk[1];  // the last published state
  const int p = int(c0.steps & 1);
  DevClock c;
  const bool g = decide_step(c0, red[p], hy, v.scheme, v.courant, v.g, v.hdry, v.ninflow, c);
  clk[1] = c;
  if (g) {
    DevRed& nx = red[p ^ 1];
    nx.dtmin = dbits(INFINITY);
    nx.hmaxc = ~0ull;
    nx.badkey = ~0ull;
  }
}

// Step head of the first kernel of every scheme: whether this step runs, and dt.
__device__ __forceinline__ void step_head(const NuView& v, DevClock* clk, DevRed* red,
                                          const Hydro* hy, int manual, double mdt, int& go,
                                          double& dt) {
  if (manual) {
    go = 1;
    dt = mdt;
    return;
  }
  const DevClock* c = clk + 1;
  go = c->active;
  dt = c->dt;
}

// Next-step reductions over the freshly written state (fused epilogue).
__device__ __forceinline__ void reduce_leaf(const NuView& v, DevRed* red, const DevClock& c,
                                            const double s[9], double sz, unsigned long long key,
                                            bool valid) {
  double dtc = INFINITY, hm = 0.0;
  unsigned long long bad = ~0ull;
  if (valid) {
    const double h = s[0];
    if (v.scheme == FM_ACC) {
      if (h > v.hdry) {
        hm = h;
        dtc = sz;
      }
    } else if (h > v.hdry) {
      const double cw = sqrt(v.g * h);
      double ux, uy;
      zdiv2(s[3], s[6], h, ux, uy);
      const double sx = fabs(ux) + cw;
      const double sy = fabs(uy) + cw;
      dtc = ddiv(sz, smax(sx, sy));
    }
    bool fin = true;
#pragma unroll
    for (int q = 0; q < 9; ++q) fin = fin && isfinite(s[q]);
    if (!fin) bad = key;
  }
  // warp minimum of the CFL candidates: they are >= 0 (or NaN), where the
  // order of the bit patterns is the numeric order, so two 32-bit REDUX
  // minima (high word, then the low word among the lanes holding that high
  // word) give the exact minimum; a NaN candidate never wins
  const unsigned long long db = dbits(dtc);
  const unsigned hi = __reduce_min_sync(0xffffffffu, unsigned(db >> 32));
  const unsigned lo = __reduce_min_sync(0xffffffffu, unsigned(db >> 32) == hi ? unsigned(db) : 0xffffffffu);
  const unsigned long long dmin = (static_cast<unsigned long long>(hi) << 32) | lo;
  if (v.scheme == FM_ACC) {  // grid-uniform: the depth maximum only for ACC
    for (int o = 16; o; o >>= 1) hm = smax(hm, __shfl_xor_sync(0xffffffffu, hm, o));
  }
  if (__any_sync(0xffffffffu, bad != ~0ull)) {  // the non-finite guard, rarely taken
    for (int o = 16; o; o >>= 1) {
      const unsigned long long b2 = __shfl_xor_sync(0xffffffffu, bad, o);
      bad = b2 < bad ? b2 : bad;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    DevRed& r = red[(c.steps) & 1];
    if (dmin < dbits(INFINITY)) atomicMin(&r.dtmin, dmin);
    if (hm > 0.0) atomicMin(&r.hmaxc, ~dbits(hm));
    if (bad != ~0ull) atomicMin(&r.badkey, bad);
  }
}

}  // namespace
}  // namespace fmh
