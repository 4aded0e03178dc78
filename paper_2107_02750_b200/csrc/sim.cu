// Host side of the device simulations: construction (make_nonuniform_sim,
// solver_nonuniform.cpp:558-636), the drive<Sim> member functions
// (run.cpp:35-141) and the device-resident step loop captured in a CUDA graph.
#include <algorithm>
#include <cstdio>
#include <memory>
#include <cmath>
#include <cstring>
#include <limits>

#include "fm_device.cuh"
#include "fm_sim.hpp"

using namespace fmd;

namespace fmh {

void nu_launch_step(Sim& s, bool manual, double mdt, int* err);
void nu_launch_reduce_init(Sim& s);
void nu_launch_close(Sim& s);
void nu_launch_inflow_add(Sim& s, const double* per_cell_dev);
void nu_launch_acc_to_soa(Sim& s, long long ntot);
bool nu_fv1_to_compact(Sim& s, long long ntot);
void nu_c3_to_u(Sim& s);
void nu_launch_acc_to_aos(Sim& s);
// uniform.cu
void un_launch_step(Sim& s, bool manual, double mdt, int* err);
void un_launch_reduce_init(Sim& s);
void un_launch_inflow_add(Sim& s, const double* per_cell_dev);
// adaptive.cu
struct AdaptState;
void adaptive_destroy(AdaptState* a);

namespace {

inline unsigned nblk(long long n, int t) { return unsigned((n + t - 1) / t); }

__device__ __forceinline__ double lsz(int L, double R, int l) { return R * double(1 << (L - l)); }

// restrict_flow_to_leaves (solver_nonuniform.cpp:529-556) for an h-only fine
// field: leaf k takes the level-l scaling of its node.
__global__ void k_ic_restrict(long long n, int M, const int8_t* __restrict__ lvl,
                              const int32_t* __restrict__ li, const int32_t* __restrict__ lj,
                              const double* const* __restrict__ sc, double* __restrict__ u) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int l = lvl[k];
  const uint64_t node = node_index(l, li[k], lj[k], M);
  const double* p = sc[l] + 3 * node;
  double* o = u + 9 * k;
  o[0] = p[0];
  o[1] = p[1];
  o[2] = p[2];
#pragma unroll
  for (int q = 3; q < 9; ++q) o[q] = 0.0;
}

// flow_from_surface (solver_uniform.cpp:60-71) / uniform initial depth.
__global__ void k_ic_simple(long long n, const double* __restrict__ z, int mode, double val,
                            double* __restrict__ u) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double f[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (mode == 1) {
    const double c0 = z[3 * k], cx = z[3 * k + 1], cy = z[3 * k + 2];
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
  double* o = u + 9 * k;
#pragma unroll
  for (int q = 0; q < 9; ++q) o[q] = f[q];
}

// Piecewise-constant schemes drop slopes (solver_nonuniform.cpp:600-607),
// then positivity (:608).
__global__ void k_ic_finish(long long n, int pc, double hdry, double* __restrict__ z,
                            double* __restrict__ u) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double f[9];
  for (int q = 0; q < 9; ++q) f[q] = u[9 * k + q];
  if (pc) {
    z[3 * k + 1] = 0.0;
    z[3 * k + 2] = 0.0;
    f[1] = f[2] = 0.0;
    for (int q = 3; q < 9; ++q) f[q] = 0.0;
  }
  positivity(f, hdry);
  for (int q = 0; q < 9; ++q) u[9 * k + q] = f[q];
}

__global__ void k_finite(long long n, const int8_t* __restrict__ lvl, const int32_t* __restrict__ li,
                         const int32_t* __restrict__ lj, const double* __restrict__ u,
                         unsigned long long* bad) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  bool fin = true;
  for (int q = 0; q < 9; ++q) fin = fin && isfinite(u[9 * k + q]);
  if (!fin) {
    const unsigned long long key = (static_cast<unsigned long long>(lvl ? lvl[k] : 0) << 58) |
                                   (static_cast<unsigned long long>(lj[k]) << 29) |
                                   static_cast<unsigned long long>(li[k]);
    atomicMin(bad, key);
  }
}

}  // namespace

Sim::HostSlots& Sim::slots() {
  if (!host) {
    void* p = nullptr;
    FM_CUDA(cudaMallocHost(&p, sizeof(HostSlots)));
    host = static_cast<HostSlots*>(p);
    *host = HostSlots{};
  }
  return *host;
}

Sim::~Sim() {
  if (host) cudaFreeHost(host);
  if (shard && shard->comm) comm_forget(shard->comm, this);
  for (auto& g : gexec)
    if (g) cudaGraphExecDestroy(g);
  if (ad) adaptive_destroy(ad);
}

NuView Sim::view() const {
  NuView v{};
  v.L = L;
  v.M = M;
  v.N = N;
  v.scheme = scheme;
  v.adaptive = adaptive ? 1 : 0;
  v.ninflow = ninflow;
  v.libm = libm;
  v.R = R;
  v.x0 = x0;
  v.y0 = y0;
  v.g = g;
  v.hdry = hdry;
  v.courant = courant;
  for (int q = 0; q < 4; ++q) v.bc[q] = bc[q];
  for (int l = 0; l <= L && l < 16; ++l) {
    v.lsz[l] = R * double(1 << (L - l));
    v.linv[l] = 1.0 / v.lsz[l];
  }
  v.n = n;
  v.lvl = lvl.p;
  v.li = li.p;
  v.lj = lj.p;
  v.z = z.p;
  v.nman = nman.p;
  v.nb = nb.p;
  v.sk = sk.p;
  v.zpair = zpair.n ? zpair.p : nullptr;
  v.infc = infc.p;
  v.seg_l = seg_l.p;
  v.seg_r = seg_r.p;
  v.seg_geo = seg_geo.p;
  v.segz = reinterpret_cast<const double2*>(segz.p);
  v.zside = zside.p;
  v.sid = sid.p;
  v.segst = segst.p;
  v.nseg = nseg;
  v.nseg_dev = nseg_lazy ? nseg_dev.p : nullptr;
  return v;
}

namespace {

double courant_for(const fm_sim_desc* d) {  // config.cpp:37-47
  if (d->courant > 0.0) return d->courant;
  switch (d->solver) {
    case FM_DG2:
    case FM_MWDG2: return 0.33;
    case FM_FV1:
    case FM_HWFV1: return 0.5;
    case FM_ACC: return 0.7;
  }
  return 0.33;
}

void common_params(Sim& s, const fm_sim_desc* d) {
  if (d->solver < FM_DG2 || d->solver > FM_HWFV1) throw Error(FM_ERR_CONFIG, "unknown solver");
  s.solver = d->solver;
  s.libm = d->libm;
  s.scheme = d->solver == FM_MWDG2 ? FM_DG2 : d->solver == FM_HWFV1 ? FM_FV1 : d->solver;
  s.g = d->g;
  s.hdry = d->h_dry;
  s.courant = courant_for(d);
  for (int q = 0; q < 4; ++q) s.bc[q] = d->bc[q];
  s.manning = d->manning;
  if (d->manning_raster) {
    const fm_raster* m = d->manning_raster;
    s.has_mr = true;
    s.mr_ncols = m->ncols;
    s.mr_nrows = m->nrows;
    s.mr_xll = m->xll;
    s.mr_yll = m->yll;
    s.mr_cs = m->cellsize;
    // A static non-uniform sim samples the raster once per leaf at creation
    // (solver_nonuniform.cpp:575-584) and never again: a raster already
    // reachable from the device -- device memory, or page-locked host memory
    // through its mapped pointer (zero-copy: ~2 leaf lookups per cell row
    // cross PCIe instead of the whole raster) -- is read in place.  Adaptive
    // sims re-sample it at every adapt and uniform sims read every cell, so
    // they keep a device copy.
    const bool once = !s.uniform && !s.adaptive;
    const double* dp = nullptr;
    if (once && m->on_device) {
      dp = m->values;
    } else if (once) {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, m->values) == cudaSuccess && at.type == cudaMemoryTypeHost &&
          at.devicePointer)
        dp = static_cast<const double*>(at.devicePointer);
      else
        cudaGetLastError();  // pageable memory: not an error
    }
    if (dp) {
      s.mr_ext = dp;
    } else if (m->on_device) {
      s.mr.alloc(size_t(m->ncols) * m->nrows);
      FM_CUDA(cudaMemcpyAsync(s.mr.p, m->values, s.mr.n * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
    } else {
      s.mr.upload(m->values, size_t(m->ncols) * m->nrows);
    }
  }
  // inflows (config.cpp:168-186; hydrograph.cpp:10-36 validation)
  if (d->n_inflows > kMaxInflows) throw Error(FM_ERR_CONFIG, "too many inflows");
  s.ninflow = d->n_inflows;
  Hydro h{};
  int at = 0;
  for (int f = 0; f < d->n_inflows; ++f) {
    const fm_inflow& in = d->inflows[f];
    if (in.nsamples < 1) throw Error(FM_ERR_IO, "hydrograph has no samples");
    if (at + in.nsamples > kMaxHydroSamples) throw Error(FM_ERR_CONFIG, "hydrograph too long");
    if (in.i0 > in.i1 || in.j0 > in.j1)
      throw Error(FM_ERR_CONFIG, "inflow: cell range must satisfy i0 <= i1 and j0 <= j1");
    h.off[f] = at;
    for (int k = 0; k < in.nsamples; ++k) {
      if (k && !(in.t[k] > in.t[k - 1])) throw Error(FM_ERR_IO, "hydrograph times must be strictly increasing");
      if (in.q[k] < 0.0) throw Error(FM_ERR_IO, "hydrograph has a negative discharge");
      h.t[at + k] = in.t[k];
      h.q[at + k] = in.q[k];
    }
    at += in.nsamples;
    h.region[f] = (long long)(in.i1 - in.i0 + 1) * (in.j1 - in.j0 + 1);
    s.region.push_back(h.region[f]);
    s.rect.insert(s.rect.end(), {in.i0, in.j0, in.i1, in.j1});
    s.hy_t.emplace_back(in.t, in.t + in.nsamples);
    s.hy_q.emplace_back(in.q, in.q + in.nsamples);
  }
  h.off[d->n_inflows] = at;
  h.n = d->n_inflows;
  s.hydro.upload(&h, 1);
  s.clk.alloc(2);
  s.red.alloc(2);
}

}  // namespace

// The P2 fast path (Sim::p2) is exact when the fine cell size R is a power of
// two, the origin is a multiple of R/4 and every coordinate (and the R/4
// offsets of sub-face centres) is an exact double: then x - xc is exactly
// rx * size for rx in {0, +-1/4, +-1/2}, as the reference computes it.
bool geometry_is_p2(double R, double x0, double y0, int L, int M, int N) {
  if (!(R > 0.0) || !std::isfinite(R)) return false;
  int e = 0;
  if (std::frexp(R, &e) != 0.5) return false;
  const double q = R / 4.0;
  for (double o : {x0, y0}) {
    const double k = o / q;
    if (k != std::floor(k) || std::fabs(k) > 1e15) return false;
  }
  const double ext = double(std::max(M, N)) * std::ldexp(1.0, L) * R;
  return std::fabs(x0) / q + ext / q < 9.0e15 && std::fabs(y0) / q + ext / q < 9.0e15;
}

// Static non-uniform sim from a device grid (solver_nonuniform.cpp:558-636).
static void nonuniform_init(Sim& s, const fm_sim_desc* d, const fm_raster* dem, const Grid& g) {
  cudaStream_t st = stream();
  s.L = g.L;
  s.M = g.M;
  s.N = g.N;
  s.R = g.R;
  s.x0 = g.x0;
  s.y0 = g.y0;
  s.p2 = geometry_is_p2(s.R, s.x0, s.y0, s.L, s.M, s.N);
  s.n = g.nleaves;
  const long long n = s.n;
  s.lvl.alloc(n);
  s.li.alloc(n);
  s.lj.alloc(n);
  s.z.alloc(3 * n);
  FM_CUDA(cudaMemcpyAsync(s.lvl.p, g.lf_l.p, n, cudaMemcpyDeviceToDevice, st));
  FM_CUDA(cudaMemcpyAsync(s.li.p, g.lf_i.p, 4 * n, cudaMemcpyDeviceToDevice, st));
  FM_CUDA(cudaMemcpyAsync(s.lj.p, g.lf_j.p, 4 * n, cudaMemcpyDeviceToDevice, st));
  FM_CUDA(cudaMemcpyAsync(s.z.p, g.lf_z.p, 24 * n, cudaMemcpyDeviceToDevice, st));
  build_topology(s, g);  // throws StructureError when not graded (is_graded, :566-567)
  s.nman.alloc(n);
  resolve_manning(s);
  s.u.alloc(9 * n);
  s.us.alloc(9 * n);
  if (d->initial_depth_raster) {
    const fm_raster* hr = d->initial_depth_raster;
    if (hr->ncols != dem->ncols || hr->nrows != dem->nrows)
      throw Error(FM_ERR_CONFIG, "initial_depth_raster geometry must match the DEM");
    DBuf<double> fine;
    project_planes(hr, s.L, s.M, s.N, fine);
    std::vector<DBuf<double>> sc;
    scaling_pyramid(std::move(fine), s.L, s.M, s.N, FM_MW, sc);
    std::vector<const double*> ptrs(s.L + 1);
    for (int l = 0; l <= s.L; ++l) ptrs[l] = sc[l].p;
    DBuf<const double*> dptrs;
    dptrs.upload(ptrs.data(), ptrs.size());
    k_ic_restrict<<<nblk(n, 256), 256, 0, st>>>(n, s.M, s.lvl.p, s.li.p, s.lj.p, dptrs.p, s.u.p);
    FM_LAUNCHED();
    FM_CUDA(cudaStreamSynchronize(st));
  } else {
    const int mode = d->has_initial_surface ? 1 : d->initial_depth > 0.0 ? 2 : 0;
    k_ic_simple<<<nblk(n, 256), 256, 0, st>>>(n, s.z.p, mode,
                                               mode == 1 ? d->initial_surface : d->initial_depth, s.u.p);
    FM_LAUNCHED();
  }
  k_ic_finish<<<nblk(n, 256), 256, 0, st>>>(n, s.scheme != FM_DG2, s.hdry, s.z.p, s.u.p);
  FM_LAUNCHED();
  build_seg_z(s);  // the topography is final now (FV1 / ACC: z slopes zeroed)
  for (int f = 0; f < s.ninflow; ++f) {
    const int* r = &s.rect[4 * f];
    if (r[0] < 0 || r[1] < 0 || r[2] >= (s.M << s.L) || r[3] >= (s.N << s.L))
      throw Error(FM_ERR_CONFIG, "inflow region outside the domain");
  }
  resolve_inflows(s, g);
  if (s.scheme == FM_ACC) {
    s.accq.alloc(std::max<int64_t>(s.nseg, 1));
    s.accq.zero();
    s.accqb.alloc(4 * n);
    s.accqb.zero();
  }
}

// Initial conditions shared with the adaptive set-up.
void ic_surface_or_depth(Sim& s, const fm_sim_desc* d) {
  const int mode = d->has_initial_surface ? 1 : d->initial_depth > 0.0 ? 2 : 0;
  k_ic_simple<<<nblk(s.n, 256), 256, 0, stream()>>>(s.n, s.z.p, mode,
                                                     mode == 1 ? d->initial_surface : d->initial_depth, s.u.p);
  FM_LAUNCHED();
}
void ic_finish(Sim& s) {
  k_ic_finish<<<nblk(s.n, 256), 256, 0, stream()>>>(s.n, s.scheme != FM_DG2, s.hdry, s.z.p, s.u.p);
  FM_LAUNCHED();
}

Sim* sim_create(const fm_sim_desc* d, const fm_raster* dem, const Grid* grid) {
  FM_RANGE("fm_sim_create");
  if (!d || !dem) throw Error(FM_ERR_CONFIG, "null descriptor or DEM");
  upload_banks();
  auto s = std::make_unique<Sim>();
  s->adaptive = d->solver == FM_MWDG2 || d->solver == FM_HWFV1;
  s->uniform = !s->adaptive && !grid;
  common_params(*s, d);
  if (s->adaptive) {
    adaptive_init(*s, d, dem);
  } else if (grid) {
    nonuniform_init(*s, d, dem, *grid);
  } else {
    uniform_init(*s, d, dem);
  }
  FM_CUDA(cudaStreamSynchronize(stream()));
  s->mr_ext = nullptr;  // the caller's raster: not referenced after creation
  return s.release();
}

namespace {

// FV1 keeps its post-step state in U* while the device loop runs.
void fv1_to_u(Sim& s) {
  if (s.fv1_in_star) {
    FM_CUDA(cudaMemcpyAsync(s.u.p, s.us.p, s.u.n * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
    s.fv1_in_star = false;
  }
}
void fv1_to_star(Sim& s) {
  if (!s.fv1_in_star) {
    FM_CUDA(cudaMemcpyAsync(s.us.p, s.u.p, s.u.n * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
    s.fv1_in_star = true;
  }
}
bool fv1_staged(const Sim& s) { return s.scheme == FM_FV1; }

// ACC on a non-uniform grid keeps h, qx, qy in compact arrays between the API
// calls that read or write U (nu_flow.cu, k_acc_*).
bool acc_compact(const Sim& s) { return s.scheme == FM_ACC && !s.uniform && !s.adaptive; }
void acc_to_soa(Sim& s) {
  if (acc_compact(s) && !s.acc_soa) {
    nu_launch_acc_to_soa(s, s.n + (s.shard ? s.shard->n_halo : 0));
    s.acc_soa = true;
  }
}
void acc_to_u(Sim& s) {
  if (s.acc_soa) {
    nu_launch_acc_to_aos(s);
    s.acc_soa = false;
  }
}
// Every U consumer first brings the state back into U (FV1: from U*, ACC:
// from the compact arrays); every stepping entry point moves it out again.
// FV1 on a non-uniform grid runs on compact rows of 3 between the API calls
// that touch U, as long as every slope is +0 (FV1 never makes one non-zero;
// only an upload could): otherwise it stays on the 72 B rows.
#ifndef FM_FV1_COMPACT
#define FM_FV1_COMPACT 1
#endif
bool fv1_compact_ok(const Sim& s) { return FM_FV1_COMPACT && s.scheme == FM_FV1 && !s.uniform && !s.adaptive; }
void fv1c_to_u(Sim& s) {
  if (s.fv1c) {
    nu_c3_to_u(s);
    s.fv1c = false;
    s.fv1_in_star = false;
  }
}
void state_to_u(Sim& s) {
  fv1c_to_u(s);
  if (fv1_staged(s)) fv1_to_u(s);
  acc_to_u(s);
}
void state_to_step(Sim& s) {
  if (fv1_compact_ok(s) && !s.fv1c) {
    if (fv1_staged(s)) fv1_to_u(s);
    if (nu_fv1_to_compact(s, s.n + (s.shard ? s.shard->n_halo : 0))) {
      s.fv1c = true;
      return;
    }
  }
  if (s.fv1c) return;
  if (fv1_staged(s)) fv1_to_star(s);
  acc_to_soa(s);
}

__global__ void k_red_reset(DevRed* red, int p) {
  red[p].dtmin = 0x7ff0000000000000ull;  // +inf
  red[p].hmaxc = ~0ull;
  red[p].badkey = ~0ull;
}

void init_red(Sim& s) {
  DevRed r[2];
  for (auto& x : r) {
    double inf = std::numeric_limits<double>::infinity();
    std::memcpy(&x.dtmin, &inf, 8);
    x.hmaxc = ~0ull;
    x.badkey = ~0ull;
    x.pad = 0;
  }
  s.red.upload(r, 2);
}

void launch_step(Sim& s, bool manual, double mdt, int* err) {
  if (s.uniform)
    un_launch_step(s, manual, mdt, err);
  else
    nu_launch_step(s, manual, mdt, err);
}
void launch_reduce_init(Sim& s) {
  if (s.uniform)
    un_launch_reduce_init(s);
  else
    nu_launch_reduce_init(s);
  // a sharded sim's slots become global (NCCL; a local group combines in group_run)
  if (s.shard) shard_allreduce_u64_min(s, reinterpret_cast<unsigned long long*>(s.red.p), 8);
}

DevClock fresh_clock(const fm_clock* c, int64_t max_steps, int stop) {
  DevClock d{};
  d.end_time = c->end_time;
  d.out_int = c->output_interval;
  d.gauge_int = c->gauge_interval;
  d.now = c->now;
  d.next_out = c->next_output;
  d.next_gauge = c->next_gauge;
  d.max_steps = max_steps;
  d.active = 1;
  d.stop_at_events = stop;
  d.dt_min = std::numeric_limits<double>::infinity();
  d.dt_max = 0.0;
  d.bad_key = ~0ull;
  return d;
}

// The device clock: clk[1] is the published state (the step-start state of
// the next step once a step has been decided).
void read_clock(Sim& s, DevClock& c) {
  FM_CUDA(cudaMemcpyAsync(&c, s.clk.p + 1, sizeof(DevClock), cudaMemcpyDeviceToHost, stream()));
}

void key_xy(const Sim& s, unsigned long long key, double* bx, double* by) {
  const int l = int(key >> 58), j = int((key >> 29) & ((1u << 29) - 1)), i = int(key & ((1u << 29) - 1));
  if (s.uniform) {
    if (bx) *bx = s.x0 + (i + 0.5) * s.R;
    if (by) *by = s.y0 + (j + 0.5) * s.R;
  } else {
    if (bx) *bx = s.x0 + (i + 0.5) * s.R * double(1 << (s.L - l));
    if (by) *by = s.y0 + (j + 0.5) * s.R * double(1 << (s.L - l));
  }
}

}  // namespace

double sim_compute_dt(Sim& s) {
  FM_RANGE("fm_sim_compute_dt");
  state_to_u(s);
  init_red(s);
  DevClock pair0[2] = {};
  s.clk.upload(pair0, 2);  // steps = 0 -> slot 0
  launch_reduce_init(s);
  DevRed r[2];
  s.red.download(r, 2);
  FM_CUDA(cudaStreamSynchronize(stream()));
  double v;
  std::memcpy(&v, &r[0].dtmin, 8);
  if (s.scheme == FM_ACC) {
    double hmax;
    const unsigned long long hb = ~r[0].hmaxc;
    std::memcpy(&hmax, &hb, 8);
    if (hmax <= s.hdry) return std::numeric_limits<double>::infinity();
    if (s.uniform) return s.courant * s.R / std::sqrt(s.g * hmax);
    return s.courant * v / std::sqrt(s.g * hmax);
  }
  return v * s.courant;
}

void sim_step(Sim& s, double dt) {
  FM_RANGE("fm_sim_step");
  DBuf<int> err(1);
  err.zero();
  state_to_step(s);
  launch_step(s, true, dt, err.p);
  int h = 0;
  err.download(&h, 1);
  FM_CUDA(cudaStreamSynchronize(stream()));
  if (h) throw Error(FM_ERR_DOMAIN, "hll_flux: negative depth");
  if (fv1_staged(s) && !s.fv1c) s.fv1_in_star = true;
  if (s.adaptive) s.since_adapt += 1;
}

// hydrograph_at (hydrograph.cpp:38-49) on the host for the API path.
static double hydro_host(const std::vector<double>& t, const std::vector<double>& q, double x) {
  if (x <= t.front()) return q.front();
  if (x >= t.back()) return q.back();
  const size_t hi = size_t(std::upper_bound(t.begin(), t.end(), x) - t.begin());
  const size_t lo = hi - 1;
  if (x == t[lo]) return q[lo];
  const double w = (x - t[lo]) / (t[hi] - t[lo]);
  return q[lo] + w * (q[hi] - q[lo]);
}

double sim_apply_inflows(Sim& s, double t, double dt) {
  state_to_u(s);
  double added = 0.0;
  double per[kMaxInflows] = {0};
  for (int f = 0; f < s.ninflow; ++f) {
    const double q = hydro_host(s.hy_t[f], s.hy_q[f], t);
    if (q <= 0.0) continue;
    const double vol = q * dt;
    per[f] = vol / double(s.region[f]);
    added += vol;
  }
  DBuf<double> dper;
  dper.upload(per, kMaxInflows);
  if (s.uniform)
    un_launch_inflow_add(s, dper.p);
  else
    nu_launch_inflow_add(s, dper.p);
  FM_CUDA(cudaStreamSynchronize(stream()));
  return added;
}

double sim_volume(Sim& s) {
  // Kahan in reference order (solver_nonuniform.cpp:467-477) over h.c0 and
  // the leaf levels, gathered into reference order on the device
  state_to_u(s);
  const int32_t* perm = sim_ref_perm(s);
  std::vector<double> h(s.n);
  std::vector<int32_t> l(s.n, 0);
  gather_col(perm, s.n, 9, 0, s.u.p, h.data());
  if (!s.uniform) gather_levels(perm, s.n, s.lvl.p, l.data());
  double sum = 0.0, comp = 0.0;
  for (int64_t c = 0; c < s.n; ++c) {
    const double sz = s.uniform ? s.R : s.R * double(1 << (s.L - l[c]));
    const double y = s.uniform ? h[c] * s.R * s.R - comp : h[c] * sz * sz - comp;
    const double t = sum + y;
    comp = (t - sum) - y;
    sum = t;
  }
  // a shard sums its own leaves; across NCCL ranks the partial sums add up
  // (an audit figure: not bit-identical to the unsharded Kahan order)
  return s.shard ? shard_allreduce_sum(s, sum) : sum;
}

bool sim_finite(Sim& s, double* bx, double* by) {
  state_to_u(s);
  DBuf<unsigned long long> bad(1);
  bad.fill_bytes(0xff);
  k_finite<<<nblk(s.n, 256), 256, 0, stream()>>>(s.n, s.uniform ? nullptr : s.lvl.p, s.li.p, s.lj.p, s.u.p, bad.p);
  FM_LAUNCHED();
  if (s.shard) shard_allreduce_u64_min(s, bad.p, 1);
  unsigned long long key = 0;
  bad.download(&key, 1);
  FM_CUDA(cudaStreamSynchronize(stream()));
  if (key == ~0ull) return true;
  key_xy(s, key, bx, by);
  return false;
}

void sim_sync_u(Sim& s) {
  state_to_u(s);
}

// Reference order: (level, j, i) for leaves (quadgrid.cpp:94-98), j*nx+i for
// rasters; permuted on the device (order.cu).
void sim_download(Sim& s, int32_t* lo, int32_t* io, int32_t* jo, double* u9, double* z3) {
  FM_RANGE("fm_sim_download");
  state_to_u(s);
  const int32_t* perm = sim_ref_perm(s);
  // U* is idle between steps (FV1's staged state was just moved back to U)
  StageScope lend(s.us.p, s.us.n * sizeof(double));
  if (lo) gather_levels(perm, s.n, s.lvl.p, lo);
  if (io) gather_i32(perm, s.n, s.li.p, io);
  if (jo) gather_i32(perm, s.n, s.lj.p, jo);
  if (u9) gather_rows(perm, s.n, 9, s.u.p, u9);
  if (z3) gather_rows(perm, s.n, 3, s.z.p, z3);
  FM_CUDA(cudaStreamSynchronize(stream()));
}

void sim_upload(Sim& s, const double* u9) {
  FM_RANGE("fm_sim_upload");
  state_to_u(s);
  scatter_rows(sim_ref_perm(s), s.n, 9, u9, s.u.p);
}

void sim_adapt(Sim& s, double t) {
  if (!s.adaptive) throw Error(FM_ERR_CONFIG, "adapt: not an adaptive simulation");
  state_to_u(s);
  adaptive_adapt(s, t);
  s.since_adapt = 0;
}

// The drive loop (run.cpp:80-111) on the device.  Static sims replay a CUDA
// graph of kBatch steps; each step's head kernel decides on the device
// whether to run (end time, step budget, events, blow-up), so surplus steps
// of the last batch are no-ops and the host syncs once per batch.
void sim_run(Sim& s, fm_clock* ck, int64_t max_steps, int stop_at_events, fm_run_result* out) {
  FM_RANGE("fm_sim_run");
  cudaStream_t st = stream();
  state_to_step(s);
  DevClock c0 = fresh_clock(ck, max_steps, stop_at_events);
  DevClock pair[2] = {c0, c0};
  s.clk.upload(pair, 2);
  init_red(s);
  launch_reduce_init(s);
  DBuf<int>& err = s.errflag;
  err.alloc(1);
  err.zero();
  EventPair ev;
  cudaEvent_t e0 = ev.a, e1 = ev.b;
  FM_CUDA(cudaEventRecord(e0, st));
  if (s.adaptive) {
    // adapt between steps on the host-driven path (device kernels, host
    // sequencing), ONE host sync per step: when an adapt is due, its
    // device-sized prefix is launched right behind the step, speculatively,
    // and the step's clock and the prefix's new leaf count come back together.
    // A prefix whose step turns out inactive (or the last one) is dropped: it
    // wrote only the grid's own buffers, which the next adapt rebuilds from
    // the sim's leaves, and the sim's state is untouched.
    Sim::HostSlots& hs = s.slots();
    for (int64_t k = 0; k < max_steps; ++k) {
      launch_step(s, false, 0.0, err.p);
      const bool due = s.since_adapt + 1 >= s.adapt_every;
      if (due) {
        state_to_u(s);
        adaptive_adapt_begin(s);
      }
      FM_CUDA(cudaMemcpyAsync(&hs.clk, s.clk.p + 1, sizeof(DevClock), cudaMemcpyDeviceToHost, st));
      FM_CUDA(cudaStreamSynchronize(st));
      s.settle_nseg();
      const DevClock c = hs.clk;
      if (!c.active || !c.had_step) {
        if (due) state_to_step(s);
        break;
      }
      s.since_adapt += 1;
      if (due && !(c.now >= c.end_time)) {
        adaptive_adapt_finish(s, c.now);
        state_to_step(s);
        s.since_adapt = 0;
        // the adapt changed the leaf set: refresh the step's reductions
        // (reset the slot on the device, no host round trip)
        k_red_reset<<<1, 1, 0, st>>>(s.red.p, int(c.steps & 1));
        FM_LAUNCHED();
        launch_reduce_init(s);
      } else if (due) {
        state_to_step(s);  // the last step: the speculative prefix is dropped
      }
    }
  } else if (shard_eager(s)) {
    // host transport: every exchange and reduction waits on the host, so the
    // steps are launched one by one (the per-step decision on the device
    // still turns surplus steps into no-ops)
    for (int64_t k = 0; k < max_steps; ++k) {
      launch_step(s, false, 0.0, err.p);
      if ((k & 31) == 31 && k + 1 < max_steps) {
        DevClock c;
        read_clock(s, c);
        FM_CUDA(cudaStreamSynchronize(st));
        if (!c.active) break;
      }
    }
  } else {
    // graphs of 32, 8 and 1 steps, captured on first use; the step count is
    // covered greedily so no graph replays surplus (no-op) steps
    static constexpr int kSizes[3] = {32, 8, 1};
    // graphs bake the state layout in (FV1: compact rows or the 72 B rows)
    const int layout = s.fv1c ? 1 : 0;
    if (layout != s.g_layout) {
      for (auto& gx : s.gexec) {
        if (gx) cudaGraphExecDestroy(gx);
        gx = nullptr;
      }
      s.g_layout = layout;
    }
    auto graph_of = [&](int q) {
      if (!s.gexec[q]) {
        const int64_t before = launches();
        cudaGraph_t gr;
        FM_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        for (int k = 0; k < kSizes[q]; ++k) launch_step(s, false, 0.0, err.p);
        FM_CUDA(cudaStreamEndCapture(st, &gr));
        FM_CUDA(cudaGraphInstantiate(&s.gexec[q], gr, 0));
        cudaGraphDestroy(gr);
        s.gkern[q] = launches() - before;  // kernels per replay
      }
      return s.gexec[q];
    };
    int64_t done = 0;
    while (done < max_steps) {
      const int64_t rem = max_steps - done;
      const int q = rem >= kSizes[0] ? 0 : rem >= kSizes[1] ? 1 : 2;
      FM_CUDA(cudaGraphLaunch(graph_of(q), st));
      count_graph_launches(s.gkern[q]);
      done += kSizes[q];
      if (q == 0 && done < max_steps) {
        DevClock c;
        read_clock(s, c);
        FM_CUDA(cudaStreamSynchronize(st));
        if (!c.active) break;
      }
    }
  }
  FM_CUDA(cudaEventRecord(e1, st));
  nu_launch_close(s);
  DevClock c;
  read_clock(s, c);
  int herr = 0;
  err.download(&herr, 1);
  FM_CUDA(cudaStreamSynchronize(st));
  s.settle_nseg();
  s.last_run_ms = elapsed_ms(e0, e1);
  if (herr) throw Error(FM_ERR_DOMAIN, "hll_flux: negative depth");
  ck->now = c.now;
  ck->next_output = c.next_out;
  ck->next_gauge = c.next_gauge;
  fm_run_result r{};
  r.steps = c.steps;
  r.dt_min = c.dt_min;
  r.dt_max = c.dt_max;
  r.volume_inflow = c.vol_in;
  r.blew_up = c.blew_up;
  r.blow_up_time = c.blow_t;
  r.finished = c.now >= c.end_time;
  r.event_due = c.event_due;
  if (c.blew_up) key_xy(s, c.bad_key, &r.bad_x, &r.bad_y);
  if (out) *out = r;
  if (c.blew_up) throw Error(FM_ERR_BLOWUP, "solver state is non-finite");
}

// The drive loop over a local group of shards (all ranks of a partition in
// this process, on this device): the same step operations as the NCCL path,
// interleaved across the shards phase by phase, with the halo exchanges done
// as device copies between the shards' buffers and the reduction slots
// min-combined.  No graph: this is the single-GPU check of the sharding logic.
void group_run(const std::vector<Sim*>& sims, fm_clock* ck, int64_t max_steps, int stop_at_events,
               fm_run_result* out) {
  cudaStream_t st = stream();
  if (sims.empty()) throw Error(FM_ERR_CONFIG, "group: no shards");
  for (Sim* s : sims)
    if (!s || !s->shard || int(sims.size()) != s->shard->nranks)
      throw Error(FM_ERR_CONFIG, "group: every rank of one local communicator is needed, in rank order");
  for (size_t r = 0; r < sims.size(); ++r)
    if (sims[r]->shard->rank != int(r) || sims[r]->shard->comm != sims[0]->shard->comm)
      throw Error(FM_ERR_CONFIG, "group: shards must be given in rank order and share a communicator");
  const DevClock c0 = fresh_clock(ck, max_steps, stop_at_events);
  for (Sim* s : sims) {
    state_to_step(*s);
    DevClock pair[2] = {c0, c0};
    s->clk.upload(pair, 2);
    init_red(*s);
    if (s->uniform)
      un_launch_reduce_init(*s);
    else
      nu_launch_reduce_init(*s);
    s->errflag.alloc(1);
    s->errflag.zero();
  }
  shard_local_reduce(sims);
  EventPair ev;
  cudaEvent_t e0 = ev.a, e1 = ev.b;
  FM_CUDA(cudaEventRecord(e0, st));
  const std::vector<int> ops = nu_step_ops(*sims[0], false);
  for (int64_t k = 0; k < max_steps; ++k) {
    for (int op : ops) {
      if (op == OP_EXCH_U || op == OP_EXCH_US) {
        for (Sim* s : sims) {
          int w = 9;
          const double* a = exch_array(*s, op, &w);
          shard_pack(*s, a, w);
        }
        for (Sim* s : sims) {
          int w = 9;
          double* a = exch_array(*s, op, &w);
          shard_local_recv(*s, a, w);
        }
      } else if (op == OP_REDUCE) {
        shard_local_reduce(sims);
      } else {
        for (Sim* s : sims) step_op(*s, op, false, 0.0, s->errflag.p);
      }
    }
    DevClock c;
    read_clock(*sims[0], c);
    FM_CUDA(cudaStreamSynchronize(st));
    if (!c.active) break;
  }
  FM_CUDA(cudaEventRecord(e1, st));
  int herr = 0;
  for (Sim* s : sims) {
    nu_launch_close(*s);
    int h = 0;
    s->errflag.download(&h, 1);
    FM_CUDA(cudaStreamSynchronize(st));
    herr |= h;
  }
  DevClock c;
  read_clock(*sims[0], c);
  FM_CUDA(cudaStreamSynchronize(st));
  for (Sim* s : sims) s->last_run_ms = elapsed_ms(e0, e1);
  if (herr) throw Error(FM_ERR_DOMAIN, "hll_flux: negative depth");
  ck->now = c.now;
  ck->next_output = c.next_out;
  ck->next_gauge = c.next_gauge;
  fm_run_result r{};
  r.steps = c.steps;
  r.dt_min = c.dt_min;
  r.dt_max = c.dt_max;
  r.volume_inflow = c.vol_in;
  r.blew_up = c.blew_up;
  r.blow_up_time = c.blow_t;
  r.finished = c.now >= c.end_time;
  r.event_due = c.event_due;
  if (c.blew_up) key_xy(*sims[0], c.bad_key, &r.bad_x, &r.bad_y);
  if (out) *out = r;
  if (c.blew_up) throw Error(FM_ERR_BLOWUP, "solver state is non-finite");
}

}  // namespace fmh

namespace fmh {

// Per-kernel timing of `steps` device-loop steps launched without a graph.
void sim_profile(Sim& s, int64_t steps, double* ms, int64_t* counts, int cap, int* nfam) {
  cudaStream_t st = stream();
  state_to_step(s);
  fm_clock ck{1e12, 0.0, 10.0, 0.0, 1, 1};
  DevClock c0 = fresh_clock(&ck, steps, 0);
  DevClock pair[2] = {c0, c0};
  s.clk.upload(pair, 2);
  init_red(s);
  launch_reduce_init(s);
  s.errflag.alloc(1);
  s.errflag.zero();
  KTimer& t = ktimer();
  t = KTimer{};
  t.on = true;
  try {
    for (int64_t k = 0; k < steps; ++k) launch_step(s, false, 0.0, s.errflag.p);
  } catch (...) {
    t.on = false;
    throw;
  }
  t.on = false;
  FM_CUDA(cudaStreamSynchronize(st));
  std::vector<double> acc(KF_COUNT, 0.0);
  std::vector<int64_t> cnt(KF_COUNT, 0);
  for (size_t q = 0; q < t.fam.size(); ++q) {
    acc[t.fam[q]] += elapsed_ms(t.a[q], t.b[q]);
    cnt[t.fam[q]] += 1;
    cudaEventDestroy(t.a[q]);
    cudaEventDestroy(t.b[q]);
  }
  t = KTimer{};
  for (int f = 0; f < std::min(cap, int(KF_COUNT)); ++f) {
    if (ms) ms[f] = acc[f];
    if (counts) counts[f] = cnt[f];
  }
  *nfam = KF_COUNT;
  nu_launch_close(s);
  FM_CUDA(cudaStreamSynchronize(st));
}

}  // namespace fmh

namespace fmh {

// ---- binary checkpoint ("a binary state dump: leaf keys + 9
// doubles + 3 topo doubles"), the restart path the reference lacks -------
namespace {
struct CkptHeader {
  char magic[8];  // "FMCKPT1"
  int32_t solver, scheme, uniform, L, M, N, nx, ny;
  double R, x0, y0;
  int64_t n, nseg, n_accq, n_accqb, n_aqx, n_aqy;
};
void write_all(FILE* f, const void* p, size_t bytes) {
  if (bytes && std::fwrite(p, 1, bytes, f) != bytes) throw Error(FM_ERR_IO, "checkpoint: write failed");
}
void read_all(FILE* f, void* p, size_t bytes) {
  if (bytes && std::fread(p, 1, bytes, f) != bytes) throw Error(FM_ERR_IO, "checkpoint: truncated file");
}
template <typename T>
std::vector<T> dev_to_host(const DBuf<T>& b, size_t n) {
  std::vector<T> v(n);
  if (n) FM_CUDA(cudaMemcpyAsync(v.data(), b.p, n * sizeof(T), cudaMemcpyDeviceToHost, stream()));
  return v;
}
}  // namespace

// The leaf keys (level, i, j in the reference order), the flow state (9 per
// leaf) and topography (3 per leaf), and ACC's face discharges (device
// order, with the leaf set they belong to).
void sim_checkpoint(Sim& s, const char* path) {
  if (s.shard) throw Error(FM_ERR_CONFIG, "checkpoint: a shard checkpoints through its own rank");
  state_to_u(s);
  const int64_t n = s.n;
  std::vector<int32_t> l(n), i(n), j(n);
  std::vector<double> u(9 * size_t(n)), z(3 * size_t(n));
  sim_download(s, l.data(), i.data(), j.data(), u.data(), z.data());
  CkptHeader h{};
  std::memcpy(h.magic, "FMCKPT1", 8);
  h.solver = s.solver, h.scheme = s.scheme, h.uniform = s.uniform ? 1 : 0;
  h.L = s.L, h.M = s.M, h.N = s.N, h.nx = s.nx, h.ny = s.ny;
  h.R = s.R, h.x0 = s.x0, h.y0 = s.y0;
  h.n = n, h.nseg = s.nseg;
  const bool acc = s.scheme == FM_ACC;
  h.n_accq = acc && !s.uniform ? int64_t(s.accq.n) : 0;
  h.n_accqb = acc && !s.uniform ? int64_t(s.accqb.n) : 0;
  h.n_aqx = acc && s.uniform ? int64_t(s.aqx.n) : 0;
  h.n_aqy = acc && s.uniform ? int64_t(s.aqy.n) : 0;
  const auto q = dev_to_host(s.accq, size_t(h.n_accq)), qb = dev_to_host(s.accqb, size_t(h.n_accqb));
  const auto ax = dev_to_host(s.aqx, size_t(h.n_aqx)), ay = dev_to_host(s.aqy, size_t(h.n_aqy));
  FM_CUDA(cudaStreamSynchronize(stream()));
  FILE* f = std::fopen(path, "wb");
  if (!f) throw Error(FM_ERR_IO, std::string("checkpoint: cannot open ") + path);
  try {
    write_all(f, &h, sizeof(h));
    write_all(f, l.data(), 4 * size_t(n));
    write_all(f, i.data(), 4 * size_t(n));
    write_all(f, j.data(), 4 * size_t(n));
    write_all(f, u.data(), 8 * u.size());
    write_all(f, z.data(), 8 * z.size());
    write_all(f, q.data(), 8 * q.size());
    write_all(f, qb.data(), 8 * qb.size());
    write_all(f, ax.data(), 8 * ax.size());
    write_all(f, ay.data(), 8 * ay.size());
  } catch (...) {
    std::fclose(f);
    throw;
  }
  if (std::fclose(f) != 0) throw Error(FM_ERR_IO, "checkpoint: close failed");
}

// Restores a checkpoint onto a sim of the same scenario and leaf set (the
// keys and topography must match bit for bit; otherwise FM_ERR_CONFIG).
void sim_resume(Sim& s, const char* path) {
  if (s.shard) throw Error(FM_ERR_CONFIG, "resume: a shard resumes through its own rank");
  FILE* f = std::fopen(path, "rb");
  if (!f) throw Error(FM_ERR_IO, std::string("resume: cannot open ") + path);
  std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
  CkptHeader h{};
  read_all(f, &h, sizeof(h));
  if (std::memcmp(h.magic, "FMCKPT1", 8) != 0) throw Error(FM_ERR_IO, "resume: not a floodmra-b200 checkpoint");
  if (h.solver != s.solver || h.uniform != (s.uniform ? 1 : 0) || h.L != s.L || h.M != s.M || h.N != s.N ||
      h.nx != s.nx || h.ny != s.ny || h.R != s.R || h.x0 != s.x0 || h.y0 != s.y0 || h.n != s.n)
    throw Error(FM_ERR_CONFIG, "resume: the checkpoint belongs to another scenario or leaf set");
  const int64_t n = h.n;
  std::vector<int32_t> l(n), i(n), j(n), l0(n), i0(n), j0(n);
  std::vector<double> u(9 * size_t(n)), z(3 * size_t(n)), z0(3 * size_t(n));
  read_all(f, l.data(), 4 * size_t(n));
  read_all(f, i.data(), 4 * size_t(n));
  read_all(f, j.data(), 4 * size_t(n));
  read_all(f, u.data(), 8 * u.size());
  read_all(f, z.data(), 8 * z.size());
  std::vector<double> q(size_t(h.n_accq)), qb(size_t(h.n_accqb)), ax(size_t(h.n_aqx)), ay(size_t(h.n_aqy));
  read_all(f, q.data(), 8 * q.size());
  read_all(f, qb.data(), 8 * qb.size());
  read_all(f, ax.data(), 8 * ax.size());
  read_all(f, ay.data(), 8 * ay.size());
  state_to_u(s);
  sim_download(s, l0.data(), i0.data(), j0.data(), nullptr, z0.data());
  if (l != l0 || i != i0 || j != j0 || std::memcmp(z.data(), z0.data(), 8 * z.size()) != 0)
    throw Error(FM_ERR_CONFIG, "resume: the leaf set or topography differs from the checkpoint's");
  if (size_t(h.n_accq) != (s.scheme == FM_ACC && !s.uniform ? s.accq.n : 0) ||
      size_t(h.n_accqb) != (s.scheme == FM_ACC && !s.uniform ? s.accqb.n : 0) ||
      size_t(h.n_aqx) != (s.scheme == FM_ACC && s.uniform ? s.aqx.n : 0) ||
      size_t(h.n_aqy) != (s.scheme == FM_ACC && s.uniform ? s.aqy.n : 0))
    throw Error(FM_ERR_CONFIG, "resume: ACC discharge arrays differ in size");
  sim_upload(s, u.data());
  if (!q.empty()) FM_CUDA(cudaMemcpyAsync(s.accq.p, q.data(), 8 * q.size(), cudaMemcpyHostToDevice, stream()));
  if (!qb.empty()) FM_CUDA(cudaMemcpyAsync(s.accqb.p, qb.data(), 8 * qb.size(), cudaMemcpyHostToDevice, stream()));
  if (!ax.empty()) FM_CUDA(cudaMemcpyAsync(s.aqx.p, ax.data(), 8 * ax.size(), cudaMemcpyHostToDevice, stream()));
  if (!ay.empty()) FM_CUDA(cudaMemcpyAsync(s.aqy.p, ay.data(), 8 * ay.size(), cudaMemcpyHostToDevice, stream()));
  FM_CUDA(cudaStreamSynchronize(stream()));
}

void sim_snapshot(Sim& s) {
  acc_to_u(s);  // the snapshot holds U (the compact states folded back)
  fv1c_to_u(s);
  auto copy = [](DBuf<double>& dst, const DBuf<double>& src) {
    dst.alloc(src.n);
    if (src.n)
      FM_CUDA(cudaMemcpyAsync(dst.p, src.p, src.n * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
  };
  copy(s.snap_u, s.u);
  copy(s.snap_us, s.us);
  copy(s.snap_q, s.accq);
  copy(s.snap_qb, s.accqb);
  copy(s.snap_aqx, s.aqx);
  copy(s.snap_aqy, s.aqy);
  s.snap_n = s.n;
  s.snap_gen = s.leaf_gen;
  s.snap_fv1 = s.fv1_in_star;
  FM_CUDA(cudaStreamSynchronize(stream()));
}

void sim_restore(Sim& s) {
  if (s.snap_n != s.n || s.snap_u.n != s.u.n || s.snap_gen != s.leaf_gen)
    throw Error(FM_ERR_CONFIG, "restore: no snapshot of the current leaf set");
  auto copy = [](DBuf<double>& dst, const DBuf<double>& src) {
    if (src.n)
      FM_CUDA(cudaMemcpyAsync(dst.p, src.p, src.n * sizeof(double), cudaMemcpyDeviceToDevice, stream()));
  };
  copy(s.u, s.snap_u);
  copy(s.us, s.snap_us);
  copy(s.accq, s.snap_q);
  copy(s.accqb, s.snap_qb);
  copy(s.aqx, s.snap_aqx);
  copy(s.aqy, s.snap_aqy);
  s.fv1_in_star = s.snap_fv1;
  s.acc_soa = false;  // U is the state again
  s.fv1c = false;
  FM_CUDA(cudaStreamSynchronize(stream()));
}

}  // namespace fmh
