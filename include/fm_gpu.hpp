// fm_gpu.hpp — header-only C++ host side over the C ABI (fm_gpu.h).
//
// Drop-in classes for the reference's duck-typed drive<Sim> loop
// (/root/reference/proj/core/src/run.cpp:35-141): each exposes the members
// drive<Sim> calls — compute_dt, step(dt, threads), apply_inflows(t, dt),
// volume, finite_state(&x, &y) and, for the adaptive solvers, adapt(t),
// steps_since_adapt, adapt_every and element_log — and raises the reference's
// exception types (errors.hpp:9-37) from the ABI's status codes.
//
// Three drive<Sim>-shaped classes mirror the reference's solver types member
// for member: UniformSim (solver_uniform.hpp:15-67), NonUniformSim (with the
// `grid` / `z` members, solver_nonuniform.hpp:18-84) and AdaptiveSim (with
// `adapt`, `steps_since_adapt`, `adapt_every`, the `element_log` data member
// and `sim.grid` / `sim.z`, solver_adaptive.hpp:16-63), so every
// `if constexpr (requires { ... })` branch of drive<Sim> (run.cpp:70-73,
// 90-95, 122-135) takes the same path as for the reference sim.  The generic
// `Sim` handle (runtime-dispatched) serves loops written without templates.
//
// Define FM_GPU_WITH_FLOODMRA before including this header (with the
// reference's include path, linking the reference library) to throw
// floodmra::ConfigError & co., to use floodmra::Raster / GaugeValue /
// QuadGrid / PlanarCoeffs as the member types, to get
// fm_gpu::view(const floodmra::Raster&) (raster.hpp:10-32), and to construct
// the sims straight from a floodmra::ScenarioConfig (run.cpp:145-164).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fm_gpu.h"

#ifdef FM_GPU_WITH_FLOODMRA
#include "floodmra/config.hpp"
#include "floodmra/errors.hpp"
#include "floodmra/field.hpp"
#include "floodmra/hydrograph.hpp"
#include "floodmra/quadgrid.hpp"
#include "floodmra/raster.hpp"
#include "floodmra/sim_common.hpp"
#endif

namespace fm_gpu {

#ifdef FM_GPU_WITH_FLOODMRA
using ConfigError = floodmra::ConfigError;
using IoError = floodmra::IoError;
using StructureError = floodmra::StructureError;
using DomainError = floodmra::DomainError;
using BlowUpError = floodmra::BlowUpError;
#else
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StructureError : std::logic_error {
  using std::logic_error::logic_error;
};
struct DomainError : std::domain_error {
  using std::domain_error::domain_error;
};
struct BlowUpError : std::runtime_error {
  BlowUpError(const std::string& w, double t_fail) : std::runtime_error(w), t(t_fail) {}
  double t;
};
#endif

#ifdef FM_GPU_WITH_FLOODMRA
// A host view of a reference raster (no copy; the raster must outlive the call).
inline fm_raster view(const floodmra::Raster& r) {
  return fm_raster{r.values.data(), r.ncols, r.nrows, r.xll, r.yll, r.cellsize, r.nodata, 0};
}
#endif

// Status -> reference exception (tools/floodmra.cpp:171-186 exit-code classes).
inline void check(int st, double t_fail = 0.0) {
  if (st == FM_OK) return;
  const std::string msg = fm_last_error();
  switch (st) {
    case FM_ERR_CONFIG: throw ConfigError(msg);
    case FM_ERR_IO: throw IoError(msg);
    case FM_ERR_STRUCTURE: throw StructureError(msg);
    case FM_ERR_DOMAIN: throw DomainError(msg);
    case FM_ERR_BLOWUP: throw BlowUpError(msg, t_fail);
    default: throw std::runtime_error(msg);
  }
}

// generate_static_grid's result (NonUniformGrid) resident on the device.
class Grid {
 public:
  Grid(const fm_raster& dem, int L, double eps, bool graded = true, int kind = FM_MW) {
    check(fm_mra_static(&dem, L, eps, graded ? 1 : 0, kind, &g_));
  }
  Grid(const Grid&) = delete;
  Grid& operator=(const Grid&) = delete;
  Grid(Grid&& o) noexcept : g_(std::exchange(o.g_, nullptr)) {}
  ~Grid() {
    if (g_) fm_grid_destroy(g_);
  }
  // read_nug's construction (quadgrid.cpp:310-327): a grid from a leaf list
  static Grid import(int L, int M, int N, double Rfine, double x0, double y0,
                     const std::vector<int32_t>& l, const std::vector<int32_t>& i,
                     const std::vector<int32_t>& j, const std::vector<double>& topo3) {
    fm_grid* g = nullptr;
    check(fm_grid_import(L, M, N, Rfine, x0, y0, int64_t(l.size()), l.data(), i.data(), j.data(),
                         topo3.data(), &g));
    return Grid(g);
  }
  // read_nug (quadgrid.cpp:304-327), or the binary side format by its magic
  static Grid read(const std::string& path) {
    fm_grid* g = nullptr;
    check(fm_grid_read(path.c_str(), &g));
    return Grid(g);
  }
  // write_nug (quadgrid.cpp:287-302), byte for byte; binary: the raw side format
  void write(const std::string& path, bool binary = false) const {
    check(fm_grid_write(g_, path.c_str(), binary ? 1 : 0));
  }
  int64_t size() const { return fm_grid_num_leaves(g_); }
  const fm_grid* get() const { return g_; }
  // leaves in the reference order (level, j, i) and their topography
  void leaves(std::vector<int32_t>& l, std::vector<int32_t>& i, std::vector<int32_t>& j,
              std::vector<double>& topo3) const {
    const int64_t n = size();
    l.resize(n);
    i.resize(n);
    j.resize(n);
    topo3.resize(3 * n);
    check(fm_grid_leaves(g_, FM_ORDER_REFERENCE, l.data(), i.data(), j.data(), topo3.data()));
  }

 private:
  explicit Grid(fm_grid* g) : g_(g) {}
  fm_grid* g_ = nullptr;
};

// read_ascii_grid (raster.cpp:22-79) into library-owned host memory
// (page-locked when a device is present); also reads the binary side format.
class HostRaster {
 public:
  explicit HostRaster(const std::string& path) { check(fm_raster_read(path.c_str(), &r_)); }
  HostRaster(const HostRaster&) = delete;
  HostRaster& operator=(const HostRaster&) = delete;
  HostRaster(HostRaster&& o) noexcept : r_(std::exchange(o.r_, fm_raster{})) {}
  ~HostRaster() { fm_raster_release(&r_); }
  const fm_raster& get() const { return r_; }
  double at(int row, int col) const { return r_.values[size_t(row) * size_t(r_.ncols) + size_t(col)]; }

 private:
  fm_raster r_{};
};
// write_ascii_grid (raster.cpp:81-96), byte for byte; binary: the raw side format
inline void write_raster(const fm_raster& r, const std::string& path, bool binary = false) {
  check(fm_raster_write(&r, path.c_str(), binary ? 1 : 0));
}

// ---- member types of the drive<Sim> contract --------------------------------
#ifdef FM_GPU_WITH_FLOODMRA
using GaugeValue = floodmra::GaugeValue;  // sim_common.hpp:47-49
using Raster = floodmra::Raster;          // raster.hpp:10-32
#else
struct GaugeValue {
  double h = 0.0, eta = 0.0, u = 0.0, v = 0.0;
};
struct Raster {
  int ncols = 0, nrows = 0;
  double xll = 0.0, yll = 0.0, cellsize = 1.0, nodata = -9999.0;
  std::vector<double> values;  // row 0 north
};
#endif

// A leaf set in the reference's (level, j, i) order with its geometry
// (QuadGrid, quadgrid.hpp:54-60) and per-leaf topography planes.
struct LeafSet {
  int L = 0, M = 1, N = 1;
  double Rfine = 1.0, x0 = 0.0, y0 = 0.0;
  std::vector<int32_t> level, i, j;
  std::vector<double> topo3;  // 3 per leaf: c0 c1x c1y
};

#ifdef FM_GPU_WITH_FLOODMRA
inline floodmra::QuadGrid to_quadgrid(const LeafSet& s) {
  std::vector<floodmra::LeafId> ids(s.level.size());
  for (size_t k = 0; k < ids.size(); ++k) ids[k] = floodmra::LeafId{s.level[k], s.i[k], s.j[k]};
  return floodmra::make_quadgrid(s.L, s.M, s.N, s.Rfine, s.x0, s.y0, std::move(ids));
}
inline std::vector<floodmra::PlanarCoeffs> to_planes(const LeafSet& s) {
  std::vector<floodmra::PlanarCoeffs> z(s.level.size());
  for (size_t k = 0; k < z.size(); ++k) z[k] = {s.topo3[3 * k], s.topo3[3 * k + 1], s.topo3[3 * k + 2]};
  return z;
}
#endif

// The members every solver type shares (drive<Sim>, run.cpp:35-141).
class SimBase {
 public:
  SimBase(const SimBase&) = delete;
  SimBase& operator=(const SimBase&) = delete;
  SimBase(SimBase&& o) noexcept : s_(std::exchange(o.s_, nullptr)) {}
  ~SimBase() {
    if (s_) fm_sim_destroy(s_);
  }

  double compute_dt() const {
    double dt = 0.0;
    check(fm_sim_compute_dt(s_, &dt));
    return dt;
  }
  void step(double dt, int /*threads*/ = 1) { check(fm_sim_step(s_, dt)); }
  double apply_inflows(double t, double dt) {
    double added = 0.0;
    check(fm_sim_apply_inflows(s_, t, dt, &added));
    return added;
  }
  double volume() const {
    double v = 0.0;
    check(fm_sim_volume(s_, &v));
    return v;
  }
  bool finite_state(double* bad_x = nullptr, double* bad_y = nullptr) const {
    int32_t ok = 1;
    double x = 0, y = 0;
    check(fm_sim_finite(s_, &ok, &x, &y));
    if (!ok) {
      if (bad_x) *bad_x = x;
      if (bad_y) *bad_y = y;
    }
    return ok != 0;
  }
  // sample_gauge (solver_nonuniform.cpp:489-506, solver_uniform.cpp:480-498)
  GaugeValue sample_gauge(double x, double y) const {
    double v[4];
    check(fm_sim_sample_gauges(s_, 1, &x, &y, v));
    GaugeValue g;
    g.h = v[0], g.eta = v[1], g.u = v[2], g.v = v[3];
    return g;
  }
  // depth_raster / qx_raster / qy_raster (solver_nonuniform.cpp:508-519,
  // solver_uniform.cpp:501-520): the fine-grid sample, row 0 north
  Raster raster(int which) const {
    Raster r;
    int32_t nc = 0, nr = 0;
    check(fm_sim_raster_shape(s_, &nc, &nr, &r.xll, &r.yll, &r.cellsize, &r.nodata));
    r.ncols = nc, r.nrows = nr;
    r.values.resize(size_t(nc) * size_t(nr));
    check(fm_sim_raster(s_, which, r.values.data(), 0));
    return r;
  }
  Raster depth_raster() const { return raster(0); }
  Raster qx_raster() const { return raster(1); }
  Raster qy_raster() const { return raster(2); }

  // The current leaf set (reference order) and its topography.
  LeafSet leaves() const {
    LeafSet o;
    int32_t L = 0, M = 1, N = 1;
    check(fm_sim_geometry(s_, &L, &M, &N, &o.Rfine, &o.x0, &o.y0));
    o.L = L, o.M = M, o.N = N;
    const int64_t n = cells();
    o.level.resize(n), o.i.resize(n), o.j.resize(n), o.topo3.resize(3 * n);
    check(fm_sim_download(s_, o.level.data(), o.i.data(), o.j.data(), nullptr, o.topo3.data()));
    return o;
  }

  // ---- device-resident loop and state access --------------------------------
  // The drive<Sim> loop body on the device for up to `max_steps` steps; clock
  // semantics of EventClock (sim_common.cpp:48-82).  Throws BlowUpError(t).
  fm_run_result run(fm_clock& clk, int64_t max_steps, bool stop_at_events = true) {
    fm_run_result r{};
    // the status first: r.blow_up_time is only filled by the call
    const int st = fm_sim_run(s_, &clk, max_steps, stop_at_events ? 1 : 0, &r);
    check(st, r.blow_up_time);
    return r;
  }
  int64_t cells() const { return fm_sim_num_cells(s_); }
  // u: 9 doubles per cell [h qx qy] x [c0 c1x c1y]; z: 3 per cell; reference order
  void download(std::vector<double>& u9, std::vector<double>* z3 = nullptr) const {
    const int64_t n = cells();
    u9.resize(9 * n);
    if (z3) z3->resize(3 * n);
    check(fm_sim_download(s_, nullptr, nullptr, nullptr, u9.data(), z3 ? z3->data() : nullptr));
  }
  void upload(const std::vector<double>& u9) { check(fm_sim_upload(s_, u9.data())); }
  fm_sim* get() const { return s_; }

 protected:
  SimBase(const fm_sim_desc& d, const fm_raster& dem, const fm_grid* grid) {
    check(fm_sim_create(&d, &dem, grid, &s_));
  }
  fm_sim* s_ = nullptr;
};

#ifdef FM_GPU_WITH_FLOODMRA
// ScenarioConfig (config.hpp:29-69) -> fm_sim_desc, owning the host inputs the
// descriptor points at: the Manning and initial-depth rasters
// (make_*_sim read them with read_ascii_grid) and the hydrographs
// (read_hydrograph_csv).
struct SimInputs {
  fm_sim_desc d{};
  floodmra::Raster manning, h0;
  fm_raster manning_v{}, h0_v{};
  std::vector<std::vector<double>> ts, qs;
  std::vector<fm_inflow> inflows;

  explicit SimInputs(const floodmra::ScenarioConfig& cfg, int libm = FM_LIBM_NATIVE) {
    d.solver = int32_t(cfg.solver);
    d.g = cfg.g;
    d.h_dry = cfg.h_dry;
    d.courant = cfg.courant;  // 0: per-solver default, as courant_for (config.cpp:37-47)
    for (int k = 0; k < 4; ++k)
      d.bc[k] = cfg.boundary[k] == floodmra::BoundaryKind::open ? FM_OPEN : FM_REFLECTIVE;
    d.manning = cfg.manning;
    if (!cfg.manning_raster.empty()) {
      manning = floodmra::read_ascii_grid(cfg.manning_raster);
      manning_v = view(manning);
      d.manning_raster = &manning_v;
    }
    if (!cfg.initial_depth_raster.empty()) {
      h0 = floodmra::read_ascii_grid(cfg.initial_depth_raster);
      h0_v = view(h0);
      d.initial_depth_raster = &h0_v;
    }
    d.has_initial_surface = cfg.initial_surface.has_value() ? 1 : 0;
    d.initial_surface = cfg.initial_surface.value_or(0.0);
    d.initial_depth = cfg.initial_depth;
    for (const floodmra::InflowSpec& f : cfg.inflows) {
      const floodmra::Hydrograph h = floodmra::read_hydrograph_csv(f.hydrograph_path);
      std::vector<double> t, q;
      for (const auto& smp : h.samples) t.push_back(smp.t), q.push_back(smp.q);
      ts.push_back(std::move(t));
      qs.push_back(std::move(q));
    }
    for (size_t k = 0; k < cfg.inflows.size(); ++k) {
      const floodmra::InflowSpec& f = cfg.inflows[k];
      inflows.push_back(fm_inflow{ts[k].data(), qs[k].data(), int32_t(ts[k].size()), f.i0, f.j0, f.i1, f.j1});
    }
    d.inflows = inflows.data();
    d.n_inflows = int32_t(inflows.size());
    d.epsilon = cfg.epsilon;
    d.max_level = cfg.max_level;
    d.adapt_every = cfg.adapt_every < 1 ? 1 : cfg.adapt_every;
    d.libm = libm;
  }
  SimInputs(const SimInputs&) = delete;
  SimInputs& operator=(const SimInputs&) = delete;
};
#endif

// UniformSim (solver_uniform.hpp:15-67): the raster solver at one level.
class UniformSim : public SimBase {
 public:
  UniformSim(const fm_sim_desc& d, const fm_raster& dem) : SimBase(d, dem, nullptr) {}
#ifdef FM_GPU_WITH_FLOODMRA
  // make_uniform_sim (solver_uniform.cpp:522)
  UniformSim(const floodmra::ScenarioConfig& cfg, const floodmra::Raster& dem)
      : UniformSim(SimInputs(cfg).d, view(dem)) {}
#endif
};

// NonUniformSim (solver_nonuniform.hpp:18-84) on a static grid.  `grid` and
// `z` are the reference's public members (read by drive's stats,
// run.cpp:128-132); the grid never changes, so they are filled once.
class NonUniformSim : public SimBase {
 public:
  NonUniformSim(const fm_sim_desc& d, const fm_raster& dem, const Grid& g) : SimBase(d, dem, g.get()) {
    fill();
  }
#ifdef FM_GPU_WITH_FLOODMRA
  // run_scenario's static branch (run.cpp:150-158): the grid from cfg.grid_file
  // (read_nug -> fm_grid_import) or generate_static_grid(dem, eps, L, graded,
  // MW) on the device, then make_nonuniform_sim
  NonUniformSim(const floodmra::ScenarioConfig& cfg, const floodmra::Raster& dem)
      : NonUniformSim(SimInputs(cfg).d, view(dem), make_grid(cfg, dem)) {}
  floodmra::QuadGrid grid;
  std::vector<floodmra::PlanarCoeffs> z;
#else
  LeafSet grid;  // leaves and topography (z) together
#endif

 private:
  void fill() {
#ifdef FM_GPU_WITH_FLOODMRA
    const LeafSet s = leaves();
    grid = to_quadgrid(s);
    z = to_planes(s);
#else
    grid = leaves();
#endif
  }
#ifdef FM_GPU_WITH_FLOODMRA
  static Grid make_grid(const floodmra::ScenarioConfig& cfg, const floodmra::Raster& dem) {
    if (!cfg.grid_file.empty()) {
      const floodmra::NonUniformGrid nug = floodmra::read_nug(cfg.grid_file);
      const floodmra::QuadGrid& q = nug.grid;
      const size_t n = q.leaves.size();
      std::vector<int32_t> l(n), i(n), j(n);
      std::vector<double> t(3 * n);
      for (size_t k = 0; k < n; ++k) {
        l[k] = q.leaves[k].level, i[k] = q.leaves[k].i, j[k] = q.leaves[k].j;
        t[3 * k] = nug.topo[k].c0, t[3 * k + 1] = nug.topo[k].c1x, t[3 * k + 2] = nug.topo[k].c1y;
      }
      return Grid::import(q.L, q.M, q.N, q.Rfine, q.x0, q.y0, l, i, j, t);
    }
    return Grid(view(dem), cfg.max_level, cfg.epsilon, true, FM_MW);
  }
#endif
};

// AdaptiveSim (solver_adaptive.hpp:16-63): MWDG2 / HWFV1 re-gridded on the
// device every `adapt_every` steps.  `element_log` is a data member, as in the
// reference, refreshed from the device after every adapt; `sim.grid` /
// `sim.z` convert to the current leaf set on access (drive's .nug dump and
// stats, run.cpp:70-73, 128-130).
class AdaptiveSim : public SimBase {
 public:
  struct GridRef {
    const SimBase* owner;
#ifdef FM_GPU_WITH_FLOODMRA
    operator floodmra::QuadGrid() const { return to_quadgrid(owner->leaves()); }
#endif
    LeafSet get() const { return owner->leaves(); }
  };
  struct TopoRef {
    const SimBase* owner;
#ifdef FM_GPU_WITH_FLOODMRA
    operator std::vector<floodmra::PlanarCoeffs>() const { return to_planes(owner->leaves()); }
#endif
    std::vector<double> get() const { return owner->leaves().topo3; }
  };
  struct Inner {
    GridRef grid;
    TopoRef z;
  };

  AdaptiveSim(const fm_sim_desc& d, const fm_raster& dem)
      : SimBase(d, dem, nullptr), adapt_every(d.adapt_every < 1 ? 1 : d.adapt_every), sim{{this}, {this}} {
    sync_log();
  }
#ifdef FM_GPU_WITH_FLOODMRA
  // make_adaptive_sim (solver_adaptive.cpp:209-236), adapt(0) included
  AdaptiveSim(const floodmra::ScenarioConfig& cfg, const floodmra::Raster& dem)
      : AdaptiveSim(SimInputs(cfg).d, view(dem)) {}
#endif
  AdaptiveSim(AdaptiveSim&& o) noexcept
      : SimBase(std::move(o)), adapt_every(o.adapt_every), steps_since_adapt(o.steps_since_adapt),
        element_log(std::move(o.element_log)), sim{{this}, {this}} {}

  void step(double dt, int threads = 1) {
    SimBase::step(dt, threads);
    ++steps_since_adapt;
  }
  void adapt(double t) {
    check(fm_sim_adapt(s_, t));
    sync_log();
  }
  fm_run_result run(fm_clock& clk, int64_t max_steps, bool stop_at_events = true) {
    const fm_run_result r = SimBase::run(clk, max_steps, stop_at_events);
    sync_log();
    return r;
  }

  int adapt_every = 1;
  int64_t steps_since_adapt = 0;
  std::vector<std::pair<double, int64_t>> element_log;  // (t, leaf count), solver_adaptive.hpp:23
  Inner sim;

 private:
  void sync_log() {  // append the entries the device side added since the last sync
    const int64_t n = fm_sim_element_log(s_, nullptr, nullptr, 0);
    if (n <= int64_t(element_log.size())) return;
    std::vector<double> t(n);
    std::vector<int64_t> c(n);
    fm_sim_element_log(s_, t.data(), c.data(), n);
    for (int64_t k = int64_t(element_log.size()); k < n; ++k) element_log.emplace_back(t[k], c[k]);
  }
};

// stats.txt's leaf_count (run.cpp:24-33, :126): the reference overloads
// sim_leaf_count for its non-uniform and adaptive sims and lets the generic
// template return 0 for the uniform one; these overloads are found by ADL
inline int64_t sim_leaf_count(const NonUniformSim& s) { return s.cells(); }
inline int64_t sim_leaf_count(const AdaptiveSim& s) { return s.cells(); }

// NonUniformSim / AdaptiveSim / UniformSim behind one runtime-dispatched
// handle (for loops written without templates, e.g. examples/drive_gpu.cpp);
// which one is decided like run_scenario (run.cpp:145-164).
class Sim : public SimBase {
 public:
  Sim(const fm_sim_desc& d, const fm_raster& dem, const Grid* grid = nullptr)
      : SimBase(d, dem, grid ? grid->get() : nullptr), adapt_every(d.adapt_every < 1 ? 1 : d.adapt_every) {
    adaptive_ = d.solver == FM_MWDG2 || d.solver == FM_HWFV1;
  }
  Sim(Sim&& o) noexcept
      : SimBase(std::move(o)), steps_since_adapt(o.steps_since_adapt), adapt_every(o.adapt_every),
        adaptive_(o.adaptive_) {}
  void step(double dt, int threads = 1) {
    SimBase::step(dt, threads);
    if (adaptive_) ++steps_since_adapt;
  }
  void adapt(double t) { check(fm_sim_adapt(s_, t)); }
  std::vector<std::pair<double, int64_t>> element_log_entries() const {
    const int64_t n = fm_sim_element_log(s_, nullptr, nullptr, 0);
    std::vector<double> t(n);
    std::vector<int64_t> c(n);
    fm_sim_element_log(s_, t.data(), c.data(), n);
    std::vector<std::pair<double, int64_t>> out(n);
    for (int64_t k = 0; k < n; ++k) out[k] = {t[k], c[k]};
    return out;
  }
  int64_t steps_since_adapt = 0;
  int adapt_every = 1;

 private:
  bool adaptive_ = false;
};

}  // namespace fm_gpu
