// fm_gpu.hpp — header-only C++ host side over the C ABI (fm_gpu.h).
//
// Drop-in classes for the reference's duck-typed drive<Sim> loop
// (/root/reference/proj/core/src/run.cpp:35-141): each exposes the members
// drive<Sim> calls — compute_dt, step(dt, threads), apply_inflows(t, dt),
// volume, finite_state(&x, &y) and, for the adaptive solvers, adapt(t),
// steps_since_adapt, adapt_every and element_log — and raises the reference's
// exception types (errors.hpp:9-37) from the ABI's status codes.
//
// Define FM_GPU_WITH_FLOODMRA before including this header (with the
// reference's include path) to throw floodmra::ConfigError & co. and to get
// fm_gpu::view(const floodmra::Raster&) (raster.hpp:10-32).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fm_gpu.h"

#ifdef FM_GPU_WITH_FLOODMRA
#include "floodmra/errors.hpp"
#include "floodmra/raster.hpp"
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
  fm_grid* g_ = nullptr;
};

// NonUniformSim / AdaptiveSim / UniformSim behind one handle; which one is
// decided like run_scenario (run.cpp:145-164).
class Sim {
 public:
  Sim(const fm_sim_desc& d, const fm_raster& dem, const Grid* grid = nullptr)
      : adapt_every(d.adapt_every < 1 ? 1 : d.adapt_every) {
    check(fm_sim_create(&d, &dem, grid ? grid->get() : nullptr, &s_));
    adaptive_ = d.solver == FM_MWDG2 || d.solver == FM_HWFV1;
  }
  Sim(const Sim&) = delete;
  Sim& operator=(const Sim&) = delete;
  Sim(Sim&& o) noexcept
      : steps_since_adapt(o.steps_since_adapt), adapt_every(o.adapt_every),
        s_(std::exchange(o.s_, nullptr)), adaptive_(o.adaptive_) {}
  ~Sim() {
    if (s_) fm_sim_destroy(s_);
  }

  // ---- drive<Sim> members ------------------------------------------------
  double compute_dt() const {
    double dt = 0.0;
    check(fm_sim_compute_dt(s_, &dt));
    return dt;
  }
  void step(double dt, int /*threads*/ = 1) {
    check(fm_sim_step(s_, dt));
    if (adaptive_) ++steps_since_adapt;
  }
  double apply_inflows(double t, double dt) {
    double added = 0.0;
    check(fm_sim_apply_inflows(s_, t, dt, &added));
    return added;
  }
  void adapt(double t) { check(fm_sim_adapt(s_, t)); }
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
  std::vector<std::pair<double, int64_t>> element_log() const {
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

 private:
  fm_sim* s_ = nullptr;
  bool adaptive_ = false;
};

}  // namespace fm_gpu
