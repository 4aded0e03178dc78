// ORACLE — TEST INFRASTRUCTURE ONLY.
// C shim over the UNMODIFIED reference library, compiled from its own sources
// under /root/reference/proj/core by oracle/Makefile into oracle/_ref/.
// It exposes the same C signatures as the oracle (prefix `ref_`) so tests can
// pin the restatement against the reference itself, and bench.py can time
// the reference CPU path (--impl reference, cpu_baseline kind "reference").
//
// The reference factories read Manning / initial-depth rasters and
// hydrographs from files (ScenarioConfig paths, config.hpp:29-69), so the
// shim writes the caller's arrays to a private temp directory with
// write_ascii_grid (17 significant digits: exact round trip) first.
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <limits>
#include <memory>
#include <string>
#include <thread>
#include <variant>

#include "../include/fm_gpu.h"
#include "floodmra/detail_tree.hpp"
#include "floodmra/errors.hpp"
#include "floodmra/metrics.hpp"
#include "floodmra/hll.hpp"
#include "floodmra/raster.hpp"
#include "floodmra/sim_common.hpp"
#include "floodmra/solver_adaptive.hpp"
#include "floodmra/solver_nonuniform.hpp"
#include "floodmra/solver_uniform.hpp"
#include "floodmra/wavelets.hpp"

namespace fm = floodmra;

namespace {
thread_local std::string g_err;
int g_threads = 1;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return FM_OK;
  } catch (const fm::BlowUpError& e) {
    g_err = e.what();
    return FM_ERR_BLOWUP;
  } catch (const fm::ConfigError& e) {
    g_err = e.what();
    return FM_ERR_CONFIG;
  } catch (const fm::ParseError& e) {
    g_err = e.what();
    return FM_ERR_IO;
  } catch (const fm::IoError& e) {
    g_err = e.what();
    return FM_ERR_IO;
  } catch (const fm::StructureError& e) {
    g_err = e.what();
    return FM_ERR_STRUCTURE;
  } catch (const fm::DomainError& e) {
    g_err = e.what();
    return FM_ERR_DOMAIN;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FM_ERR_OTHER;
  }
}

fm::Raster to_raster(const fm_raster* r) {
  fm::Raster o;
  o.ncols = r->ncols;
  o.nrows = r->nrows;
  o.xll = r->xll;
  o.yll = r->yll;
  o.cellsize = r->cellsize;
  o.nodata = r->nodata;
  o.values.assign(r->values, r->values + size_t(r->ncols) * r->nrows);
  return o;
}

std::string scratch() {
  static int counter = 0;
  const auto dir = std::filesystem::temp_directory_path() /
                   ("fmref_" + std::to_string(getpid()) + "_" + std::to_string(counter++));
  std::filesystem::create_directories(dir);
  return dir.string();
}

fm::ScenarioConfig to_cfg(const fm_sim_desc* d, std::string& dir) {
  fm::ScenarioConfig c;
  c.solver = static_cast<fm::SolverKind>(d->solver);
  c.g = d->g;
  c.h_dry = d->h_dry;
  c.courant = d->courant;
  for (int q = 0; q < 4; ++q) c.boundary[q] = static_cast<fm::BoundaryKind>(d->bc[q]);
  c.manning = d->manning;
  dir = scratch();
  if (d->manning_raster) {
    c.manning_raster = dir + "/manning.asc";
    fm::write_ascii_grid(to_raster(d->manning_raster), c.manning_raster);
  }
  if (d->initial_depth_raster) {
    c.initial_depth_raster = dir + "/h0.asc";
    fm::write_ascii_grid(to_raster(d->initial_depth_raster), c.initial_depth_raster);
  }
  if (d->has_initial_surface) c.initial_surface = d->initial_surface;
  c.initial_depth = d->initial_depth;
  for (int k = 0; k < d->n_inflows; ++k) {
    const fm_inflow& f = d->inflows[k];
    const std::string p = dir + "/hydro_" + std::to_string(k) + ".csv";
    std::ofstream out(p);
    out.precision(17);
    out << "t,Q\n";
    for (int s = 0; s < f.nsamples; ++s) out << f.t[s] << "," << f.q[s] << "\n";
    out.close();
    c.inflows.push_back({p, f.i0, f.j0, f.i1, f.j1});
  }
  c.epsilon = d->epsilon;
  c.max_level = d->max_level;
  c.adapt_every = d->adapt_every;
  c.threads = g_threads;
  return c;
}
}  // namespace

struct ref_grid {
  fm::DetailTree tree;
  fm::NonUniformGrid nug;
  double eps = 0;
};

struct ref_sim {
  std::variant<fm::NonUniformSim, fm::AdaptiveSim, fm::UniformSim> s;
  template <typename F>
  auto visit(F&& f) {
    return std::visit(f, s);
  }
  fm::NonUniformSim* nu() {
    if (auto* p = std::get_if<fm::NonUniformSim>(&s)) return p;
    if (auto* a = std::get_if<fm::AdaptiveSim>(&s)) return &a->sim;
    return nullptr;
  }
};

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_set_threads(int32_t n) { g_threads = n < 1 ? 1 : n; }
int32_t ref_hw_threads(void) { return int32_t(std::max(1u, std::thread::hardware_concurrency())); }

// detail_tree.cpp:172-178, with the tree kept for flags / details.
int ref_mra_static(const fm_raster* dem, int32_t L, double eps, int32_t graded, int32_t kind,
                   ref_grid** out) {
  return guard([&] {
    auto g = std::make_unique<ref_grid>();
    const fm::Raster r = to_raster(dem);
    const auto k = static_cast<fm::WaveletKind>(kind);
    g->tree = fm::topography_tree(r, L, k);
    fm::flag_significant(g->tree, eps);
    if (graded) fm::grade_flags(g->tree);
    g->nug = fm::assemble_grid(g->tree, fm::filter_bank(k));
    g->eps = eps;
    *out = g.release();
  });
}

// The one-call pipeline, for timing the reference (bench cpu leg).
int ref_generate_static_grid(const fm_raster* dem, int32_t L, double eps, int32_t graded,
                             int32_t kind, int64_t* nleaves) {
  return guard([&] {
    const fm::NonUniformGrid g =
        fm::generate_static_grid(to_raster(dem), eps, L, graded != 0, static_cast<fm::WaveletKind>(kind));
    *nleaves = int64_t(g.grid.leaves.size());
  });
}

// read_nug's construction (quadgrid.cpp:310-327) from arrays: make_quadgrid +
// topography re-aligned to the sorted leaves.
int ref_grid_import(int32_t L, int32_t M, int32_t N, double R, double x0, double y0, int64_t n,
                    const int32_t* lv, const int32_t* ii, const int32_t* jj, const double* topo3,
                    ref_grid** out) {
  return guard([&] {
    auto g = std::make_unique<ref_grid>();
    std::vector<fm::LeafId> leaves(n);
    for (int64_t k = 0; k < n; ++k) leaves[k] = fm::LeafId{lv[k], ii[k], jj[k]};
    g->nug.grid = fm::make_quadgrid(L, M, N, R, x0, y0, leaves);
    g->nug.topo.resize(n);
    for (int64_t k = 0; k < n; ++k) {
      const int idx = g->nug.grid.find(lv[k], ii[k], jj[k]);
      g->nug.topo[idx] = fm::PlanarCoeffs{topo3[3 * k], topo3[3 * k + 1], topo3[3 * k + 2]};
    }
    *out = g.release();
  });
}

// The reference's own file formats (raster.cpp:22-96, quadgrid.cpp:287-327),
// for the byte-level checks of fm_raster_read / fm_raster_write / fm_grid_write
// / fm_grid_read (tests/test_io.py).  `binary` must be 0: the binary side
// formats are the GPU library's own.
int ref_raster_read(const char* path, fm_raster* out) {
  return guard([&] {
    const fm::Raster r = fm::read_ascii_grid(path);
    double* v = static_cast<double*>(std::malloc(std::max<size_t>(1, r.values.size()) * sizeof(double)));
    std::memcpy(v, r.values.data(), r.values.size() * sizeof(double));
    *out = fm_raster{v, r.ncols, r.nrows, r.xll, r.yll, r.cellsize, r.nodata, 0};
  });
}
int ref_raster_release(fm_raster* r) {
  std::free(const_cast<double*>(r->values));
  r->values = nullptr;
  return FM_OK;
}
int ref_raster_write(const fm_raster* r, const char* path, int32_t binary) {
  return guard([&] {
    if (binary) throw fm::ConfigError("the reference has no binary raster format");
    fm::write_ascii_grid(to_raster(r), path);
  });
}
int ref_grid_write(const ref_grid* g, const char* path, int32_t binary) {
  return guard([&] {
    if (binary) throw fm::ConfigError("the reference has no binary grid format");
    fm::write_nug(g->nug, path);
  });
}
int ref_grid_read(const char* path, ref_grid** out) {
  return guard([&] {
    auto g = std::make_unique<ref_grid>();
    g->nug = fm::read_nug(path);
    *out = g.release();
  });
}

int ref_grid_destroy(ref_grid* g) {
  delete g;
  return FM_OK;
}
int64_t ref_grid_num_leaves(const ref_grid* g) { return int64_t(g->nug.grid.leaves.size()); }

int ref_grid_info(const ref_grid* g, int32_t* L, int32_t* M, int32_t* N, double* R, double* x0,
                  double* y0, double* norm) {
  if (L) *L = g->nug.grid.L;
  if (M) *M = g->nug.grid.M;
  if (N) *N = g->nug.grid.N;
  if (R) *R = g->nug.grid.Rfine;
  if (x0) *x0 = g->nug.grid.x0;
  if (y0) *y0 = g->nug.grid.y0;
  if (norm) *norm = g->tree.field_norm;
  return FM_OK;
}

int ref_grid_leaves(const ref_grid* g, int32_t, int32_t* lv, int32_t* i, int32_t* j, double* topo3) {
  const auto& L = g->nug.grid.leaves;
  for (size_t k = 0; k < L.size(); ++k) {
    if (lv) lv[k] = L[k].level;
    if (i) i[k] = L[k].i;
    if (j) j[k] = L[k].j;
    if (topo3) {
      topo3[3 * k] = g->nug.topo[k].c0;
      topo3[3 * k + 1] = g->nug.topo[k].c1x;
      topo3[3 * k + 2] = g->nug.topo[k].c1y;
    }
  }
  return FM_OK;
}

int ref_grid_flags(const ref_grid* g, int32_t level, uint8_t* out) {
  std::memcpy(out, g->tree.flags[level].data(), g->tree.flags[level].size());
  return FM_OK;
}

int ref_grid_dhat(const ref_grid* g, int32_t level, double* out) {
  for (size_t k = 0; k < g->tree.details[level].size(); ++k)
    out[k] = fm::normalize_detail(g->tree.details[level][k], g->tree.field_norm);
  return FM_OK;
}

int ref_grid_details(const ref_grid* g, int32_t level, double* out9) {
  for (size_t k = 0; k < g->tree.details[level].size(); ++k) {
    const fm::DetailTriple& d = g->tree.details[level][k];
    const double v[9] = {d.dh.c0, d.dh.c1x, d.dh.c1y, d.dv.c0, d.dv.c1x,
                         d.dv.c1y, d.dd.c0, d.dd.c1x, d.dd.c1y};
    std::memcpy(out9 + 9 * k, v, sizeof(v));
  }
  return FM_OK;
}

int ref_grid_near_threshold(const ref_grid* g, double rel, int64_t* count) {
  int64_t c = 0;
  for (const auto& lvl : g->tree.details)
    for (const auto& d : lvl)
      if (std::abs(fm::normalize_detail(d, g->tree.field_norm) - g->eps) <= rel * g->eps) ++c;
  *count = c;
  return FM_OK;
}

int ref_sim_create(const fm_sim_desc* d, const fm_raster* dem, const ref_grid* grid, ref_sim** out) {
  return guard([&] {
    std::string dir;
    const fm::ScenarioConfig c = to_cfg(d, dir);
    const fm::Raster r = to_raster(dem);
    auto s = std::make_unique<ref_sim>();
    if (fm::solver_is_adaptive(c.solver))
      s->s = fm::make_adaptive_sim(c, r);
    else if (grid)
      s->s = fm::make_nonuniform_sim(c, r, grid->nug);
    else
      s->s = fm::make_uniform_sim(c, r);
    std::filesystem::remove_all(dir);
    *out = s.release();
  });
}

int ref_sim_destroy(ref_sim* s) {
  delete s;
  return FM_OK;
}

int64_t ref_sim_num_cells(ref_sim* s) {
  if (auto* u = std::get_if<fm::UniformSim>(&s->s)) return int64_t(u->u.size());
  return int64_t(s->nu()->u.size());
}

int64_t ref_sim_num_segments(ref_sim* s) {
  if (auto* u = std::get_if<fm::UniformSim>(&s->s))
    return int64_t(u->nx + 1) * u->ny + int64_t(u->nx) * (u->ny + 1);
  return int64_t(s->nu()->faces.interior.size());
}

int ref_sim_compute_dt(ref_sim* s, double* dt) {
  return guard([&] { *dt = s->visit([](auto& x) { return x.compute_dt(); }); });
}
int ref_sim_step(ref_sim* s, double dt) {
  return guard([&] { s->visit([&](auto& x) { x.step(dt, g_threads); }); });
}
int ref_sim_apply_inflows(ref_sim* s, double t, double dt, double* added) {
  return guard([&] { *added = s->visit([&](auto& x) { return x.apply_inflows(t, dt); }); });
}
int ref_sim_adapt(ref_sim* s, double t) {
  return guard([&] {
    auto* a = std::get_if<fm::AdaptiveSim>(&s->s);
    if (!a) throw fm::ConfigError("adapt: not an adaptive simulation");
    a->adapt(t);
    a->steps_since_adapt = 0;
  });
}
int ref_sim_volume(ref_sim* s, double* v) {
  return guard([&] { *v = s->visit([](auto& x) { return x.volume(); }); });
}
int ref_sim_finite(ref_sim* s, int32_t* ok, double* bx, double* by) {
  return guard([&] { *ok = s->visit([&](auto& x) { return x.finite_state(bx, by); }) ? 1 : 0; });
}

int ref_sim_download(ref_sim* s, int32_t* lv, int32_t* ii, int32_t* jj, double* u9, double* z3) {
  return guard([&] {
    static_assert(sizeof(fm::FlowCoeffs) == 9 * sizeof(double));
    static_assert(sizeof(fm::PlanarCoeffs) == 3 * sizeof(double));
    if (auto* u = std::get_if<fm::UniformSim>(&s->s)) {
      for (int j = 0; j < u->ny; ++j)
        for (int i = 0; i < u->nx; ++i) {
          const size_t c = u->cell(i, j);
          if (lv) lv[c] = 0;
          if (ii) ii[c] = i;
          if (jj) jj[c] = j;
        }
      if (u9) std::memcpy(u9, u->u.data(), u->u.size() * sizeof(fm::FlowCoeffs));
      if (z3) std::memcpy(z3, u->z.data(), u->z.size() * sizeof(fm::PlanarCoeffs));
      return;
    }
    fm::NonUniformSim* n = s->nu();
    for (size_t k = 0; k < n->grid.leaves.size(); ++k) {
      if (lv) lv[k] = n->grid.leaves[k].level;
      if (ii) ii[k] = n->grid.leaves[k].i;
      if (jj) jj[k] = n->grid.leaves[k].j;
    }
    if (u9) std::memcpy(u9, n->u.data(), n->u.size() * sizeof(fm::FlowCoeffs));
    if (z3) std::memcpy(z3, n->z.data(), n->z.size() * sizeof(fm::PlanarCoeffs));
  });
}

// depth_raster()/qx_raster()/qy_raster() and sample_gauge() of the reference
// sims (solver_nonuniform.cpp:489-519, solver_uniform.cpp:480-520).
static fm::Raster ref_raster(ref_sim* s, int which) {
  return s->visit([&](auto& sim) {
    return which == 0 ? sim.depth_raster() : which == 1 ? sim.qx_raster() : sim.qy_raster();
  });
}

int ref_sim_raster_shape(ref_sim* s, int32_t* nc, int32_t* nr, double* xll, double* yll,
                         double* cs, double* nodata) {
  return guard([&] {
    const fm::Raster r = ref_raster(s, 0);
    *nc = r.ncols, *nr = r.nrows, *xll = r.xll, *yll = r.yll, *cs = r.cellsize, *nodata = r.nodata;
  });
}

int ref_sim_raster(ref_sim* s, int32_t which, double* out, int32_t on_device) {
  return guard([&] {
    if (on_device) throw fm::ConfigError("reference rasters are host-only");
    const fm::Raster r = ref_raster(s, which);
    std::memcpy(out, r.values.data(), r.values.size() * sizeof(double));
  });
}

int ref_sim_sample_gauges(ref_sim* s, int32_t n, const double* x, const double* y, double* out4) {
  return guard([&] {
    for (int32_t k = 0; k < n; ++k) {
      const fm::GaugeValue v = s->visit([&](auto& sim) { return sim.sample_gauge(x[k], y[k]); });
      out4[4 * k] = v.h, out4[4 * k + 1] = v.eta, out4[4 * k + 2] = v.u, out4[4 * k + 3] = v.v;
    }
  });
}

int ref_extent_metrics(const fm_raster* test, const fm_raster* ref, double wet, int64_t* counts,
                       double* rates) {
  return guard([&] {
    const fm::ExtentMetrics m = fm::extent_metrics(to_raster(test), to_raster(ref), wet);
    counts[0] = m.hits, counts[1] = m.misses, counts[2] = m.false_alarms;
    rates[0] = m.hit_rate, rates[1] = m.false_alarm, rates[2] = m.csi;
  });
}

int ref_sim_upload(ref_sim* s, const double* u9) {
  return guard([&] {
    auto& u = std::get_if<fm::UniformSim>(&s->s) ? std::get_if<fm::UniformSim>(&s->s)->u : s->nu()->u;
    std::memcpy(u.data(), u9, u.size() * sizeof(fm::FlowCoeffs));
  });
}

int ref_sim_acc_q(ref_sim* s, double* a, double* b) {
  return guard([&] {
    if (auto* u = std::get_if<fm::UniformSim>(&s->s)) {
      if (a) std::copy(u->acc_qx.begin(), u->acc_qx.end(), a);
      if (b) std::copy(u->acc_qy.begin(), u->acc_qy.end(), b);
      return;
    }
    fm::NonUniformSim* n = s->nu();
    if (a) std::copy(n->acc_q.begin(), n->acc_q.end(), a);
    if (b) std::copy(n->acc_qb.begin(), n->acc_qb.end(), b);
  });
}

int64_t ref_sim_element_log(ref_sim* s, double* t, int64_t* count, int64_t cap) {
  auto* a = std::get_if<fm::AdaptiveSim>(&s->s);
  if (!a) return 0;
  const int64_t n = int64_t(a->element_log.size());
  for (int64_t k = 0; k < std::min(n, cap); ++k) {
    if (t) t[k] = a->element_log[k].first;
    if (count) count[k] = a->element_log[k].second;
  }
  return n;
}

// The drive<Sim> loop body (run.cpp:80-111) over the reference sim and the
// reference EventClock, without file output.
int ref_sim_run(ref_sim* s, fm_clock* ck, int64_t max_steps, int32_t stop_at_events,
                fm_run_result* out) {
  return guard([&] {
    fm::EventClock clock;
    clock.end_time = ck->end_time;
    clock.output_interval = ck->output_interval;
    clock.gauge_interval = ck->gauge_interval;
    clock.now = ck->now;
    clock.next_output = ck->next_output;
    clock.next_gauge = ck->next_gauge;
    fm_run_result r{};
    r.dt_min = std::numeric_limits<double>::infinity();
    s->visit([&](auto& sim) {
      while (r.steps < max_steps && !clock.finished()) {
        double dt = clock.clip(sim.compute_dt());
        if (!(dt > 0.0)) dt = clock.clip(clock.end_time);
        sim.step(dt, g_threads);
        r.volume_inflow += sim.apply_inflows(clock.now, dt);
        clock.advance(dt);
        ++r.steps;
        r.dt_min = std::min(r.dt_min, dt);
        r.dt_max = std::max(r.dt_max, dt);
        if constexpr (requires { sim.adapt(0.0); }) {
          if (sim.steps_since_adapt >= sim.adapt_every && !clock.finished()) {
            sim.adapt(clock.now);
            sim.steps_since_adapt = 0;
          }
        }
        double bx = 0, by = 0;
        if (!sim.finite_state(&bx, &by)) {
          r.blew_up = 1;
          r.blow_up_time = clock.now;
          r.bad_x = bx;
          r.bad_y = by;
          break;
        }
        const bool g = clock.gauge_due();
        const bool o = clock.output_due();
        if ((g || o) && stop_at_events) {
          r.event_due = 1;
          break;
        }
      }
    });
    ck->now = clock.now;
    ck->next_output = clock.next_output;
    ck->next_gauge = clock.next_gauge;
    r.finished = clock.finished();
    *out = r;
    if (r.blew_up) throw fm::BlowUpError("solver state is non-finite", r.blow_up_time);
  });
}

int ref_grade_flags(int32_t L, int32_t M, int32_t N, int32_t graded, uint8_t* flags) {
  return guard([&] {
    fm::DetailTree t;
    t.L = L;
    t.M = M;
    t.N = N;
    t.flags.resize(L);
    size_t at = 0;
    for (int l = 0; l < L; ++l) {
      const size_t n = size_t(t.width(l)) * t.height(l);
      t.flags[l].assign(flags + at, flags + at + n);
      at += n;
    }
    fm::ancestor_closure(t);
    if (graded) fm::grade_flags(t);
    at = 0;
    for (int l = 0; l < L; ++l) {
      std::memcpy(flags + at, t.flags[l].data(), t.flags[l].size());
      at += t.flags[l].size();
    }
  });
}

void ref_hll(double hl, double qnl, double qtl, double hr, double qnr, double qtr, double g,
             double hdry, double* out3) {
  const fm::Flux3 f = fm::hll_flux(hl, qnl, qtl, hr, qnr, qtr, g, hdry);
  out3[0] = f.mass;
  out3[1] = f.mom_n;
  out3[2] = f.mom_t;
}

void ref_friction(double h0, double* qx3, double* qy3, double n, double g, double hdry, double dt) {
  fm::PlanarCoeffs a{qx3[0], qx3[1], qx3[2]}, b{qy3[0], qy3[1], qy3[2]};
  fm::friction_update(h0, a, b, n, g, hdry, dt);
  qx3[0] = a.c0;
  qx3[1] = a.c1x;
  qx3[2] = a.c1y;
  qy3[0] = b.c0;
  qy3[1] = b.c1x;
  qy3[2] = b.c1y;
}

void ref_encode(const double* kids12, int32_t kind, double* parent3, double* det9) {
  std::array<fm::PlanarCoeffs, 4> k;
  for (int c = 0; c < 4; ++c) k[c] = {kids12[3 * c], kids12[3 * c + 1], kids12[3 * c + 2]};
  const fm::EncodeResult e = fm::encode(k, fm::filter_bank(static_cast<fm::WaveletKind>(kind)));
  parent3[0] = e.parent.c0;
  parent3[1] = e.parent.c1x;
  parent3[2] = e.parent.c1y;
  const double v[9] = {e.d.dh.c0, e.d.dh.c1x, e.d.dh.c1y, e.d.dv.c0, e.d.dv.c1x,
                       e.d.dv.c1y, e.d.dd.c0, e.d.dd.c1x, e.d.dd.c1y};
  std::memcpy(det9, v, sizeof(v));
}

void ref_decode(const double* parent3, const double* det9, int32_t kind, double* kids12) {
  fm::DetailTriple d;
  d.dh = {det9[0], det9[1], det9[2]};
  d.dv = {det9[3], det9[4], det9[5]};
  d.dd = {det9[6], det9[7], det9[8]};
  const auto k = fm::decode({parent3[0], parent3[1], parent3[2]}, d,
                            fm::filter_bank(static_cast<fm::WaveletKind>(kind)));
  for (int c = 0; c < 4; ++c) {
    kids12[3 * c] = k[c].c0;
    kids12[3 * c + 1] = k[c].c1x;
    kids12[3 * c + 2] = k[c].c1y;
  }
}

}  // extern "C"
