// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle_core.hpp).
// C ABI of the CPU restatement: the same signatures as include/fm_gpu.h with
// an `orc_` prefix, so the parity tests can call both sides identically.
#include <algorithm>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <variant>

#include "../include/fm_gpu.h"
#include "oracle_sims.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

int fail_code(int c) {
  switch (c) {
    case E_CONFIG: return FM_ERR_CONFIG;
    case E_IO: return FM_ERR_IO;
    case E_BLOWUP: return FM_ERR_BLOWUP;
    case E_STRUCT: return FM_ERR_STRUCTURE;
    case E_DOMAIN: return FM_ERR_DOMAIN;
  }
  return FM_ERR_OTHER;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return FM_OK;
  } catch (const Fail& e) {
    g_err = e.what();
    return fail_code(e.code);
  } catch (const std::exception& e) {
    g_err = e.what();
    return FM_ERR_OTHER;
  }
}

Raster to_raster(const fm_raster* r) {
  if (!r || !r->values) throw Fail(E_CONFIG, "null raster");
  if (r->on_device) throw Fail(E_CONFIG, "oracle takes host rasters only");
  Raster o;
  o.ncols = r->ncols;
  o.nrows = r->nrows;
  o.xll = r->xll;
  o.yll = r->yll;
  o.cell = r->cellsize;
  o.nodata = r->nodata;
  o.v.assign(r->values, r->values + size_t(r->ncols) * r->nrows);
  return o;
}

Cfg to_cfg(const fm_sim_desc* d) {
  Cfg c;
  c.solver = d->solver;
  c.g = d->g;
  c.hdry = d->h_dry;
  c.courant = d->courant;
  for (int q = 0; q < 4; ++q) c.bc[q] = d->bc[q];
  c.manning = d->manning;
  if (d->manning_raster) {
    c.has_mr = true;
    c.mr = to_raster(d->manning_raster);
  }
  if (d->initial_depth_raster) {
    c.has_h0 = true;
    c.h0 = to_raster(d->initial_depth_raster);
  }
  c.has_eta0 = d->has_initial_surface != 0;
  c.eta0 = d->initial_surface;
  c.depth0 = d->initial_depth;
  for (int k = 0; k < d->n_inflows; ++k) {
    const fm_inflow& f = d->inflows[k];
    Inflow r;
    r.hy.t.assign(f.t, f.t + f.nsamples);
    r.hy.q.assign(f.q, f.q + f.nsamples);
    r.i0 = f.i0;
    r.j0 = f.j0;
    r.i1 = f.i1;
    r.j1 = f.j1;
    c.inflows.push_back(r);
  }
  c.eps = d->epsilon;
  c.L = d->max_level;
  c.adapt_every = d->adapt_every;
  c.libm = d->libm;
  return c;
}
}  // namespace

struct orc_grid {
  Tree tree;
  Grid grid;
  std::vector<Pl> topo;
  double eps = 0;
};

struct orc_sim {
  std::variant<NU, AD, UN> s;
  NU* nu() {
    if (auto* p = std::get_if<NU>(&s)) return p;
    if (auto* a = std::get_if<AD>(&s)) return &a->sim;
    return nullptr;
  }
  AD* ad() { return std::get_if<AD>(&s); }
  UN* un() { return std::get_if<UN>(&s); }
  double compute_dt() { return un() ? un()->compute_dt() : nu()->compute_dt(); }
  void step(double dt) {
    if (un())
      un()->step(dt);
    else
      nu()->step(dt);
    if (ad()) ad()->since += 1;
  }
  double inflow(double t, double dt) { return un() ? un()->apply_inflows(t, dt) : nu()->apply_inflows(t, dt); }
  bool finite(double* x, double* y) { return un() ? un()->finite(x, y) : nu()->finite(x, y); }
  double volume() { return un() ? un()->volume() : nu()->volume(); }
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_mra_static(const fm_raster* dem, int32_t L, double eps, int32_t graded, int32_t kind,
                   orc_grid** out) {
  return guard([&] {
    auto g = std::make_unique<orc_grid>();
    const Raster r = to_raster(dem);
    int M = 0, N = 0;
    const Field f = project_padded(r, L, &M, &N);
    g->tree = encode_tree(f, L, M, N, kind);
    threshold(g->tree, eps);
    if (graded) grade(g->tree);
    g->grid = make_grid(L, M, N, f.R, f.x0, f.y0, tree_leaves(g->tree));
    tree_decode(g->tree, g->grid, g->topo);
    g->eps = eps;
    *out = g.release();
  });
}

// read_nug (quadgrid.cpp:310-327): make_quadgrid over a leaf list plus the
// per-leaf topography, re-aligned to the sorted leaf order.
int orc_grid_import(int32_t L, int32_t M, int32_t N, double R, double x0, double y0, int64_t n,
                    const int32_t* lv, const int32_t* ii, const int32_t* jj, const double* topo3,
                    orc_grid** out) {
  return guard([&] {
    auto g = std::make_unique<orc_grid>();
    std::vector<Leaf> leaves(n);
    for (int64_t k = 0; k < n; ++k) leaves[k] = Leaf{lv[k], ii[k], jj[k]};
    g->grid = make_grid(L, M, N, R, x0, y0, leaves);
    g->topo.assign(n, Pl{});
    for (int64_t k = 0; k < n; ++k) {
      const int idx = g->grid.find(lv[k], ii[k], jj[k]);
      if (idx < 0) throw Fail(E_STRUCT, "grid import: duplicate leaf");
      g->topo[idx] = Pl{topo3[3 * k], topo3[3 * k + 1], topo3[3 * k + 2]};
    }
    *out = g.release();
  });
}

int orc_grid_destroy(orc_grid* g) {
  delete g;
  return FM_OK;
}

int64_t orc_grid_num_leaves(const orc_grid* g) { return int64_t(g->grid.lv.size()); }

int orc_grid_info(const orc_grid* g, int32_t* L, int32_t* M, int32_t* N, double* R, double* x0,
                  double* y0, double* norm) {
  if (L) *L = g->grid.L;
  if (M) *M = g->grid.M;
  if (N) *N = g->grid.N;
  if (R) *R = g->grid.R;
  if (x0) *x0 = g->grid.x0;
  if (y0) *y0 = g->grid.y0;
  if (norm) *norm = g->tree.norm;
  return FM_OK;
}

int orc_grid_leaves(const orc_grid* g, int32_t, int32_t* lv, int32_t* i, int32_t* j, double* topo3) {
  for (size_t k = 0; k < g->grid.lv.size(); ++k) {
    if (lv) lv[k] = g->grid.lv[k].l;
    if (i) i[k] = g->grid.lv[k].i;
    if (j) j[k] = g->grid.lv[k].j;
    if (topo3) {
      topo3[3 * k] = g->topo[k].c0;
      topo3[3 * k + 1] = g->topo[k].cx;
      topo3[3 * k + 2] = g->topo[k].cy;
    }
  }
  return FM_OK;
}

int orc_grid_flags(const orc_grid* g, int32_t level, uint8_t* out) {
  if (level < 0 || level >= g->tree.L) {
    g_err = "level out of range";
    return FM_ERR_DOMAIN;
  }
  std::memcpy(out, g->tree.flag[level].data(), g->tree.flag[level].size());
  return FM_OK;
}

int orc_grid_dhat(const orc_grid* g, int32_t level, double* out) {
  if (level < 0 || level >= g->tree.L) {
    g_err = "level out of range";
    return FM_ERR_DOMAIN;
  }
  for (size_t k = 0; k < g->tree.det[level].size(); ++k)
    out[k] = dhat(g->tree.det[level][k], g->tree.norm);
  return FM_OK;
}

// Raw details (9 per node) — for the golden fixtures.
int orc_grid_details(const orc_grid* g, int32_t level, double* out9) {
  if (level < 0 || level >= g->tree.L) {
    g_err = "level out of range";
    return FM_ERR_DOMAIN;
  }
  for (size_t k = 0; k < g->tree.det[level].size(); ++k)
    for (int n = 0; n < 9; ++n) out9[9 * k + n] = g->tree.det[level][k].v[n];
  return FM_OK;
}

int orc_grid_near_threshold(const orc_grid* g, double rel, int64_t* count) {
  int64_t c = 0;
  for (int l = 0; l < g->tree.L; ++l)
    for (const Det& d : g->tree.det[l])
      if (std::abs(dhat(d, g->tree.norm) - g->eps) <= rel * g->eps) ++c;
  *count = c;
  return FM_OK;
}

int orc_sim_create(const fm_sim_desc* d, const fm_raster* dem, const orc_grid* grid,
                   orc_sim** out) {
  return guard([&] {
    auto s = std::make_unique<orc_sim>();
    const Cfg c = to_cfg(d);
    const Raster r = to_raster(dem);
    if (c.solver == S_MWDG2 || c.solver == S_HWFV1)
      s->s = make_ad(c, r);
    else if (grid)
      s->s = make_nu(c, r, grid->grid, grid->topo);
    else
      s->s = make_un(c, r);
    *out = s.release();
  });
}

int orc_sim_destroy(orc_sim* s) {
  delete s;
  return FM_OK;
}

int64_t orc_sim_num_cells(orc_sim* s) {
  return s->un() ? int64_t(s->un()->u.size()) : int64_t(s->nu()->u.size());
}

int64_t orc_sim_num_segments(orc_sim* s) {
  return s->un() ? int64_t(s->un()->nx + 1) * s->un()->ny + int64_t(s->un()->nx) * (s->un()->ny + 1)
                 : int64_t(s->nu()->F.in.size());
}

int orc_sim_compute_dt(orc_sim* s, double* dt) {
  return guard([&] { *dt = s->compute_dt(); });
}
int orc_sim_step(orc_sim* s, double dt) {
  return guard([&] { s->step(dt); });
}
int orc_sim_apply_inflows(orc_sim* s, double t, double dt, double* added) {
  return guard([&] { *added = s->inflow(t, dt); });
}
int orc_sim_adapt(orc_sim* s, double t) {
  return guard([&] {
    if (!s->ad()) throw Fail(E_CONFIG, "adapt: not an adaptive simulation");
    s->ad()->adapt(t);
    s->ad()->since = 0;
  });
}
int orc_sim_volume(orc_sim* s, double* v) {
  return guard([&] { *v = s->volume(); });
}
int orc_sim_finite(orc_sim* s, int32_t* ok, double* bx, double* by) {
  return guard([&] { *ok = s->finite(bx, by) ? 1 : 0; });
}

int orc_sim_download(orc_sim* s, int32_t* lv, int32_t* ii, int32_t* jj, double* u9, double* z3) {
  return guard([&] {
    if (UN* u = s->un()) {
      for (int j = 0; j < u->ny; ++j)
        for (int i = 0; i < u->nx; ++i) {
          const size_t c = u->cell(i, j);
          if (lv) lv[c] = 0;
          if (ii) ii[c] = i;
          if (jj) jj[c] = j;
        }
      if (u9) std::memcpy(u9, u->u.data(), u->u.size() * sizeof(Fl));
      if (z3) std::memcpy(z3, u->z.data(), u->z.size() * sizeof(Pl));
      return;
    }
    NU* n = s->nu();
    for (size_t k = 0; k < n->grid.lv.size(); ++k) {
      if (lv) lv[k] = n->grid.lv[k].l;
      if (ii) ii[k] = n->grid.lv[k].i;
      if (jj) jj[k] = n->grid.lv[k].j;
    }
    if (u9) std::memcpy(u9, n->u.data(), n->u.size() * sizeof(Fl));
    if (z3) std::memcpy(z3, n->z.data(), n->z.size() * sizeof(Pl));
  });
}

// Raster geometry of depth_raster()/qx_raster()/qy_raster() (quadgrid.cpp:266-272,
// solver_uniform.cpp:503-509).
int orc_sim_raster_shape(orc_sim* s, int32_t* nc, int32_t* nr, double* xll, double* yll,
                         double* cs, double* nodata) {
  return guard([&] {
    if (UN* u = s->un()) {
      *nc = u->nx, *nr = u->ny, *xll = u->x0, *yll = u->y0, *cs = u->R, *nodata = -9999.0;
      return;
    }
    const Grid& g = s->nu()->grid;
    *nc = g.M << g.L, *nr = g.N << g.L, *xll = g.x0, *yll = g.y0, *cs = g.R, *nodata = -9999.0;
  });
}

int orc_sim_raster(orc_sim* s, int32_t which, double* out, int32_t on_device) {
  return guard([&] {
    if (on_device) throw Fail(E_CONFIG, "oracle rasters are host-only");
    if (which < 0 || which > 2) throw Fail(E_CONFIG, "raster: which must be 0 (h), 1 (qx) or 2 (qy)");
    if (UN* u = s->un())
      raster(*u, which, out);
    else
      raster(*s->nu(), which, out);
  });
}

int orc_sim_sample_gauges(orc_sim* s, int32_t n, const double* x, const double* y, double* out4) {
  return guard([&] {
    for (int32_t k = 0; k < n; ++k) {
      if (UN* u = s->un())
        gauge(*u, x[k], y[k], out4 + 4 * k);
      else
        gauge(*s->nu(), x[k], y[k], out4 + 4 * k);
    }
  });
}

// Leaves (reference order) and interior segments (enumerate_faces order,
// quadgrid.cpp:184-260) of a non-uniform sim: the topology the shard plan of
// the GPU library partitions.
int orc_sim_topology(orc_sim* s, int32_t* lv, int32_t* ii, int32_t* jj, int32_t* sl, int32_t* sr) {
  return guard([&] {
    NU* n = s->nu();
    if (!n) throw Fail(E_CONFIG, "topology: uniform sims have no leaf list");
    for (size_t k = 0; k < n->grid.lv.size(); ++k) {
      if (lv) lv[k] = n->grid.lv[k].l;
      if (ii) ii[k] = n->grid.lv[k].i;
      if (jj) jj[k] = n->grid.lv[k].j;
    }
    for (size_t q = 0; q < n->F.in.size(); ++q) {
      if (sl) sl[q] = n->F.in[q].l;
      if (sr) sr[q] = n->F.in[q].r;
    }
  });
}
// extent_metrics (metrics.cpp:51-73)
int orc_extent_metrics(const fm_raster* test, const fm_raster* ref, double wet, int64_t* counts,
                       double* rates) {
  return guard([&] {
    if (test->ncols != ref->ncols || test->nrows != ref->nrows || test->xll != ref->xll ||
        test->yll != ref->yll || test->cellsize != ref->cellsize)
      throw Fail(E_IO, "extent_metrics: raster geometries do not match");
    long long h = 0, m = 0, f = 0;
    const size_t n = size_t(ref->ncols) * ref->nrows;
    for (size_t k = 0; k < n; ++k) {
      const double a = test->values[k], b = ref->values[k];
      if (a == test->nodata || b == ref->nodata) continue;
      const bool wt = a >= wet, wr = b >= wet;
      if (wt && wr)
        ++h;
      else if (!wt && wr)
        ++m;
      else if (wt && !wr)
        ++f;
    }
    counts[0] = h, counts[1] = m, counts[2] = f;
    rates[0] = (h + m) > 0 ? double(h) / double(h + m) : 1.0;
    rates[1] = (h + f) > 0 ? double(f) / double(h + f) : 0.0;
    rates[2] = (h + m + f) > 0 ? double(h) / double(h + m + f) : 1.0;
  });
}

int orc_sim_upload(orc_sim* s, const double* u9) {
  return guard([&] {
    auto& u = s->un() ? s->un()->u : s->nu()->u;
    std::memcpy(static_cast<void*>(u.data()), u9, u.size() * sizeof(Fl));
  });
}

// ACC face discharges (acc_q / acc_qb, or acc_qx / acc_qy for the raster).
int orc_sim_acc_q(orc_sim* s, double* a, double* b) {
  return guard([&] {
    if (UN* u = s->un()) {
      if (a) std::copy(u->aqx.begin(), u->aqx.end(), a);
      if (b) std::copy(u->aqy.begin(), u->aqy.end(), b);
      return;
    }
    NU* n = s->nu();
    if (a) std::copy(n->accq.begin(), n->accq.end(), a);
    if (b) std::copy(n->accqb.begin(), n->accqb.end(), b);
  });
}

int64_t orc_sim_element_log(orc_sim* s, double* t, int64_t* count, int64_t cap) {
  AD* a = s->ad();
  if (!a) return 0;
  const int64_t n = int64_t(a->log.size());
  for (int64_t k = 0; k < std::min(n, cap); ++k) {
    if (t) t[k] = a->log[k].first;
    if (count) count[k] = a->log[k].second;
  }
  return n;
}

// run.cpp:80-111 — the drive loop body, with EventClock (sim_common.cpp:48-82).
int orc_sim_run(orc_sim* s, fm_clock* ck, int64_t max_steps, int32_t stop_at_events,
                fm_run_result* out) {
  return guard([&] {
    fm_run_result r{};
    r.dt_min = std::numeric_limits<double>::infinity();
    auto next_event = [&] {
      double e = ck->end_time;
      if (ck->output_interval > 0.0) e = mn(e, ck->next_output * ck->output_interval);
      if (ck->gauge_interval > 0.0) e = mn(e, ck->next_gauge * ck->gauge_interval);
      return e;
    };
    auto clip = [&](double dt) { return mn(dt, mx(next_event() - ck->now, 0.0)); };
    auto reached = [&](double target) { return ck->now >= target - 1e-9 * mx(1.0, target); };
    while (r.steps < max_steps && !(ck->now >= ck->end_time)) {
      double dt = clip(s->compute_dt());
      if (!(dt > 0.0)) dt = clip(ck->end_time);
      s->step(dt);
      r.volume_inflow += s->inflow(ck->now, dt);
      ck->now += dt;
      ++r.steps;
      r.dt_min = mn(r.dt_min, dt);
      r.dt_max = mx(r.dt_max, dt);
      if (AD* a = s->ad())
        if (a->since >= a->adapt_every && !(ck->now >= ck->end_time)) {
          a->adapt(ck->now);
          a->since = 0;
        }
      double bx = 0, by = 0;
      if (!s->finite(&bx, &by)) {
        r.blew_up = 1;
        r.blow_up_time = ck->now;
        r.bad_x = bx;
        r.bad_y = by;
        break;
      }
      bool ev = false;
      if (ck->gauge_interval > 0.0 && reached(ck->next_gauge * ck->gauge_interval)) {
        ++ck->next_gauge;
        ev = true;
      }
      if (ck->output_interval > 0.0 && reached(ck->next_output * ck->output_interval)) {
        ++ck->next_output;
        ev = true;
      }
      if (ev && stop_at_events) {
        r.event_due = 1;
        break;
      }
    }
    r.finished = ck->now >= ck->end_time;
    *out = r;
    if (r.blew_up) throw Fail(E_BLOWUP, "solver state is non-finite");
  });
}

// Raw point kernels for the known-answer tests (hll.cpp, sim_common.cpp,
// wavelets.cpp).
void orc_hll(double hl, double qnl, double qtl, double hr, double qnr, double qtr, double g,
             double hdry, double* out3) {
  const Flux f = hll(hl, qnl, qtl, hr, qnr, qtr, g, hdry);
  out3[0] = f.m;
  out3[1] = f.n;
  out3[2] = f.t;
}
void orc_friction(double h0, double* qx3, double* qy3, double n, double g, double hdry, double dt) {
  Pl a{qx3[0], qx3[1], qx3[2]}, b{qy3[0], qy3[1], qy3[2]};
  friction(h0, a, b, n, g, hdry, dt);
  qx3[0] = a.c0;
  qy3[0] = b.c0;
  qx3[1] = a.cx;
  qx3[2] = a.cy;
  qy3[1] = b.cx;
  qy3[2] = b.cy;
}
double orc_pcbrt(double x) { return pcbrt(x); }

// detail_tree.cpp:56-64 then :97-113 on caller flags (levels back to back).
int orc_grade_flags(int32_t L, int32_t M, int32_t N, int32_t graded, uint8_t* flags) {
  return guard([&] {
    Tree t;
    t.L = L;
    t.M = M;
    t.N = N;
    t.flag.resize(L);
    size_t at = 0;
    for (int l = 0; l < L; ++l) {
      const size_t n = size_t(t.w(l)) * t.h(l);
      t.flag[l].assign(flags + at, flags + at + n);
      at += n;
    }
    closure(t);
    if (graded) grade(t);
    at = 0;
    for (int l = 0; l < L; ++l) {
      std::memcpy(flags + at, t.flag[l].data(), t.flag[l].size());
      at += t.flag[l].size();
    }
  });
}
void orc_encode(const double* kids12, int32_t kind, double* parent3, double* det9) {
  Pl k[4];
  for (int c = 0; c < 4; ++c) k[c] = {kids12[3 * c], kids12[3 * c + 1], kids12[3 * c + 2]};
  Pl p;
  Det d;
  enc(k, kind, p, d);
  parent3[0] = p.c0;
  parent3[1] = p.cx;
  parent3[2] = p.cy;
  std::memcpy(det9, d.v, sizeof(d.v));
}
void orc_decode(const double* parent3, const double* det9, int32_t kind, double* kids12) {
  Pl p{parent3[0], parent3[1], parent3[2]}, k[4];
  Det d;
  std::memcpy(d.v, det9, sizeof(d.v));
  dec(p, d, kind, k);
  for (int c = 0; c < 4; ++c) {
    kids12[3 * c] = k[c].c0;
    kids12[3 * c + 1] = k[c].cx;
    kids12[3 * c + 2] = k[c].cy;
  }
}
void orc_bank(int32_t kind, double* out144) { std::memcpy(out144, bank(kind), sizeof(double) * 144); }

}  // extern "C"
