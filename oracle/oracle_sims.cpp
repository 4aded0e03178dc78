// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle_core.hpp).
// Restatement of solver_nonuniform.cpp, solver_adaptive.cpp and
// solver_uniform.cpp arithmetic.
#include "oracle_sims.hpp"

#include <algorithm>
#include <limits>
#include <map>

namespace orc {

namespace {
constexpr double kK = 1.0 / (2.0 * kS3);  // solver_nonuniform.cpp:48

// solver_nonuniform.cpp:18-46 (same in solver_uniform.cpp:28-57)
inline void pfx(double h, double qx, double qy, double g, double hd, double& a, double& b,
                double& c) {
  const double p = 0.5 * g * h * h;
  if (h <= hd) {
    a = 0.0;
    b = p;
    c = 0.0;
    return;
  }
  const double u = qx / h;
  a = qx;
  b = qx * u + p;
  c = qx * (qy / h);
}
inline void pfy(double h, double qx, double qy, double g, double hd, double& a, double& b,
                double& c) {
  const double p = 0.5 * g * h * h;
  if (h <= hd) {
    a = 0.0;
    b = 0.0;
    c = p;
    return;
  }
  const double v = qy / h;
  a = qy;
  b = qy * (qx / h);
  c = qy * v + p;
}
inline double vel(double h, double q, double hd) { return h > hd ? q / h : 0.0; }  // sim_common.hpp:20-22

struct Pt {
  double h, qx, qy, z, eta, u, v;
};

// The L operator shared by the static non-uniform and uniform DG2/FV1
// assemblies (solver_nonuniform.cpp:228-271, solver_uniform.cpp:199-227).
struct DirM {
  double h0, h1, qx0, qx1, qy0, qy1, z1;
};
Fl l_operator(const Flux& fn, const Flux& fe, const Flux& fs, const Flux& fw, const DirM& X,
              const DirM& Y, double sz, double g, double hd, bool dg2) {
  Fl L{};
  L.h.c0 = -((fe.m - fw.m) + (fn.m - fs.m)) / sz;
  L.qx.c0 = -((fe.n - fw.n) + (fn.t - fs.t)) / sz - g * X.h0 * (2.0 * kS3 * X.z1) / sz;
  L.qy.c0 = -((fe.t - fw.t) + (fn.n - fs.n)) / sz - g * Y.h0 * (2.0 * kS3 * Y.z1) / sz;
  if (dg2) {
    double a, b, c, d, e, f;
    pfx(X.h0 + X.h1, X.qx0 + X.qx1, X.qy0 + X.qy1, g, hd, a, b, c);
    pfx(X.h0 - X.h1, X.qx0 - X.qx1, X.qy0 - X.qy1, g, hd, d, e, f);
    L.h.cx = -(kS3 / sz) * (fe.m + fw.m - a - d);
    L.qx.cx = -(kS3 / sz) * (fe.n + fw.n - b - e) - g * X.h1 * (2.0 * kS3 * X.z1) / sz;
    L.qy.cx = -(kS3 / sz) * (fe.t + fw.t - c - f);
    pfy(Y.h0 + Y.h1, Y.qx0 + Y.qx1, Y.qy0 + Y.qy1, g, hd, a, b, c);
    pfy(Y.h0 - Y.h1, Y.qx0 - Y.qx1, Y.qy0 - Y.qy1, g, hd, d, e, f);
    L.h.cy = -(kS3 / sz) * (fn.m + fs.m - a - d);
    L.qx.cy = -(kS3 / sz) * (fn.t + fs.t - b - e);
    L.qy.cy = -(kS3 / sz) * (fn.n + fs.n - c - f) - g * Y.h1 * (2.0 * kS3 * Y.z1) / sz;
  }
  return L;
}

// FlowCoeffs arithmetic of step_rk (solver_nonuniform.cpp:317-347).
inline void axpy_stage(const Fl& u, const Fl& r, double dt, Fl& out) {
  const double* pu = &u.h.c0;
  const double* pr = &r.h.c0;
  double* po = &out.h.c0;
  for (int n = 0; n < 9; ++n) po[n] = pu[n] + pr[n] * dt;
}
inline void rk2_final(const Fl& st, const Fl& r, const Fl& u, double dt, Fl& out) {
  const double* ps = &st.h.c0;
  const double* pr = &r.h.c0;
  const double* pu = &u.h.c0;
  double* po = &out.h.c0;
  for (int n = 0; n < 9; ++n) {
    double s = ps[n];
    s += pr[n] * dt;
    s += pu[n];
    s *= 0.5;
    po[n] = s;
  }
}

bool fl_finite(const Fl& f) {
  const double* p = &f.h.c0;
  for (int n = 0; n < 9; ++n)
    if (!std::isfinite(p[n])) return false;
  return true;
}

// Manning lookup (solver_nonuniform.cpp:575-584, solver_adaptive.cpp:175-185)
double manning_at(const Raster& mr, double xc, double yc) {
  const int col = std::clamp(int((xc - mr.xll) / mr.cell), 0, mr.ncols - 1);
  const int row = std::clamp(mr.nrows - 1 - int((yc - mr.yll) / mr.cell), 0, mr.nrows - 1);
  return mr.at(row, col);
}

// Inflow target resolution against a leaf grid (solver_nonuniform.cpp:611-628).
Inflow resolve_leaf_inflow(const Grid& g, const Inflow& spec) {
  Inflow f = spec;
  f.targets.clear();
  f.region = 0;
  std::map<int32_t, int32_t> counts;  // sorted by leaf index
  for (int j = spec.j0; j <= spec.j1; ++j)
    for (int i = spec.i0; i <= spec.i1; ++i) {
      const int k = g.containing(i, j);
      if (k < 0) throw Fail(E_STRUCT, "inflow cell not covered by any leaf");
      counts[k] += 1;
      f.region += 1;
    }
  f.targets.assign(counts.begin(), counts.end());
  return f;
}
}  // namespace

double Cfg::courant_for() const {
  if (courant > 0.0) return courant;
  switch (solver) {
    case S_DG2:
    case S_MWDG2: return 0.33;
    case S_FV1:
    case S_HWFV1: return 0.5;
    case S_ACC: return 0.7;
  }
  return 0.33;
}

// ======================= NonUniformSim ===================================

// solver_nonuniform.cpp:80-89
Pl NU::region_topo(int l, int i, int j) const {
  const int k = grid.find(l, i, j);
  if (k >= 0) return z[k];
  Pl kids[4];
  for (int c = 0; c < 4; ++c) kids[c] = region_topo(l + 1, 2 * i + (c & 1), 2 * j + (c >> 1));
  Pl p;
  Det d;
  enc(kids, pairing, p, d);
  return p;
}

// solver_nonuniform.cpp:91-115 with limit_at (:52-66) inlined.
void NU::seg_pass(const std::vector<Fl>& s) {
  seg.resize(F.in.size());
  auto lim = [&](int k, double x, double y) {
    const double cx = grid.xc(k), cy = grid.yc(k), sz = grid.size(k);
    Pt p;
    p.h = mx(0.0, eval_plane(s[k].h, cx, cy, sz, x, y));
    p.qx = eval_plane(s[k].qx, cx, cy, sz, x, y);
    p.qy = eval_plane(s[k].qy, cx, cy, sz, x, y);
    p.z = eval_plane(z[k], cx, cy, sz, x, y);
    p.eta = p.h + p.z;
    p.u = vel(p.h, p.qx, hdry);
    p.v = vel(p.h, p.qy, hdry);
    return p;
  };
  for (size_t q = 0; q < F.in.size(); ++q) {
    const Seg& e = F.in[q];
    const Pt a = lim(e.l, e.cx, e.cy), b = lim(e.r, e.cx, e.cy);
    const double zs = mx(a.z, b.z);
    const double hl = mx(0.0, a.eta - zs), hr = mx(0.0, b.eta - zs);
    SegS o;
    o.zs = zs;
    o.hl = hl;
    o.hr = hr;
    o.f = e.xn ? hll(hl, hl * a.u, hl * a.v, hr, hr * b.u, hr * b.v, g, hdry)
               : hll(hl, hl * a.v, hl * a.u, hr, hr * b.v, hr * b.u, g, hdry);
    seg[q] = o;
  }
}

// solver_nonuniform.cpp:117-178 (the encode_cache_ fill at :121-135 is never
// read and is skipped).
void NU::side_pass(const std::vector<Fl>& s) {
  const int n = int(grid.lv.size());
  sd.resize(size_t(n) * 4);
  for (int k = 0; k < n; ++k) {
    const Leaf& f = grid.lv[k];
    const double sz = grid.size(k), cx = grid.xc(k), cy = grid.yc(k);
    for (int side = 0; side < 4; ++side) {
      const double fx = cx + (side == 1 ? sz / 2 : side == 3 ? -sz / 2 : 0.0);
      const double fy = cy + (side == 0 ? sz / 2 : side == 2 ? -sz / 2 : 0.0);
      Pt me;
      me.h = mx(0.0, eval_plane(s[k].h, cx, cy, sz, fx, fy));
      me.qx = eval_plane(s[k].qx, cx, cy, sz, fx, fy);
      me.qy = eval_plane(s[k].qy, cx, cy, sz, fx, fy);
      me.z = eval_plane(z[k], cx, cy, sz, fx, fy);
      me.eta = me.h + me.z;
      me.u = vel(me.h, me.qx, hdry);
      me.v = vel(me.h, me.qy, hdry);
      const auto& L = F.sides[size_t(k) * 4 + side];
      SideS e;
      if (L.size() == 1 && L[0] < 0) {
        e.zs = me.z;
      } else if (L.size() == 1) {
        e.zs = seg[L[0]].zs;
      } else if (pairing >= 0) {
        const int ni = f.i + (side == 1 ? 1 : side == 3 ? -1 : 0);
        const int nj = f.j + (side == 0 ? 1 : side == 2 ? -1 : 0);
        const Pl zt = region_topo(f.l, ni, nj);
        e.zs = mx(me.z, face_val(zt, (side + 2) & 3));
      } else {
        double acc = 0.0;
        for (int id : L) acc += (F.in[id].len / sz) * seg[id].zs;
        e.zs = acc;
      }
      e.h = mx(0.0, me.eta - e.zs);
      e.qx = e.h * me.u;
      e.qy = e.h * me.v;
      e.zd = e.zs - mx(0.0, e.zs - me.eta);
      sd[size_t(k) * 4 + side] = e;
    }
  }
}

// solver_nonuniform.cpp:180-274
void NU::rate_pass() {
  const int n = int(grid.lv.size());
  rate.resize(n);
  const bool dg2 = scheme == S_DG2;
  for (int k = 0; k < n; ++k) {
    const double sz = grid.size(k);
    Flux fs[4];
    for (int side = 0; side < 4; ++side) {
      const SideS& e = sd[size_t(k) * 4 + side];
      Flux acc;
      for (int id : F.sides[size_t(k) * 4 + side]) {
        if (id < 0) {
          const bool xn = (side == 1 || side == 3);
          const double qn = xn ? e.qx : e.qy, qt = xn ? e.qy : e.qx;
          const double qg = bc[side] == 0 ? -qn : qn;
          const Flux f = (side == 1 || side == 0) ? hll(e.h, qn, qt, e.h, qg, qt, g, hdry)
                                                  : hll(e.h, qg, qt, e.h, qn, qt, g, hdry);
          acc.m += f.m;
          acc.n += f.n;
          acc.t += f.t;
          continue;
        }
        const Seg& q = F.in[id];
        const SegS& ss = seg[id];
        const double w = q.len / sz;
        const double hme = (side == 1 || side == 0) ? ss.hl : ss.hr;
        const double corr = 0.5 * g * (e.h * e.h - hme * hme);
        acc.m += w * ss.f.m;
        acc.n += w * (ss.f.n + corr);
        acc.t += w * ss.f.t;
      }
      fs[side] = acc;
    }
    const SideS& en = sd[size_t(k) * 4 + 0];
    const SideS& ee = sd[size_t(k) * 4 + 1];
    const SideS& es = sd[size_t(k) * 4 + 2];
    const SideS& ew = sd[size_t(k) * 4 + 3];
    const DirM X = {0.5 * (ee.h + ew.h),   (ee.h - ew.h) * kK,   0.5 * (ee.qx + ew.qx),
                  (ee.qx - ew.qx) * kK,  0.5 * (ee.qy + ew.qy), (ee.qy - ew.qy) * kK,
                  (ee.zd - ew.zd) * kK};
    const DirM Y = {0.5 * (en.h + es.h),   (en.h - es.h) * kK,   0.5 * (en.qx + es.qx),
                  (en.qx - es.qx) * kK,  0.5 * (en.qy + es.qy), (en.qy - es.qy) * kK,
                  (en.zd - es.zd) * kK};
    rate[k] = l_operator(fs[0], fs[1], fs[2], fs[3], X, Y, sz, g, hdry, dg2);
  }
}

// solver_nonuniform.cpp:306-348
void NU::step_rk(double dt) {
  const size_t n = u.size();
  for (size_t c = 0; c < n; ++c) friction(u[c].h.c0, u[c].qx, u[c].qy, nman[c], g, hdry, dt, libm);
  seg_pass(u);
  side_pass(u);
  rate_pass();
  stage.resize(n);
  for (size_t c = 0; c < n; ++c) {
    axpy_stage(u[c], rate[c], dt, stage[c]);
    positivity(stage[c], hdry);
  }
  if (scheme != S_DG2) {
    u.swap(stage);
    return;
  }
  seg_pass(stage);
  side_pass(stage);
  rate_pass();
  for (size_t c = 0; c < n; ++c) {
    rk2_final(stage[c], rate[c], u[c], dt, u[c]);
    positivity(u[c], hdry);
  }
}

// solver_nonuniform.cpp:350-418
void NU::step_acc(double dt) {
  for (size_t q = 0; q < F.in.size(); ++q) {
    const Seg& e = F.in[q];
    const int l = e.l, r = e.r;
    const double el = u[l].h.c0 + z[l].c0, er = u[r].h.c0 + z[r].c0;
    const double hf = mx(el, er) - mx(z[l].c0, z[r].c0);
    double& Q = accq[q];
    if (hf <= hdry) {
      Q = 0.0;
      continue;
    }
    const double dist = 0.5 * (grid.size(l) + grid.size(r));
    const double nf = 0.5 * (nman[l] + nman[r]);
    Q = (Q - g * hf * dt * (er - el) / dist) /
        (1.0 + g * dt * nf * nf * std::abs(Q) / pow73_m(hf, libm));
  }
  for (size_t q = 0; q < F.bd.size(); ++q) {
    const BSeg& b = F.bd[q];
    double& Q = accqb[q];
    if (bc[b.side] == 0) {
      Q = 0.0;
      continue;
    }
    const double hf = u[b.leaf].h.c0;
    if (hf <= hdry) {
      Q = 0.0;
      continue;
    }
    const double nf = nman[b.leaf];
    Q = Q / (1.0 + g * dt * nf * nf * std::abs(Q) / pow73_m(hf, libm));
  }
  for (int k = 0; k < int(grid.lv.size()); ++k) {
    const double sz = grid.size(k), area = sz * sz;
    double net = 0.0, sx = 0.0, sy = 0.0;
    for (int side = 0; side < 4; ++side) {
      const double sign = (side == 1 || side == 0) ? -1.0 : 1.0;
      for (int id : F.sides[size_t(k) * 4 + side]) {
        const double Q = id >= 0 ? accq[id] : accqb[-1 - id];
        const double len = id >= 0 ? F.in[id].len : F.bd[-1 - id].len;
        net += sign * Q * len;
        if (side == 1 || side == 3)
          sx += Q * len;
        else
          sy += Q * len;
      }
    }
    u[k].h.c0 += dt * net / area;
    u[k].qx.c0 = 0.5 * sx / sz;
    u[k].qy.c0 = 0.5 * sy / sz;
  }
}

void NU::step(double dt) {
  if (scheme == S_ACC)
    step_acc(dt);
  else
    step_rk(dt);
}

// solver_nonuniform.cpp:427-449
double NU::compute_dt() const {
  const double inf = std::numeric_limits<double>::infinity();
  if (scheme == S_ACC) {
    double hmax = 0.0, rmin = inf;
    for (size_t c = 0; c < u.size(); ++c) {
      if (u[c].h.c0 <= hdry) continue;
      hmax = mx(hmax, u[c].h.c0);
      rmin = mn(rmin, grid.size(int(c)));
    }
    if (hmax <= hdry) return inf;
    return cour * rmin / std::sqrt(g * hmax);
  }
  double dt = inf;
  for (size_t c = 0; c < u.size(); ++c) {
    const double h = u[c].h.c0;
    if (h <= hdry) continue;
    const double cw = std::sqrt(g * h);
    const double sx = std::abs(u[c].qx.c0 / h) + cw;
    const double sy = std::abs(u[c].qy.c0 / h) + cw;
    dt = mn(dt, grid.size(int(c)) / mx(sx, sy));
  }
  return dt * cour;
}

// solver_nonuniform.cpp:451-465
double NU::apply_inflows(double t, double dt) {
  double added = 0.0;
  for (const Inflow& f : inflows) {
    const double q = hydro_at(f.hy, t);
    if (q <= 0.0) continue;
    const double vol = q * dt;
    const double per = vol / double(f.region);
    for (const auto& [k, cnt] : f.targets) {
      const double area = grid.size(k) * grid.size(k);
      u[k].h.c0 += per * cnt / area;
    }
    added += vol;
  }
  return added;
}

// solver_nonuniform.cpp:467-477 (Kahan)
double NU::volume() const {
  double sum = 0.0, comp = 0.0;
  for (size_t c = 0; c < u.size(); ++c) {
    const double sz = grid.size(int(c));
    const double y = u[c].h.c0 * sz * sz - comp;
    const double t = sum + y;
    comp = (t - sum) - y;
    sum = t;
  }
  return sum;
}

bool NU::finite(double* bx, double* by) const {
  for (size_t c = 0; c < u.size(); ++c)
    if (!fl_finite(u[c])) {
      if (bx) *bx = grid.xc(int(c));
      if (by) *by = grid.yc(int(c));
      return false;
    }
  return true;
}

// solver_nonuniform.cpp:521-527
void NU::rebuild() {
  F = faces_of(grid, true);
  if (scheme == S_ACC) {
    accq.assign(F.in.size(), 0.0);
    accqb.assign(F.bd.size(), 0.0);
  }
}

// solver_nonuniform.cpp:529-556
std::vector<Fl> restrict_to_leaves(const Grid& g, const std::vector<Fl>& fine, int kind) {
  std::vector<Fl> out(g.lv.size());
  std::vector<Fl> cur = fine, up;
  int w = g.M << g.L;
  for (int l = g.L; l >= 0; --l) {
    for (size_t k = 0; k < g.lv.size(); ++k)
      if (g.lv[k].l == l) out[k] = cur[size_t(g.lv[k].j) * w + g.lv[k].i];
    if (l == 0) break;
    const int cw = w / 2, ch = g.N << (l - 1);
    up.assign(size_t(cw) * ch, Fl{});
    for (int j = 0; j < ch; ++j)
      for (int i = 0; i < cw; ++i) {
        const size_t s = size_t(2 * j) * w + 2 * i, n = s + w;
        const Fl* kids[4] = {&cur[s], &cur[s + 1], &cur[n], &cur[n + 1]};
        Pl a[4], b[4], c[4];
        for (int q = 0; q < 4; ++q) {
          a[q] = kids[q]->h;
          b[q] = kids[q]->qx;
          c[q] = kids[q]->qy;
        }
        Det d;
        Fl& o = up[size_t(j) * cw + i];
        enc(a, kind, o.h, d);
        enc(b, kind, o.qx, d);
        enc(c, kind, o.qy, d);
      }
    cur.swap(up);
    w = cw;
  }
  return out;
}

// solver_uniform.cpp:60-71
Fl from_surface(const Pl& z, double eta0) {
  Fl f;
  const double span = kS3 * (std::abs(z.cx) + std::abs(z.cy));
  if (z.c0 + span < eta0)
    f.h = {eta0 - z.c0, -z.cx, -z.cy};
  else if (z.c0 - span >= eta0)
    f.h = {};
  else
    f.h = {mx(0.0, eta0 - z.c0), 0.0, 0.0};
  return f;
}

// solver_nonuniform.cpp:558-636
NU make_nu(const Cfg& c, const Raster& dem, const Grid& grid, const std::vector<Pl>& topo) {
  NU s;
  s.scheme = c.solver == S_MWDG2 ? S_DG2 : c.solver == S_HWFV1 ? S_FV1 : c.solver;
  s.libm = c.libm;
  s.grid = grid;
  s.z = topo;
  if (!graded(s.grid)) throw Fail(E_STRUCT, "non-uniform solvers require a graded (2:1) grid");
  s.g = c.g;
  s.hdry = c.hdry;
  s.cour = c.courant_for();
  for (int q = 0; q < 4; ++q) s.bc[q] = c.bc[q];
  const size_t n = s.grid.lv.size();
  s.nman.assign(n, c.manning);
  if (c.has_mr)
    for (size_t k = 0; k < n; ++k) s.nman[k] = manning_at(c.mr, s.grid.xc(int(k)), s.grid.yc(int(k)));
  s.u.assign(n, Fl{});
  if (c.has_h0) {
    if (c.h0.ncols != dem.ncols || c.h0.nrows != dem.nrows)
      throw Fail(E_CONFIG, "initial_depth_raster geometry must match the DEM");
    const Field hf = project_padded(c.h0, s.grid.L, nullptr, nullptr);
    std::vector<Fl> fine(hf.c.size());
    for (size_t q = 0; q < hf.c.size(); ++q) fine[q].h = hf.c[q];
    s.u = restrict_to_leaves(s.grid, fine, 0);
  } else if (c.has_eta0) {
    for (size_t k = 0; k < n; ++k) s.u[k] = from_surface(s.z[k], c.eta0);
  } else if (c.depth0 > 0.0) {
    for (size_t k = 0; k < n; ++k) s.u[k].h = {c.depth0, 0.0, 0.0};
  }
  if (s.scheme != S_DG2)
    for (size_t k = 0; k < n; ++k) {
      s.z[k].cx = s.z[k].cy = 0.0;
      s.u[k].h.cx = s.u[k].h.cy = 0.0;
      s.u[k].qx = {};
      s.u[k].qy = {};
    }
  for (Fl& f : s.u) positivity(f, s.hdry);
  for (const Inflow& spec : c.inflows) {
    if (spec.i0 < 0 || spec.j0 < 0 || spec.i1 >= (s.grid.M << s.grid.L) ||
        spec.j1 >= (s.grid.N << s.grid.L))
      throw Fail(E_CONFIG, "inflow region outside the domain");
    s.inflows.push_back(resolve_leaf_inflow(s.grid, spec));
  }
  s.rebuild();
  return s;
}

// ======================= AdaptiveSim =====================================

// solver_adaptive.cpp:16-57
void AD::encode_up() {
  const int L = zt.L;
  lev.resize(L + 1);
  for (int l = 0; l <= L; ++l) {
    const size_t n = size_t(zt.w(l)) * zt.h(l);
    lev[l].sc.assign(n, Fl{});
    lev[l].known.assign(n, 0);
    if (l < L) {
      lev[l].dh.assign(n, Det{});
      lev[l].dqx.assign(n, Det{});
      lev[l].dqy.assign(n, Det{});
    }
  }
  for (size_t k = 0; k < sim.grid.lv.size(); ++k) {
    const Leaf& f = sim.grid.lv[k];
    const size_t nd = zt.node(f.l, f.i, f.j);
    lev[f.l].sc[nd] = sim.u[k];
    lev[f.l].known[nd] = 1;
  }
  for (int l = L - 1; l >= 0; --l) {
    const int w = zt.w(l), h = zt.h(l), cw = 2 * w;
    for (int j = 0; j < h; ++j)
      for (int i = 0; i < w; ++i) {
        const size_t nd = zt.node(l, i, j);
        if (lev[l].known[nd] != 0) continue;
        const size_t k0 = size_t(2 * j) * cw + 2 * i, k2 = k0 + cw;
        const auto& kn = lev[l + 1].known;
        if (!(kn[k0] && kn[k0 + 1] && kn[k2] && kn[k2 + 1])) continue;
        const auto& sc = lev[l + 1].sc;
        const Fl* kids[4] = {&sc[k0], &sc[k0 + 1], &sc[k2], &sc[k2 + 1]};
        Pl a[4], b[4], c[4];
        for (int q = 0; q < 4; ++q) {
          a[q] = kids[q]->h;
          b[q] = kids[q]->qx;
          c[q] = kids[q]->qy;
        }
        Fl& p = lev[l].sc[nd];
        enc(a, kind, p.h, lev[l].dh[nd]);
        enc(b, kind, p.qx, lev[l].dqx[nd]);
        enc(c, kind, p.qy, lev[l].dqy[nd]);
        lev[l].known[nd] = 2;
      }
  }
}

// solver_adaptive.cpp:59-73
void AD::flag(double nh, double nqx, double nqy) {
  for (int l = 0; l < zt.L; ++l)
    for (size_t k = 0; k < zt.det[l].size(); ++k) {
      double d = dhat(zt.det[l][k], zt.norm);
      if (lev[l].known[k] == 2) {
        d = mx(d, dhat(lev[l].dh[k], nh));
        d = mx(d, dhat(lev[l].dqx[k], nqx));
        d = mx(d, dhat(lev[l].dqy[k], nqy));
      }
      zt.flag[l][k] = d >= eps;
    }
  closure(zt);
}

// solver_adaptive.cpp:75-94
void AD::ring() {
  for (int l = 0; l < zt.L; ++l) {
    const int w = zt.w(l), h = zt.h(l);
    std::vector<uint8_t> extra(zt.flag[l].size(), 0);
    for (int j = 0; j < h; ++j)
      for (int i = 0; i < w; ++i) {
        if (!zt.flag[l][zt.node(l, i, j)]) continue;
        for (int dj = -1; dj <= 1; ++dj)
          for (int di = -1; di <= 1; ++di) {
            const int ni = i + di, nj = j + dj;
            if (ni < 0 || nj < 0 || ni >= w || nj >= h) continue;
            extra[zt.node(l, ni, nj)] = 1;
          }
      }
    for (size_t k = 0; k < extra.size(); ++k)
      if (extra[k]) zt.flag[l][k] = 1;
  }
  closure(zt);
}

// solver_adaptive.cpp:96-134 — top-down per level (each leaf's value depends
// only on its ancestor chain, as in the DFS).
std::vector<Fl> AD::transfer(const Grid& ng) const {
  std::vector<Fl> out(ng.lv.size());
  std::vector<Fl> cur(size_t(zt.M) * zt.N), nxt;
  for (size_t q = 0; q < cur.size(); ++q) cur[q] = lev[0].sc[q];
  for (int l = 0; l <= zt.L; ++l) {
    const int w = zt.w(l), h = zt.h(l);
    if (l < zt.L) nxt.assign(size_t(4) * w * h, Fl{});
    for (int j = 0; j < h; ++j)
      for (int i = 0; i < w; ++i) {
        const bool active = l == 0 || zt.flag[l - 1][zt.node(l - 1, i / 2, j / 2)];
        if (!active) continue;
        const Fl& v = cur[size_t(j) * w + i];
        if (l == zt.L || !zt.flag[l][zt.node(l, i, j)]) {
          const int k = ng.find(l, i, j);
          if (k < 0) throw Fail(E_STRUCT, "adaptive transfer: leaf set does not match flags");
          const int old = sim.grid.find(l, i, j);
          out[k] = old >= 0 ? sim.u[old] : v;
          continue;
        }
        const size_t nd = zt.node(l, i, j);
        const bool in = lev[l].known[nd] == 2;
        const Det zero{};
        Pl a[4], b[4], c[4];
        dec(v.h, in ? lev[l].dh[nd] : zero, kind, a);
        dec(v.qx, in ? lev[l].dqx[nd] : zero, kind, b);
        dec(v.qy, in ? lev[l].dqy[nd] : zero, kind, c);
        for (int q = 0; q < 4; ++q) {
          Fl& o = nxt[size_t(2 * j + (q >> 1)) * (2 * w) + 2 * i + (q & 1)];
          o.h = a[q];
          o.qx = b[q];
          o.qy = c[q];
        }
      }
    cur.swap(nxt);
  }
  return out;
}

// solver_adaptive.cpp:173-202
void AD::remap() {
  const size_t n = sim.grid.lv.size();
  sim.nman.assign(n, man);
  if (has_mr)
    for (size_t k = 0; k < n; ++k) sim.nman[k] = manning_at(mr, sim.grid.xc(int(k)), sim.grid.yc(int(k)));
  sim.inflows.clear();
  for (const Inflow& r : raw) sim.inflows.push_back(resolve_leaf_inflow(sim.grid, r));
}

// solver_adaptive.cpp:136-171
void AD::adapt(double t) {
  encode_up();
  double nh = 0.0, nqx = 0.0, nqy = 0.0;
  for (const Fl& f : sim.u) {
    nh = mx(nh, std::abs(f.h.c0));
    nqx = mx(nqx, std::abs(f.qx.c0));
    nqy = mx(nqy, std::abs(f.qy.c0));
  }
  flag(nh, nqx, nqy);
  ring();
  grade(zt);
  Grid ng = make_grid(zt.L, zt.M, zt.N, zt.R, zt.x0, zt.y0, tree_leaves(zt));
  std::vector<Pl> topo;
  tree_decode(zt, ng, topo);
  std::vector<Fl> nu = transfer(ng);
  sim.grid = std::move(ng);
  sim.z = std::move(topo);
  sim.u = std::move(nu);
  if (sim.scheme != S_DG2)
    for (size_t k = 0; k < sim.u.size(); ++k) {
      sim.z[k].cx = sim.z[k].cy = 0.0;
      sim.u[k].h.cx = sim.u[k].h.cy = 0.0;
      sim.u[k].qx.cx = sim.u[k].qx.cy = 0.0;
      sim.u[k].qy.cx = sim.u[k].qy.cy = 0.0;
    }
  remap();
  sim.rebuild();
  log.emplace_back(t, int64_t(sim.grid.lv.size()));
}

// solver_adaptive.cpp:209-236
AD make_ad(const Cfg& c, const Raster& dem) {
  if (c.solver != S_MWDG2 && c.solver != S_HWFV1)
    throw Fail(E_CONFIG, "adaptive sim requires solver mwdg2 or hwfv1");
  AD a;
  a.kind = c.solver == S_MWDG2 ? 0 : 1;
  a.eps = c.eps;
  a.adapt_every = c.adapt_every;
  int M = 0, N = 0;
  const Field fine = project_padded(dem, c.L, &M, &N);
  a.zt = encode_tree(fine, c.L, M, N, a.kind);
  std::vector<Leaf> leaves;
  leaves.reserve(size_t(M << c.L) * size_t(N << c.L));
  for (int j = 0; j < (N << c.L); ++j)
    for (int i = 0; i < (M << c.L); ++i) leaves.push_back({c.L, i, j});
  const Grid g0 = make_grid(c.L, M, N, fine.R, fine.x0, fine.y0, std::move(leaves));
  a.sim = make_nu(c, dem, g0, fine.c);
  a.sim.pairing = a.kind;
  a.man = c.manning;
  a.has_mr = c.has_mr;
  if (c.has_mr) a.mr = c.mr;
  for (size_t k = 0; k < c.inflows.size(); ++k) {
    Inflow r = c.inflows[k];
    r.hy = a.sim.inflows[k].hy;
    a.raw.push_back(r);
  }
  a.adapt(0.0);
  return a;
}

// ======================= UniformSim ======================================

// solver_uniform.cpp:73-137
void UN::revise(const std::vector<Fl>& s) {
  const size_t n = s.size();
  se.resize(n);
  sw.resize(n);
  sn.resize(n);
  ss.resize(n);
  dmx.resize(n);
  dmy.resize(n);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const size_t c = cell(i, j);
      const Fl& uc = s[c];
      Pt lim[4];
      for (int side = 0; side < 4; ++side) {
        Pt& p = lim[side];
        p.h = mx(0.0, face_val(uc.h, side));
        p.qx = face_val(uc.qx, side);
        p.qy = face_val(uc.qy, side);
        p.z = face_val(z[c], side);
        p.eta = p.h + p.z;
        p.u = vel(p.h, p.qx, hdry);
        p.v = vel(p.h, p.qy, hdry);
      }
      const Pt &ln = lim[0], &le = lim[1], &ls = lim[2], &lw = lim[3];
      const double zwe = i + 1 < nx ? face_val(z[cell(i + 1, j)], 3) : le.z;
      const double zew = i > 0 ? face_val(z[cell(i - 1, j)], 1) : lw.z;
      const double zsn = j + 1 < ny ? face_val(z[cell(i, j + 1)], 2) : ln.z;
      const double zns = j > 0 ? face_val(z[cell(i, j - 1)], 0) : ls.z;
      const double zse = mx(le.z, zwe), zsw = mx(lw.z, zew), zsn2 = mx(ln.z, zsn),
                   zss = mx(ls.z, zns);
      const double he = mx(0.0, le.eta - zse), hw = mx(0.0, lw.eta - zsw),
                   hn = mx(0.0, ln.eta - zsn2), hs = mx(0.0, ls.eta - zss);
      se[c] = {he, he * le.u, he * le.v};
      sw[c] = {hw, hw * lw.u, hw * lw.v};
      sn[c] = {hn, hn * ln.u, hn * ln.v};
      ss[c] = {hs, hs * ls.u, hs * ls.v};
      const double de = zse - mx(0.0, zse - le.eta), dw = zsw - mx(0.0, zsw - lw.eta),
                   dn = zsn2 - mx(0.0, zsn2 - ln.eta), ds = zss - mx(0.0, zss - ls.eta);
      dmx[c] = {0.5 * (he + hw),         (he - hw) * kK,
                0.5 * (se[c].qx + sw[c].qx), (se[c].qx - sw[c].qx) * kK,
                0.5 * (se[c].qy + sw[c].qy), (se[c].qy - sw[c].qy) * kK,
                (de - dw) * kK};
      dmy[c] = {0.5 * (hn + hs),         (hn - hs) * kK,
                0.5 * (sn[c].qx + ss[c].qx), (sn[c].qx - ss[c].qx) * kK,
                0.5 * (sn[c].qy + ss[c].qy), (sn[c].qy - ss[c].qy) * kK,
                (dn - ds) * kK};
    }
}

// solver_uniform.cpp:139-185
void UN::fluxes() {
  fx.resize(size_t(nx + 1) * ny);
  fy.resize(size_t(nx) * (ny + 1));
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i <= nx; ++i) {
      St l, r;
      if (i == 0) {
        r = sw[cell(0, j)];
        l = r;
        if (bc[3] == 0) l.qx = -l.qx;
      } else if (i == nx) {
        l = se[cell(nx - 1, j)];
        r = l;
        if (bc[1] == 0) r.qx = -r.qx;
      } else {
        l = se[cell(i - 1, j)];
        r = sw[cell(i, j)];
      }
      fx[size_t(j) * (nx + 1) + i] = hll(l.h, l.qx, l.qy, r.h, r.qx, r.qy, g, hdry);
    }
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i < nx; ++i) {
      St l, r;
      if (j == 0) {
        r = ss[cell(i, 0)];
        l = r;
        if (bc[2] == 0) l.qy = -l.qy;
      } else if (j == ny) {
        l = sn[cell(i, ny - 1)];
        r = l;
        if (bc[0] == 0) r.qy = -r.qy;
      } else {
        l = sn[cell(i, j - 1)];
        r = ss[cell(i, j)];
      }
      fy[size_t(j) * nx + i] = hll(l.h, l.qy, l.qx, r.h, r.qy, r.qx, g, hdry);
    }
}

// solver_uniform.cpp:187-251
void UN::assemble(bool dg2) {
  rate.resize(size_t(nx) * ny);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const size_t c = cell(i, j);
      const Flux& fe = fx[size_t(j) * (nx + 1) + i + 1];
      const Flux& fw = fx[size_t(j) * (nx + 1) + i];
      const Flux& fn = fy[size_t(j + 1) * nx + i];
      const Flux& fs = fy[size_t(j) * nx + i];
      const DirM X = {dmx[c].h0, dmx[c].h1, dmx[c].qx0, dmx[c].qx1, dmx[c].qy0, dmx[c].qy1, dmx[c].z1};
      const DirM Y = {dmy[c].h0, dmy[c].h1, dmy[c].qx0, dmy[c].qx1, dmy[c].qy0, dmy[c].qy1, dmy[c].z1};
      rate[c] = l_operator(fn, fe, fs, fw, X, Y, R, g, hdry, dg2);
    }
}

// solver_uniform.cpp:283-328
void UN::step_rk(double dt) {
  const size_t n = u.size();
  for (size_t c = 0; c < n; ++c) friction(u[c].h.c0, u[c].qx, u[c].qy, nman[c], g, hdry, dt, libm);
  revise(u);
  fluxes();
  assemble(kind == S_DG2);
  stage.resize(n);
  for (size_t c = 0; c < n; ++c) {
    axpy_stage(u[c], rate[c], dt, stage[c]);
    positivity(stage[c], hdry);
  }
  if (kind != S_DG2) {
    u.swap(stage);
    return;
  }
  revise(stage);
  fluxes();
  assemble(true);
  for (size_t c = 0; c < n; ++c) {
    rk2_final(stage[c], rate[c], u[c], dt, u[c]);
    positivity(u[c], hdry);
  }
}

// solver_uniform.cpp:330-415
void UN::step_acc(double dt) {
  auto face = [&](double& q, size_t l, size_t r) {
    const double el = u[l].h.c0 + z[l].c0, er = u[r].h.c0 + z[r].c0;
    const double hf = mx(el, er) - mx(z[l].c0, z[r].c0);
    if (hf <= hdry) {
      q = 0.0;
      return;
    }
    const double nf = 0.5 * (nman[l] + nman[r]);
    q = (q - g * hf * dt * (er - el) / R) / (1.0 + g * dt * nf * nf * std::abs(q) / pow73_m(hf, libm));
  };
  auto edge = [&](double& q, int side, size_t c) {
    if (bc[side] == 0) {
      q = 0.0;
      return;
    }
    const double hf = u[c].h.c0;
    if (hf <= hdry) {
      q = 0.0;
      return;
    }
    q = q / (1.0 + g * dt * nman[c] * nman[c] * std::abs(q) / pow73_m(hf, libm));
  };
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i <= nx; ++i) {
      double& q = aqx[size_t(j) * (nx + 1) + i];
      if (i == 0 || i == nx)
        edge(q, i == 0 ? 3 : 1, cell(i == 0 ? 0 : nx - 1, j));
      else
        face(q, cell(i - 1, j), cell(i, j));
    }
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i < nx; ++i) {
      double& q = aqy[size_t(j) * nx + i];
      if (j == 0 || j == ny)
        edge(q, j == 0 ? 2 : 0, cell(i, j == 0 ? 0 : ny - 1));
      else
        face(q, cell(i, j - 1), cell(i, j));
    }
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const size_t c = cell(i, j);
      const double qw = aqx[size_t(j) * (nx + 1) + i], qe = aqx[size_t(j) * (nx + 1) + i + 1];
      const double qs = aqy[size_t(j) * nx + i], qn = aqy[size_t(j + 1) * nx + i];
      u[c].h.c0 -= dt * ((qe - qw) + (qn - qs)) / R;
      u[c].qx.c0 = 0.5 * (qw + qe);
      u[c].qy.c0 = 0.5 * (qs + qn);
    }
}

void UN::step(double dt) {
  if (kind == S_ACC)
    step_acc(dt);
  else
    step_rk(dt);
}

// solver_uniform.cpp:424-442
double UN::compute_dt() const {
  const double inf = std::numeric_limits<double>::infinity();
  if (kind == S_ACC) {
    double hmax = 0.0;
    for (const Fl& f : u) hmax = mx(hmax, f.h.c0);
    if (hmax <= hdry) return inf;
    return cour * R / std::sqrt(g * hmax);
  }
  double dt = inf;
  for (const Fl& f : u) {
    const double h = f.h.c0;
    if (h <= hdry) continue;
    const double c = std::sqrt(g * h);
    const double sx = std::abs(f.qx.c0 / h) + c;
    const double sy = std::abs(f.qy.c0 / h) + c;
    dt = mn(dt, R / mx(sx, sy));
  }
  return dt * cour;
}

// solver_uniform.cpp:444-455
double UN::apply_inflows(double t, double dt) {
  double added = 0.0;
  for (const Inflow& f : inflows) {
    const double q = hydro_at(f.hy, t);
    if (q <= 0.0) continue;
    const double vol = q * dt;
    const double per = vol / double(f.region);
    for (const auto& [c, cnt] : f.targets) u[c].h.c0 += per * cnt / (R * R);
    added += vol;
  }
  return added;
}

double UN::volume() const {
  double sum = 0.0, comp = 0.0;
  for (const Fl& f : u) {
    const double y = f.h.c0 * R * R - comp;
    const double t = sum + y;
    comp = (t - sum) - y;
    sum = t;
  }
  return sum;
}

bool UN::finite(double* bx, double* by) const {
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i)
      if (!fl_finite(u[cell(i, j)])) {
        if (bx) *bx = x0 + (i + 0.5) * R;
        if (by) *by = y0 + (j + 0.5) * R;
        return false;
      }
  return true;
}

// solver_uniform.cpp:522-601
UN make_un(const Cfg& c, const Raster& dem) {
  UN s;
  s.kind = c.solver;
  s.libm = c.libm;
  if (c.solver == S_MWDG2 || c.solver == S_HWFV1)
    throw Fail(E_CONFIG, "uniform solver cannot run adaptive kinds");
  const Field f = project_plain(dem);
  s.nx = f.nx;
  s.ny = f.ny;
  s.R = f.R;
  s.x0 = f.x0;
  s.y0 = f.y0;
  s.z = f.c;
  s.g = c.g;
  s.hdry = c.hdry;
  s.cour = c.courant_for();
  for (int q = 0; q < 4; ++q) s.bc[q] = c.bc[q];
  const size_t n = s.z.size();
  s.nman.assign(n, c.manning);
  if (c.has_mr)
    for (int j = 0; j < s.ny; ++j)
      for (int i = 0; i < s.nx; ++i) {
        const int row = std::clamp(c.mr.nrows - 1 - j, 0, c.mr.nrows - 1);
        const int col = std::clamp(i, 0, c.mr.ncols - 1);
        s.nman[s.cell(i, j)] = c.mr.at(row, col);
      }
  s.u.assign(n, Fl{});
  if (c.has_h0) {
    if (c.h0.ncols != dem.ncols || c.h0.nrows != dem.nrows)
      throw Fail(E_CONFIG, "initial_depth_raster geometry must match the DEM");
    const Field hg = project_plain(c.h0);
    for (size_t q = 0; q < n; ++q) s.u[q].h = hg.c[q];
  } else if (c.has_eta0) {
    for (size_t q = 0; q < n; ++q) s.u[q] = from_surface(s.z[q], c.eta0);
  } else if (c.depth0 > 0.0) {
    for (size_t q = 0; q < n; ++q) s.u[q].h = {c.depth0, 0.0, 0.0};
  }
  if (s.kind != S_DG2) {
    for (Pl& p : s.z) p.cx = p.cy = 0.0;
    for (Fl& f2 : s.u) {
      f2.h.cx = f2.h.cy = 0.0;
      f2.qx = {};
      f2.qy = {};
    }
  }
  for (Fl& f2 : s.u) positivity(f2, s.hdry);
  // element_nodata_mask (sim_common.cpp:118-131) decides "any active".
  for (const Inflow& spec : c.inflows) {
    if (spec.i0 < 0 || spec.j0 < 0 || spec.i1 >= s.nx || spec.j1 >= s.ny)
      throw Fail(E_CONFIG, "inflow region outside the domain");
    Inflow r = spec;
    r.targets.clear();
    bool any = false;
    for (int j = spec.j0; j <= spec.j1; ++j)
      for (int i = spec.i0; i <= spec.i1; ++i) {
        r.targets.push_back({int32_t(s.cell(i, j)), 1});
        const int rs = dem.nrows - 1 - j;
        const bool bad = dem.at(rs, i) == dem.nodata || dem.at(rs, i + 1) == dem.nodata ||
                         dem.at(rs - 1, i) == dem.nodata || dem.at(rs - 1, i + 1) == dem.nodata;
        if (!bad) any = true;
      }
    r.region = int64_t(r.targets.size());
    if (!any) throw Fail(E_CONFIG, "inflow region lies entirely on nodata cells");
    s.inflows.push_back(std::move(r));
  }
  if (s.kind == S_ACC) {
    s.aqx.assign(size_t(s.nx + 1) * s.ny, 0.0);
    s.aqy.assign(size_t(s.nx) * (s.ny + 1), 0.0);
  }
  return s;
}


// ---- output sampling --------------------------------------------------------

// NonUniformSim::sample_gauge (solver_nonuniform.cpp:489-506) via
// QuadGrid::find_point (quadgrid.cpp:70-74).
void gauge(const NU& s, double x, double y, double out[4]) {
  const Grid& g = s.grid;
  const int fi = int(std::floor((x - g.x0) / g.R));
  const int fj = int(std::floor((y - g.y0) / g.R));
  const int k = g.containing(std::clamp(fi, 0, (g.M << g.L) - 1), std::clamp(fj, 0, (g.N << g.L) - 1));
  out[0] = out[1] = out[2] = out[3] = 0.0;
  if (k < 0) return;
  const Fl& u = s.u[k];
  if (s.scheme == S_DG2) {
    const double cx = g.xc(k), cy = g.yc(k), sz = g.size(k);
    const double h = std::max(0.0, eval_plane(u.h, cx, cy, sz, x, y));
    const double zv = eval_plane(s.z[k], cx, cy, sz, x, y);
    const double qx = eval_plane(u.qx, cx, cy, sz, x, y);
    const double qy = eval_plane(u.qy, cx, cy, sz, x, y);
    out[0] = h;
    out[1] = h + zv;
    out[2] = vel(h, qx, s.hdry);
    out[3] = vel(h, qy, s.hdry);
  } else {
    const double h = u.h.c0;
    out[0] = h;
    out[1] = h + s.z[k].c0;
    out[2] = vel(h, u.qx.c0, s.hdry);
    out[3] = vel(h, u.qy.c0, s.hdry);
  }
}

// UniformSim::sample_gauge (solver_uniform.cpp:480-498)
void gauge(const UN& s, double x, double y, double out[4]) {
  const int i = std::clamp(int(std::floor((x - s.x0) / s.R)), 0, s.nx - 1);
  const int j = std::clamp(int(std::floor((y - s.y0) / s.R)), 0, s.ny - 1);
  const size_t c = s.cell(i, j);
  const Fl& u = s.u[c];
  if (s.kind == S_DG2) {
    const double xc = s.x0 + (i + 0.5) * s.R, yc = s.y0 + (j + 0.5) * s.R;
    const double h = std::max(0.0, eval_plane(u.h, xc, yc, s.R, x, y));
    const double zv = eval_plane(s.z[c], xc, yc, s.R, x, y);
    const double qx = eval_plane(u.qx, xc, yc, s.R, x, y);
    const double qy = eval_plane(u.qy, xc, yc, s.R, x, y);
    out[0] = h;
    out[1] = h + zv;
    out[2] = vel(h, qx, s.hdry);
    out[3] = vel(h, qy, s.hdry);
  } else {
    const double h = u.h.c0;
    out[0] = h;
    out[1] = h + s.z[c].c0;
    out[2] = vel(h, u.qx.c0, s.hdry);
    out[3] = vel(h, u.qy.c0, s.hdry);
  }
}

static const Pl& field_of(const Fl& f, int which) { return which == 0 ? f.h : which == 1 ? f.qx : f.qy; }

// sample_to_raster (quadgrid.cpp:262-285) of leaf_raster (solver_nonuniform.cpp:508-514)
void raster(const NU& s, int which, double* out) {
  const Grid& g = s.grid;
  const int nc = g.M << g.L, nr = g.N << g.L;
  for (int fj = 0; fj < nr; ++fj)
    for (int fi = 0; fi < nc; ++fi) {
      const int k = g.containing(fi, fj);
      if (k < 0) throw Fail(E_STRUCT, "sample_to_raster: hole in grid");
      const double x = g.x0 + (fi + 0.5) * g.R;
      const double y = g.y0 + (fj + 0.5) * g.R;
      out[size_t(nr - 1 - fj) * nc + fi] =
          eval_plane(field_of(s.u[k], which), g.xc(k), g.yc(k), g.size(k), x, y);
    }
}

// field_raster (solver_uniform.cpp:501-516)
void raster(const UN& s, int which, double* out) {
  for (int j = 0; j < s.ny; ++j)
    for (int i = 0; i < s.nx; ++i)
      out[size_t(s.ny - 1 - j) * s.nx + i] = field_of(s.u[s.cell(i, j)], which).c0;
}

}  // namespace orc
