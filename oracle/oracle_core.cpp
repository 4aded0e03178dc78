// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle_core.hpp).
// Restatement of field.cpp, wavelets.cpp, detail_tree.cpp, quadgrid.cpp,
// hll.cpp, sim_common.cpp and hydrograph.cpp arithmetic.
#include "oracle_core.hpp"

#include <algorithm>
#include <cstring>
#include <limits>

namespace orc {

// field.cpp:11-19 — Eq. 8 plane from the four corner samples.
Pl project4(double nw, double ne, double sw, double se) {
  if (!(std::isfinite(nw) && std::isfinite(ne) && std::isfinite(sw) && std::isfinite(se)))
    throw Fail(E_DOMAIN, "project_vertices: non-finite vertex value");
  Pl p;
  p.c0 = 0.25 * (ne + nw + se + sw);
  p.cx = (ne - nw + se - sw) / (4.0 * kS3);
  p.cy = (ne - se + nw - sw) / (4.0 * kS3);
  return p;
}

// field.cpp:21-24
double eval_plane(const Pl& c, double xc, double yc, double R, double x, double y) {
  if (R <= 0.0) throw Fail(E_DOMAIN, "evaluate: element size must be positive");
  return c.c0 + c.cx * 2.0 * kS3 * (x - xc) / R + c.cy * 2.0 * kS3 * (y - yc) / R;
}

// field.cpp:26-34 (side 0=N 1=E 2=S 3=W)
double face_val(const Pl& c, int side) {
  switch (side) {
    case 1: return c.c0 + kS3 * c.cx;
    case 3: return c.c0 - kS3 * c.cx;
    case 0: return c.c0 + kS3 * c.cy;
    case 2: return c.c0 - kS3 * c.cy;
  }
  return c.c0;
}

// wavelets.cpp:14-59.  Layout a[row][child][mode] flattened; child order
// SW, SE, NW, NE (wavelets.hpp:17-23).
static void fill_bank(double* a, int kind) {
  std::memset(a, 0, sizeof(double) * 144);
  auto at = [a](int row, int k, int n) -> double& { return a[(row * 4 + k) * 3 + n]; };
  for (int k = 0; k < 4; ++k) {
    const double sx = (k & 1) ? 1.0 : -1.0;
    const double sy = (k & 2) ? 1.0 : -1.0;
    if (kind == 0) {
      at(0, k, 0) = 0.25;
      at(1, k, 0) = sx * kS3 / 8.0;
      at(1, k, 1) = 1.0 / 8.0;
      at(2, k, 0) = sy * kS3 / 8.0;
      at(2, k, 2) = 1.0 / 8.0;
      at(3, k, 0) = sx / 8.0;
      at(3, k, 1) = -kS3 / 8.0;
      at(4, k, 1) = sx / 4.0;
      at(5, k, 2) = sx / 4.0;
      at(6, k, 0) = sy / 8.0;
      at(6, k, 2) = -kS3 / 8.0;
      at(7, k, 2) = sy / 4.0;
      at(8, k, 1) = sy / 4.0;
      at(9, k, 0) = sx * sy / 4.0;
      at(10, k, 1) = sx * sy / 4.0;
      at(11, k, 2) = sx * sy / 4.0;
    } else {
      at(0, k, 0) = 0.25;
      at(3, k, 0) = sx / 4.0;
      at(6, k, 0) = sy / 4.0;
      at(9, k, 0) = sx * sy / 4.0;
    }
  }
}

const double* bank(int kind) {
  static double mw[144], hw[144];
  static bool ready = [] {
    fill_bank(mw, 0);
    fill_bank(hw, 1);
    return true;
  }();
  (void)ready;
  return kind == 0 ? mw : hw;
}

// wavelets.cpp:61-67 row_dot, :77-86 encode.
void enc(const Pl k[4], int kind, Pl& parent, Det& d) {
  const double* a = bank(kind);
  double out[12];
  for (int row = 0; row < 12; ++row) {
    double acc = 0.0;
    for (int c = 0; c < 4; ++c) {
      const double* r = a + (row * 4 + c) * 3;
      acc += r[0] * k[c].c0 + r[1] * k[c].cx + r[2] * k[c].cy;
    }
    out[row] = acc;
  }
  parent = {out[0], out[1], out[2]};
  for (int n = 0; n < 9; ++n) d.v[n] = out[3 + n];
}

// wavelets.cpp:88-100 — synthesis is 4x the transpose, rows summed in order.
void dec(const Pl& p, const Det& d, int kind, Pl out[4]) {
  const double* a = bank(kind);
  const double v[12] = {p.c0,   p.cx,   p.cy,   d.v[0], d.v[1], d.v[2],
                        d.v[3], d.v[4], d.v[5], d.v[6], d.v[7], d.v[8]};
  for (int c = 0; c < 4; ++c) {
    double z[3] = {0.0, 0.0, 0.0};
    for (int n = 0; n < 3; ++n)
      for (int row = 0; row < 12; ++row) z[n] += 4.0 * a[(row * 4 + c) * 3 + n] * v[row];
    out[c] = {z[0], z[1], z[2]};
  }
}

// wavelets.cpp:137-149
double dhat(const Det& d, double norm) {
  double m = 0.0;
  for (int n = 0; n < 9; ++n) m = mx(m, std::abs(d.v[n]));
  return m / mx(1.0, norm);
}

// field.cpp:48-54 nodata wall, :57-91 padded projection.
static Field project_core(const Raster& dem, int nx, int ny) {
  double zmax = -std::numeric_limits<double>::infinity();
  for (double v : dem.v)
    if (v != dem.nodata) zmax = mx(zmax, v);
  if (!std::isfinite(zmax)) zmax = 0.0;
  const double wall = zmax + 100.0;
  const int n = dem.ncols - 1, m = dem.nrows - 1;
  Field f;
  f.nx = nx;
  f.ny = ny;
  f.R = dem.cell;
  f.x0 = dem.xll;
  f.y0 = dem.yll;
  f.c.resize(size_t(nx) * ny);
  auto vx = [&](int r, int c) {
    const double v = dem.at(r, c);
    return v == dem.nodata ? wall : v;
  };
  for (int j = 0; j < ny; ++j) {
    const int je = std::min(j, m - 1);
    const int rs = dem.nrows - 1 - je, rn = rs - 1;
    for (int i = 0; i < nx; ++i) {
      const int ie = std::min(i, n - 1);
      f.c[size_t(j) * nx + i] = project4(vx(rn, ie), vx(rn, ie + 1), vx(rs, ie), vx(rs, ie + 1));
    }
  }
  return f;
}

Field project_padded(const Raster& dem, int L, int* M, int* N) {
  if (dem.ncols < 2 || dem.nrows < 2)
    throw Fail(E_CONFIG, "DEM must have at least 2x2 samples to define elements");
  if (L < 0) throw Fail(E_CONFIG, "max_level must be >= 0");
  const int step = 1 << L;
  const int m0 = (dem.ncols - 1 + step - 1) / step, n0 = (dem.nrows - 1 + step - 1) / step;
  if (M) *M = m0;
  if (N) *N = n0;
  return project_core(dem, m0 << L, n0 << L);
}

Field project_plain(const Raster& dem) {
  if (dem.ncols < 2 || dem.nrows < 2)
    throw Fail(E_CONFIG, "DEM must have at least 2x2 samples to define elements");
  return project_core(dem, dem.ncols - 1, dem.nrows - 1);
}

// detail_tree.cpp:10-54
Tree encode_tree(const Field& f, int L, int M, int N, int kind) {
  if (f.nx != (M << L) || f.ny != (N << L))
    throw Fail(E_STRUCT, "build_detail_tree: field is not an (M 2^L) x (N 2^L) grid");
  Tree t;
  t.L = L;
  t.M = M;
  t.N = N;
  t.kind = kind;
  t.R = f.R;
  t.x0 = f.x0;
  t.y0 = f.y0;
  t.norm = 0.0;
  for (const Pl& c : f.c) t.norm = mx(t.norm, std::abs(c.c0));
  t.det.resize(L);
  t.flag.resize(L);
  for (int l = 0; l < L; ++l) {
    t.det[l].resize(size_t(t.w(l)) * t.h(l));
    t.flag[l].assign(size_t(t.w(l)) * t.h(l), 0);
  }
  std::vector<Pl> cur = f.c, up;
  for (int l = L - 1; l >= 0; --l) {
    const int w = t.w(l), h = t.h(l), cw = 2 * w;
    up.assign(size_t(w) * h, Pl{});
    for (int j = 0; j < h; ++j)
      for (int i = 0; i < w; ++i) {
        const size_t s = size_t(2 * j) * cw + 2 * i, n = s + cw;
        const Pl kids[4] = {cur[s], cur[s + 1], cur[n], cur[n + 1]};
        enc(kids, kind, up[t.node(l, i, j)], t.det[l][t.node(l, i, j)]);
      }
    cur.swap(up);
  }
  t.coarse = cur;
  return t;
}

// detail_tree.cpp:56-64
void closure(Tree& t) {
  for (int l = t.L - 1; l >= 1; --l)
    for (int j = 0; j < t.h(l); ++j)
      for (int i = 0; i < t.w(l); ++i)
        if (t.flag[l][t.node(l, i, j)]) t.flag[l - 1][t.node(l - 1, i / 2, j / 2)] = 1;
}

// detail_tree.cpp:66-74 (non-strict >=)
void threshold(Tree& t, double eps) {
  if (eps < 0.0) throw Fail(E_DOMAIN, "flag_significant: eps must be >= 0");
  for (int l = 0; l < t.L; ++l)
    for (size_t k = 0; k < t.det[l].size(); ++k) t.flag[l][k] = dhat(t.det[l][k], t.norm) >= eps;
  closure(t);
}

// detail_tree.cpp:97-113
void grade(Tree& t) {
  static const int di[4] = {1, -1, 0, 0}, dj[4] = {0, 0, 1, -1};
  for (int l = t.L - 1; l >= 1; --l)
    for (int j = 0; j < t.h(l); ++j)
      for (int i = 0; i < t.w(l); ++i) {
        if (!t.flag[l][t.node(l, i, j)]) continue;
        for (int d = 0; d < 4; ++d) {
          const int ni = i + di[d], nj = j + dj[d];
          if (ni < 0 || nj < 0 || ni >= t.w(l) || nj >= t.h(l)) continue;
          t.flag[l - 1][t.node(l - 1, ni / 2, nj / 2)] = 1;
        }
      }
}

// detail_tree.cpp:115-130 — level-major, row-major (already make_quadgrid order).
std::vector<Leaf> tree_leaves(const Tree& t) {
  std::vector<Leaf> out;
  for (int l = 0; l <= t.L; ++l)
    for (int j = 0; j < (t.N << l); ++j)
      for (int i = 0; i < (t.M << l); ++i) {
        const bool self = l < t.L && t.flag[l][t.node(l, i, j)];
        const bool par = l == 0 || t.flag[l - 1][t.node(l - 1, i / 2, j / 2)];
        if (!self && par) out.push_back({l, i, j});
      }
  return out;
}

int Grid::find(int l, int i, int j) const {
  if (!inside(l, i, j)) throw Fail(E_DOMAIN, "QuadGrid::find: index out of range");
  return idx[l][size_t(j) * (M << l) + i];
}

// quadgrid.cpp:62-69
int Grid::containing(int fi, int fj) const {
  if (!inside(L, fi, fj)) return -1;
  for (int l = L; l >= 0; --l) {
    const int k = idx[l][size_t(fj >> (L - l)) * (M << l) + (fi >> (L - l))];
    if (k >= 0) return k;
  }
  return -1;
}

// quadgrid.cpp:85-110 — sort (level, j, i), index, tiling check.
Grid make_grid(int L, int M, int N, double R, double x0, double y0, std::vector<Leaf> leaves) {
  Grid g;
  g.L = L;
  g.M = M;
  g.N = N;
  g.R = R;
  g.x0 = x0;
  g.y0 = y0;
  std::sort(leaves.begin(), leaves.end(), [](const Leaf& a, const Leaf& b) {
    if (a.l != b.l) return a.l < b.l;
    if (a.j != b.j) return a.j < b.j;
    return a.i < b.i;
  });
  g.lv = std::move(leaves);
  g.idx.resize(L + 1);
  for (int l = 0; l <= L; ++l) g.idx[l].assign(size_t(M << l) * size_t(N << l), -1);
  int64_t weight = 0;
  for (size_t k = 0; k < g.lv.size(); ++k) {
    const Leaf& f = g.lv[k];
    if (!g.inside(f.l, f.i, f.j)) throw Fail(E_STRUCT, "make_quadgrid: leaf outside domain");
    g.idx[f.l][size_t(f.j) * (M << f.l) + f.i] = int32_t(k);
    weight += int64_t(1) << (2 * (L - f.l));
  }
  if (weight != int64_t(M) * N * (int64_t(1) << (2 * L)))
    throw Fail(E_STRUCT, "make_quadgrid: leaves do not tile the domain");
  return g;
}

// detail_tree.cpp:132-164 — the DFS result per leaf depends only on its
// ancestor chain, so a level-by-level top-down decode is identical.
void tree_decode(const Tree& t, const Grid& g, std::vector<Pl>& topo) {
  topo.assign(g.lv.size(), Pl{});
  std::vector<Pl> cur = t.coarse, nxt;
  for (int l = 0; l <= t.L; ++l) {
    const int w = t.w(l), h = t.h(l);
    if (l < t.L) nxt.assign(size_t(4) * w * h, Pl{});
    for (int j = 0; j < h; ++j)
      for (int i = 0; i < w; ++i) {
        const bool active = l == 0 || t.flag[l - 1][t.node(l - 1, i / 2, j / 2)];
        if (!active) continue;
        const Pl z = cur[size_t(j) * w + i];
        if (l == t.L || !t.flag[l][t.node(l, i, j)]) {
          const int k = g.find(l, i, j);
          if (k < 0) throw Fail(E_STRUCT, "assemble_grid: leaf set does not match flags");
          topo[k] = z;
          continue;
        }
        Pl kids[4];
        dec(z, t.det[l][t.node(l, i, j)], t.kind, kids);
        for (int c = 0; c < 4; ++c)
          nxt[size_t(2 * j + (c >> 1)) * (2 * w) + 2 * i + (c & 1)] = kids[c];
      }
    cur.swap(nxt);
  }
}

// quadgrid.cpp:121-171
Nbr neighbours(const Grid& g, int k, int side) {
  const Leaf f = g.lv[k];
  const int di = side == 1 ? 1 : side == 3 ? -1 : 0;
  const int dj = side == 0 ? 1 : side == 2 ? -1 : 0;
  const int ni = f.i + di, nj = f.j + dj;
  Nbr out;
  if (!g.inside(f.l, ni, nj)) {
    out.boundary = true;
    return out;
  }
  for (int l = f.l; l >= 0; --l) {
    const int s = f.l - l;
    const int q = g.find(l, ni >> s, nj >> s);
    if (q >= 0) {
      out.leaves.push_back(q);
      return out;
    }
  }
  std::vector<Leaf> stack{{f.l, ni, nj}};
  const int ci0 = side == 3 ? 1 : 0, ci1 = side == 1 ? 0 : 1;
  const int cj0 = side == 2 ? 1 : 0, cj1 = side == 0 ? 0 : 1;
  while (!stack.empty()) {
    const Leaf n = stack.back();
    stack.pop_back();
    const int q = n.l <= g.L ? g.find(n.l, n.i, n.j) : -1;
    if (q >= 0) {
      out.leaves.push_back(q);
      continue;
    }
    if (n.l >= g.L) throw Fail(E_STRUCT, "neighbors: grid does not tile the domain");
    for (int cj = cj0; cj <= cj1; ++cj)
      for (int ci = ci0; ci <= ci1; ++ci) stack.push_back({n.l + 1, 2 * n.i + ci, 2 * n.j + cj});
  }
  std::sort(out.leaves.begin(), out.leaves.end(), [&g](int a, int b) {
    const Leaf& la = g.lv[a];
    const Leaf& lb = g.lv[b];
    const int ja = la.j << (g.L - la.l), jb = lb.j << (g.L - lb.l);
    if (ja != jb) return ja < jb;
    return (la.i << (g.L - la.l)) < (lb.i << (g.L - lb.l));
  });
  return out;
}

// quadgrid.cpp:173-182
bool graded(const Grid& g) {
  for (int k = 0; k < int(g.lv.size()); ++k)
    for (int s = 0; s < 4; ++s) {
      const Nbr q = neighbours(g, k, s);
      for (int b : q.leaves)
        if (std::abs(g.lv[b].l - g.lv[k].l) > 1) return false;
    }
  return true;
}

// quadgrid.cpp:184-260
Faces faces_of(const Grid& g, bool need_graded) {
  Faces F;
  const int n = int(g.lv.size());
  F.sides.resize(size_t(n) * 4);
  for (int k = 0; k < n; ++k) {
    const Leaf f = g.lv[k];
    const double sz = g.size(k), xc = g.xc(k), yc = g.yc(k);
    for (int s = 0; s < 4; ++s) {
      const Nbr q = neighbours(g, k, s);
      const bool xn = (s == 1 || s == 3);
      if (q.boundary) {
        BSeg b;
        b.leaf = k;
        b.side = s;
        b.len = sz;
        b.cx = xc + (s == 1 ? sz / 2 : s == 3 ? -sz / 2 : 0.0);
        b.cy = yc + (s == 0 ? sz / 2 : s == 2 ? -sz / 2 : 0.0);
        F.bd.push_back(b);
        F.sides[size_t(k) * 4 + s].push_back(-1 - int(F.bd.size() - 1));
        continue;
      }
      const int nl = g.lv[q.leaves.front()].l;
      if (nl < f.l) continue;
      if (nl == f.l && (s == 3 || s == 2)) continue;
      if (need_graded && q.leaves.size() > 2)
        throw Fail(E_STRUCT, "enumerate_faces: grid is not graded");
      for (int b : q.leaves) {
        if (need_graded && g.lv[b].l > f.l + 1)
          throw Fail(E_STRUCT, "enumerate_faces: grid is not graded");
        Seg e;
        e.xn = xn;
        e.len = std::min(sz, g.size(b));
        if (xn) {
          e.cx = xc + (s == 1 ? sz / 2 : -sz / 2);
          e.cy = g.yc(b);
          e.l = s == 1 ? k : b;
          e.r = s == 1 ? b : k;
        } else {
          e.cy = yc + (s == 0 ? sz / 2 : -sz / 2);
          e.cx = g.xc(b);
          e.l = s == 0 ? k : b;
          e.r = s == 0 ? b : k;
        }
        F.in.push_back(e);
      }
    }
  }
  for (int si = 0; si < int(F.in.size()); ++si) {
    const Seg& e = F.in[si];
    F.sides[size_t(e.l) * 4 + (e.xn ? 1 : 0)].push_back(si);
    F.sides[size_t(e.r) * 4 + (e.xn ? 3 : 2)].push_back(si);
  }
  for (auto& lst : F.sides)
    std::sort(lst.begin(), lst.end(), [&F](int a, int b) {
      if (a < 0 || b < 0) return a > b;
      const Seg& sa = F.in[a];
      const Seg& sb = F.in[b];
      if (sa.cy != sb.cy) return sa.cy < sb.cy;
      return sa.cx < sb.cx;
    });
  return F;
}

// hll.cpp:10-58
Flux hll(double hl, double qnl, double qtl, double hr, double qnr, double qtr, double g,
         double hdry) {
  if (hl < 0.0 || hr < 0.0) throw Fail(E_DOMAIN, "hll_flux: negative depth");
  const bool dl = hl <= hdry, dr = hr <= hdry;
  if (dl && dr) return {};
  const double ul = dl ? 0.0 : qnl / hl;
  const double vl = dl ? 0.0 : qtl / hl;
  const double ur = dr ? 0.0 : qnr / hr;
  const double vr = dr ? 0.0 : qtr / hr;
  const double al = std::sqrt(g * mx(hl, 0.0));
  const double ar = std::sqrt(g * mx(hr, 0.0));
  double sl, sr;
  if (dl) {
    sl = ur - 2.0 * ar;
    sr = ur + ar;
  } else if (dr) {
    sl = ul - al;
    sr = ul + 2.0 * al;
  } else {
    const double us = 0.5 * (ul + ur) + al - ar;
    const double as = 0.5 * (al + ar) + 0.25 * (ul - ur);
    sl = mn(ul - al, us - as);
    sr = mx(ur + ar, us + as);
  }
  const double fml = dl ? 0.0 : qnl;
  const double fnl = dl ? 0.5 * g * hl * hl : qnl * ul + 0.5 * g * hl * hl;
  const double fmr = dr ? 0.0 : qnr;
  const double fnr = dr ? 0.5 * g * hr * hr : qnr * ur + 0.5 * g * hr * hr;
  Flux f;
  if (sl >= 0.0) {
    f.m = fml;
    f.n = fnl;
  } else if (sr <= 0.0) {
    f.m = fmr;
    f.n = fnr;
  } else {
    const double inv = 1.0 / (sr - sl);
    f.m = (sr * fml - sl * fmr + sl * sr * (hr - hl)) * inv;
    f.n = (sr * fnl - sl * fnr + sl * sr * (qnr - qnl)) * inv;
  }
  f.t = f.m >= 0.0 ? f.m * vl : f.m * vr;
  return f;
}

// sim_common.cpp:30-46
// Portable cube root for positive finite x: split x = f 2^E (f in [1,2)),
// E = 3k + r, solve y^3 = f 2^r in [1,8) with six Newton steps from a linear
// guess, rescale by 2^k.  Only IEEE +,-,*,/ and exact power-of-two scalings.
double pcbrt(double x) {
  if (!(x > 0.0) || !std::isfinite(x)) return x;  // callers pass h > h_dry > 0
  uint64_t b;
  std::memcpy(&b, &x, 8);
  int e = int((b >> 52) & 0x7ff), shift = 0;
  if (e == 0) {
    const double y = x * 18014398509481984.0;  // 2^54
    std::memcpy(&b, &y, 8);
    e = int((b >> 52) & 0x7ff);
    shift = 54;
  }
  const int E = e - 1023 - shift;
  const int k = E >= 0 ? E / 3 : -((2 - E) / 3);
  const int r = E - 3 * k;
  uint64_t fb = (b & 0x000fffffffffffffull) | (uint64_t(1023 + r) << 52);
  double m;
  std::memcpy(&m, &fb, 8);
  double y = 0.8 + 0.15 * m;
  for (int it = 0; it < 6; ++it) y = (2.0 * y + m / (y * y)) / 3.0;
  const uint64_t sb = uint64_t(1023 + k) << 52;
  double sc;
  std::memcpy(&sc, &sb, 8);
  return y * sc;
}

double cbrt_m(double x, int libm) { return libm ? pcbrt(x) : std::cbrt(x); }
double pow73_m(double x, int libm) { return libm ? x * x * pcbrt(x) : std::pow(x, 7.0 / 3.0); }

void friction(double h0, Pl& qx, Pl& qy, double n, double g, double hdry, double dt, int libm) {
  if (h0 <= hdry) {
    qx = {};
    qy = {};
    return;
  }
  if (n <= 0.0) return;
  const double u = qx.c0 / h0, v = qy.c0 / h0;
  const double sp = std::sqrt(u * u + v * v);
  if (sp == 0.0) return;
  const double cf = g * n * n / cbrt_m(h0, libm);
  const double den = 1.0 + dt * cf * sp / h0;
  qx.c0 /= den;
  qy.c0 /= den;
}

// solver_nonuniform.cpp:276-304 (identical in solver_uniform.cpp:253-281)
void positivity(Fl& f, double hdry) {
  if (!(f.h.c0 > 0.0)) {
    f.h = {mx(f.h.c0, 0.0), 0.0, 0.0};
    f.qx = {};
    f.qy = {};
    return;
  }
  if (f.h.c0 <= hdry) {
    f.h.cx = f.h.cy = 0.0;
    f.qx = {};
    f.qy = {};
    return;
  }
  const double span = kS3 * (std::abs(f.h.cx) + std::abs(f.h.cy));
  if (f.h.c0 - span < 0.0) {
    const double th = f.h.c0 / span;
    f.h.cx *= th;
    f.h.cy *= th;
    f.qx.cx *= th;
    f.qx.cy *= th;
    f.qy.cx *= th;
    f.qy.cy *= th;
  }
}

// hydrograph.cpp:38-49
double hydro_at(const Hydro& h, double t) {
  if (h.t.empty()) throw Fail(E_CONFIG, "hydrograph_at: empty hydrograph");
  if (t <= h.t.front()) return h.q.front();
  if (t >= h.t.back()) return h.q.back();
  const size_t hi = size_t(std::upper_bound(h.t.begin(), h.t.end(), t) - h.t.begin());
  const size_t lo = hi - 1;
  if (t == h.t[lo]) return h.q[lo];
  const double w = (t - h.t[lo]) / (h.t[hi] - h.t[lo]);
  return h.q[lo] + w * (h.q[hi] - h.q[lo]);
}

}  // namespace orc
