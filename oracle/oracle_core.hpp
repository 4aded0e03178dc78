// ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into or called by the
// product (paper_2107_02750_b200/).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it.
//
// A CPU restatement of the reference floodmra hot path
// (/root/reference/proj/core), written as free functions over flat arrays.
// Every function cites the reference file:line whose arithmetic it restates;
// the floating-point expression trees and summation orders are kept
// identical so that, built without FMA contraction, results are
// bit-identical to the reference library (pinned by tests/test_oracle_vs_ref.py
// against oracle/_ref, the reference compiled from its own sources).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

// field.hpp:11
constexpr double kS3 = 1.7320508075688772;

struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
enum { E_OTHER = 1, E_CONFIG = 2, E_IO = 3, E_BLOWUP = 4, E_STRUCT = 5, E_DOMAIN = 6 };

// std::max / std::min semantics (first argument wins ties and NaNs).
inline double mx(double a, double b) { return (a < b) ? b : a; }
inline double mn(double a, double b) { return (b < a) ? b : a; }

struct Pl {  // PlanarCoeffs, field.hpp:15-47
  double c0 = 0.0, cx = 0.0, cy = 0.0;
};
struct Fl {  // FlowCoeffs, field.hpp:49-67
  Pl h, qx, qy;
};
struct Det {  // DetailTriple, wavelets.hpp:13-15: [dh(3) dv(3) dd(3)]
  double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
};
struct Flux {  // Flux3, hll.hpp:7-11
  double m = 0.0, n = 0.0, t = 0.0;
};

struct Raster {
  int ncols = 0, nrows = 0;
  double xll = 0, yll = 0, cell = 1, nodata = -9999;
  std::vector<double> v;
  double at(int r, int c) const { return v[size_t(r) * ncols + c]; }
};

// ---- basis / wavelets ---------------------------------------------------
Pl project4(double nw, double ne, double sw, double se);                 // field.cpp:11-19
double eval_plane(const Pl& c, double xc, double yc, double R, double x, double y);  // field.cpp:21-24
double face_val(const Pl& c, int side);                                  // field.cpp:26-34
const double* bank(int kind);                                            // wavelets.cpp:14-75 (12x4x3)
void enc(const Pl k[4], int kind, Pl& parent, Det& d);                   // wavelets.cpp:61-86
void dec(const Pl& p, const Det& d, int kind, Pl out[4]);                // wavelets.cpp:88-100
double dhat(const Det& d, double norm);                                  // wavelets.cpp:137-149

// padded fine field (field.cpp:48-117)
struct Field {
  int nx = 0, ny = 0;
  double R = 1, x0 = 0, y0 = 0;
  std::vector<Pl> c;
};
Field project_padded(const Raster& dem, int L, int* M, int* N);
Field project_plain(const Raster& dem);

// ---- static MRA ----------------------------------------------------------
struct Tree {  // DetailTree, detail_tree.hpp:13-30 (row-major per level)
  int L = 0, M = 1, N = 1, kind = 0;
  double R = 1, x0 = 0, y0 = 0, norm = 1;
  std::vector<std::vector<Det>> det;
  std::vector<std::vector<uint8_t>> flag;
  std::vector<Pl> coarse;
  int w(int l) const { return M << l; }
  int h(int l) const { return N << l; }
  size_t node(int l, int i, int j) const { return size_t(j) * w(l) + i; }
};
Tree encode_tree(const Field& f, int L, int M, int N, int kind);          // detail_tree.cpp:10-54
void closure(Tree& t);                                                   // detail_tree.cpp:56-64
void threshold(Tree& t, double eps);                                     // detail_tree.cpp:66-74
void grade(Tree& t);                                                     // detail_tree.cpp:97-113

struct Leaf {
  int l, i, j;
};
struct Grid {  // QuadGrid, quadgrid.hpp:54-84, with a dense per-level index in place of the hash
  int L = 0, M = 1, N = 1;
  double R = 1, x0 = 0, y0 = 0;
  std::vector<Leaf> lv;
  std::vector<std::vector<int32_t>> idx;  // [level][j*w+i] -> leaf or -1
  double size(int k) const { return R * double(1 << (L - lv[k].l)); }
  double xc(int k) const { return x0 + (lv[k].i + 0.5) * R * double(1 << (L - lv[k].l)); }
  double yc(int k) const { return y0 + (lv[k].j + 0.5) * R * double(1 << (L - lv[k].l)); }
  bool inside(int l, int i, int j) const {
    return l >= 0 && l <= L && i >= 0 && j >= 0 && i < (M << l) && j < (N << l);
  }
  int find(int l, int i, int j) const;
  int containing(int fi, int fj) const;
};
Grid make_grid(int L, int M, int N, double R, double x0, double y0, std::vector<Leaf> leaves);  // quadgrid.cpp:85-110
std::vector<Leaf> tree_leaves(const Tree& t);                            // detail_tree.cpp:115-130
void tree_decode(const Tree& t, const Grid& g, std::vector<Pl>& topo);   // detail_tree.cpp:132-164

// ---- topology -------------------------------------------------------------
struct Nbr {
  bool boundary = false;
  std::vector<int> leaves;
};
Nbr neighbours(const Grid& g, int k, int side);                          // quadgrid.cpp:121-171
bool graded(const Grid& g);                                              // quadgrid.cpp:173-182
struct Seg {
  int l = -1, r = -1;
  bool xn = true;
  double cx = 0, cy = 0, len = 0;
};
struct BSeg {
  int leaf = -1, side = 0;
  double cx = 0, cy = 0, len = 0;
};
struct Faces {
  std::vector<Seg> in;
  std::vector<BSeg> bd;
  std::vector<std::vector<int32_t>> sides;  // 4 per leaf
};
Faces faces_of(const Grid& g, bool need_graded);                         // quadgrid.cpp:184-260

// ---- point kernels ----------------------------------------------------------
Flux hll(double hl, double qnl, double qtl, double hr, double qnr, double qtr, double g,
         double hdry);                                                   // hll.cpp:10-58
void friction(double h0, Pl& qx, Pl& qy, double n, double g, double hdry, double dt,
              int libm = 0);  // sim_common.cpp:30-46
// Deterministic cube root / h^(7/3) from +,-,*,/ only (parity harness,
// FM_LIBM_PORTABLE); the CUDA path implements the same operation sequence.
double pcbrt(double x);
double cbrt_m(double x, int libm);
double pow73_m(double x, int libm);
void positivity(Fl& f, double hdry);                                     // solver_nonuniform.cpp:276-304

struct Hydro {
  std::vector<double> t, q;
};
double hydro_at(const Hydro& h, double t);                               // hydrograph.cpp:38-49
struct Inflow {  // ResolvedInflow, sim_common.hpp:86-91
  Hydro hy;
  std::vector<std::pair<int32_t, int32_t>> targets;
  int64_t region = 0;
  int i0 = 0, j0 = 0, i1 = 0, j1 = 0;
};

}  // namespace orc
