// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle_core.hpp).
#pragma once

#include <memory>

#include "oracle_core.hpp"

namespace orc {

enum { S_DG2 = 0, S_FV1 = 1, S_ACC = 2, S_MWDG2 = 3, S_HWFV1 = 4 };

// The ScenarioConfig fields the solvers read (config.hpp:29-69).
struct Cfg {
  int solver = 0;
  double g = 9.80665, hdry = 1e-6, courant = 0.0;
  int bc[4] = {0, 0, 0, 0};
  double manning = 0.0;
  bool has_mr = false;
  Raster mr;  // cell-centred Manning raster
  bool has_h0 = false;
  Raster h0;  // initial depth vertex raster
  bool has_eta0 = false;
  double eta0 = 0.0, depth0 = 0.0;
  std::vector<Inflow> inflows;  // hydrograph + rectangle (targets unresolved)
  double eps = 1e-3;
  int L = -1, adapt_every = 1;
  int libm = 0;  // FM_LIBM_NATIVE / FM_LIBM_PORTABLE
  double courant_for() const;  // config.cpp:37-47
};

// Static / adaptive non-uniform solver (solver_nonuniform.hpp:18-84).
struct NU {
  int scheme = S_DG2;
  Grid grid;
  Faces F;
  double g = 9.80665, hdry = 1e-6, cour = 0.33;
  int bc[4] = {0, 0, 0, 0};
  std::vector<Pl> z;
  std::vector<Fl> u;
  std::vector<double> nman;
  std::vector<Inflow> inflows;
  int pairing = -1;  // encode_pairing bank (adaptive) or -1
  int libm = 0;
  std::vector<double> accq, accqb;

  // scratch
  struct SegS {
    Flux f;
    double zs = 0, hl = 0, hr = 0;
  };
  struct SideS {
    double h = 0, qx = 0, qy = 0, zs = 0, zd = 0;
  };
  std::vector<SegS> seg;
  std::vector<SideS> sd;
  std::vector<Fl> rate, stage;

  void rebuild();                 // solver_nonuniform.cpp:508-514
  double compute_dt() const;      // :427-449
  void step(double dt);           // :420-425
  double apply_inflows(double t, double dt);  // :451-465
  double volume() const;          // :467-477
  bool finite(double* bx, double* by) const;  // :479-487

  void seg_pass(const std::vector<Fl>& s);   // :91-115
  void side_pass(const std::vector<Fl>& s);  // :117-178
  void rate_pass();                          // :180-274
  void step_rk(double dt);                   // :306-348
  void step_acc(double dt);                  // :350-418
  Pl region_topo(int l, int i, int j) const; // :80-89
};

// solver_nonuniform.cpp:516-556 restrict_flow_to_leaves
std::vector<Fl> restrict_to_leaves(const Grid& g, const std::vector<Fl>& fine, int kind);
// solver_uniform.cpp:60-71
Fl from_surface(const Pl& z, double eta0);
// solver_nonuniform.cpp:558-636
NU make_nu(const Cfg& c, const Raster& dem, const Grid& grid, const std::vector<Pl>& topo);

// Adaptive MWDG2/HWFV1 (solver_adaptive.hpp:16-63).
struct AD {
  NU sim;
  Tree zt;
  int kind = 0;
  double eps = 1e-3;
  int adapt_every = 1;
  int64_t since = 0;
  std::vector<std::pair<double, int64_t>> log;
  double man = 0.0;
  bool has_mr = false;
  Raster mr;
  std::vector<Inflow> raw;
  struct Lev {
    std::vector<Fl> sc;
    std::vector<Det> dh, dqx, dqy;
    std::vector<uint8_t> known;
  };
  std::vector<Lev> lev;
  void encode_up();                       // solver_adaptive.cpp:16-57
  void flag(double nh, double nqx, double nqy);  // :59-73
  void ring();                            // :75-94
  std::vector<Fl> transfer(const Grid& ng) const;  // :96-134
  void remap();                           // :173-202
  void adapt(double t);                   // :136-171
};
AD make_ad(const Cfg& c, const Raster& dem);  // solver_adaptive.cpp:209-236

// Uniform raster solver (solver_uniform.hpp:15-67).
struct UN {
  int kind = S_DG2;
  int nx = 0, ny = 0;
  double R = 1, x0 = 0, y0 = 0, g = 9.80665, hdry = 1e-6, cour = 0.33;
  int bc[4] = {0, 0, 0, 0};
  int libm = 0;
  std::vector<Pl> z;
  std::vector<Fl> u;
  std::vector<double> nman;
  std::vector<Inflow> inflows;
  std::vector<double> aqx, aqy;
  struct St {
    double h = 0, qx = 0, qy = 0;
  };
  struct Dm {
    double h0 = 0, h1 = 0, qx0 = 0, qx1 = 0, qy0 = 0, qy1 = 0, z1 = 0;
  };
  std::vector<St> se, sw, sn, ss;
  std::vector<Dm> dmx, dmy;
  std::vector<Flux> fx, fy;
  std::vector<Fl> rate, stage;
  size_t cell(int i, int j) const { return size_t(j) * nx + i; }
  void revise(const std::vector<Fl>& s);  // solver_uniform.cpp:73-137
  void fluxes();                          // :139-185
  void assemble(bool dg2);                // :187-251
  void step_rk(double dt);                // :283-328
  void step_acc(double dt);               // :330-415
  void step(double dt);
  double compute_dt() const;              // :424-442
  double apply_inflows(double t, double dt);  // :444-455
  double volume() const;
  bool finite(double* bx, double* by) const;
};
UN make_un(const Cfg& c, const Raster& dem);  // solver_uniform.cpp:522-601

// ---- output sampling --------------------------------------------------------
// GaugeValue {h, eta, u, v} (sim_common.hpp:47-49)
void gauge(const NU& s, double x, double y, double out[4]);  // solver_nonuniform.cpp:489-506
void gauge(const UN& s, double x, double y, double out[4]);  // solver_uniform.cpp:480-498
// Fine-grid rasters, row 0 north.  NU: leaf_raster -> sample_to_raster
// (solver_nonuniform.cpp:508-519, quadgrid.cpp:262-285), (N<<L) x (M<<L);
// UN: field_raster (solver_uniform.cpp:501-516), ny x nx.  which: 0 h, 1 qx, 2 qy.
void raster(const NU& s, int which, double* out);
void raster(const UN& s, int which, double* out);

}  // namespace orc
