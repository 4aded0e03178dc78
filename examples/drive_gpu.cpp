// drive_gpu — the reference's drive<Sim> loop (run.cpp:79-107) written in C++
// against the drop-in classes of include/fm_gpu.hpp, with no Python in the
// process.  It is what a floodmra maintainer's run_scenario would look like
// with the GPU solvers plugged in.
//
//   drive_gpu DEM.f64 NCELLS CELLSIZE SOLVER L EPS SURFACE MANNING STEPS LIBM OUT.f64
//
// DEM.f64 holds (NCELLS+1)^2 row-major vertex elevations (row 0 north, lower
// left corner at the origin); the domain is a closed box (reflective walls)
// filled to the free surface SURFACE.  SOLVER is an FM_* solver id (10 + id for
// the uniform raster solver).  After
// STEPS steps the state (9 doubles per cell, reference order) is written to
// OUT.f64 and one JSON line with the run statistics goes to stdout.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "fm_gpu.hpp"

int main(int argc, char** argv) {
  if (argc != 12) {
    std::fprintf(stderr, "usage: %s DEM.f64 NCELLS CELLSIZE SOLVER L EPS SURFACE MANNING "
                         "STEPS LIBM OUT.f64\n", argv[0]);
    return 2;
  }
  const int n = std::atoi(argv[2]);
  const double cs = std::atof(argv[3]);
  const int solver = std::atoi(argv[4]) % 10;
  const bool uniform = std::atoi(argv[4]) >= 10;  // 10 + FM_DG2 etc.: the uniform raster sim
  const int L = std::atoi(argv[5]);
  const double eps = std::atof(argv[6]);
  const double surface = std::atof(argv[7]);
  const double manning = std::atof(argv[8]);
  const long steps = std::atol(argv[9]);
  const int libm = std::atoi(argv[10]);

  std::vector<double> dem((size_t)(n + 1) * (n + 1));
  FILE* f = std::fopen(argv[1], "rb");
  if (!f || std::fread(dem.data(), sizeof(double), dem.size(), f) != dem.size()) {
    std::fprintf(stderr, "cannot read %s\n", argv[1]);
    return 3;
  }
  std::fclose(f);

  try {
    fm_gpu::check(fm_init(0));
    fm_raster r{dem.data(), n + 1, n + 1, 0.0, 0.0, cs, -9999.0, 0};
    fm_sim_desc d{};
    d.solver = solver;
    d.g = 9.80665;
    d.h_dry = 1e-6;
    d.courant = 0.0;  // solver default
    d.manning = manning;
    d.has_initial_surface = 1;
    d.initial_surface = surface;
    d.epsilon = eps;
    d.max_level = L;
    d.adapt_every = 1;
    d.libm = libm;

    const bool adaptive = solver == FM_MWDG2 || solver == FM_HWFV1;
    std::unique_ptr<fm_gpu::Grid> grid;
    if (!adaptive && !uniform) grid = std::make_unique<fm_gpu::Grid>(r, L, eps);
    fm_gpu::Sim sim(d, r, grid.get());

    // drive<Sim> (run.cpp:79-107) with an open-ended clock and no events.
    const double v0 = sim.volume();
    double now = 0.0, dt_min = std::numeric_limits<double>::infinity(), dt_max = 0.0;
    double inflow = 0.0;
    for (long k = 0; k < steps; ++k) {
      double dt = sim.compute_dt();
      if (!(dt > 0.0) || !(dt < std::numeric_limits<double>::infinity())) dt = 1.0;
      sim.step(dt);
      inflow += sim.apply_inflows(now, dt);
      now += dt;
      dt_min = std::min(dt_min, dt);
      dt_max = std::max(dt_max, dt);
      if (adaptive && sim.steps_since_adapt >= sim.adapt_every) {
        sim.adapt(now);
        sim.steps_since_adapt = 0;
      }
      double bx = 0, by = 0;
      if (!sim.finite_state(&bx, &by)) throw fm_gpu::BlowUpError("non-finite state", now);
    }
    std::vector<double> u9;
    sim.download(u9);
    FILE* o = std::fopen(argv[11], "wb");
    if (!o || std::fwrite(u9.data(), sizeof(double), u9.size(), o) != u9.size()) {
      std::fprintf(stderr, "cannot write %s\n", argv[11]);
      return 3;
    }
    std::fclose(o);
    std::printf("{\"cells\": %lld, \"steps\": %ld, \"t\": %.17g, \"dt_min\": %.17g, "
                "\"dt_max\": %.17g, \"volume0\": %.17g, \"volume\": %.17g, \"inflow\": %.17g}\n",
                (long long)sim.cells(), steps, now, dt_min, dt_max, v0, sim.volume(), inflow);
  } catch (const fm_gpu::BlowUpError& e) {
    std::fprintf(stderr, "blow-up at t=%g: %s\n", e.t, e.what());
    return 5;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
