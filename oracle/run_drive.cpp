// run_drive — the reference's OWN batch driver with the GPU solvers plugged in.
//
// TEST INFRASTRUCTURE (oracle/): built by `make -C oracle ref` into
// oracle/_ref/run_drive from the reference's unmodified sources where they lie
// under /root/reference (never copied into this repository).
//
// This translation unit compiles the reference's run.cpp itself
// (proj/core/src/run.cpp, included below) so that its anonymous-namespace
// template drive<Sim> (run.cpp:35-141) is instantiated with the drop-in
// classes of include/fm_gpu.hpp — fm_gpu::UniformSim / NonUniformSim /
// AdaptiveSim — exactly as INTEGRATION.md's maintainer patch does inside
// run_scenario (run.cpp:145-164).  Every output drive writes (stats.txt, gauge
// CSVs, depth/qx/qy ASCII rasters, elements.csv, the per-output .nug dumps)
// therefore comes from the reference's code on both arms.
//
//   run_drive ref|gpu CONFIG OUTPUT_DIR
//
// `ref` runs the unmodified run_scenario; `gpu` runs run_scenario_gpu below.
// Exit codes follow the reference CLI (tools/floodmra.cpp:171-186):
// 2 config, 3 I/O / parse, 4 blow-up, 1 other.
#define FM_GPU_WITH_FLOODMRA 1
#include "fm_gpu.hpp"

#include "src/run.cpp"  // the reference's run.cpp, verbatim, from -I$(REF_ROOT)
#include "floodmra/metrics.hpp"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

namespace floodmra {

// run_scenario (run.cpp:145-164) with each reference sim replaced by its
// GPU drop-in; the dispatch is the reference's.
RunResult run_scenario_gpu(const ScenarioConfig& cfg) {
  fm_gpu::check(fm_init(0));
  const Raster dem = read_ascii_grid(cfg.dem_path);
  if (solver_is_adaptive(cfg.solver)) {
    fm_gpu::AdaptiveSim sim(cfg, dem);
    return drive(sim, cfg, dem);
  }
  if (cfg.grid_mode == GridMode::nonuniform || !cfg.grid_file.empty()) {
    fm_gpu::NonUniformSim sim(cfg, dem);
    return drive(sim, cfg, dem);
  }
  fm_gpu::UniformSim sim(cfg, dem);
  return drive(sim, cfg, dem);
}

}  // namespace floodmra

int main(int argc, char** argv) {
  if (argc == 5 && std::strcmp(argv[1], "compare") == 0) {
    // the reference's own post-processing (metrics.cpp:100-143) of two run
    // directories: rmse of every gauge (h, eta, speed) and the extent
    // metrics of every depth raster
    try {
      const floodmra::CompareReport r = floodmra::compare_runs(argv[2], argv[3], std::atof(argv[4]));
      for (const auto& row : r.rows)
        std::printf("%s %s %s %.17g %d\n", row.kind.c_str(), row.id.c_str(), row.metric.c_str(), row.value,
                    row.absent ? 1 : 0);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "compare error: %s\n", e.what());
      return 3;
    }
    return 0;
  }
  if (argc != 4 || (std::strcmp(argv[1], "ref") && std::strcmp(argv[1], "gpu"))) {
    std::fprintf(stderr, "usage: %s ref|gpu CONFIG OUTPUT_DIR | compare TEST_DIR REF_DIR WET\n", argv[0]);
    return 2;
  }
  try {
    floodmra::ScenarioConfig cfg = floodmra::read_config(argv[2]);
    cfg.output_dir = argv[3];
    const floodmra::RunResult r = std::strcmp(argv[1], "gpu") == 0 ? floodmra::run_scenario_gpu(cfg)
                                                                   : floodmra::run_scenario(cfg);
    std::printf("steps=%lld outputs=%d\n", (long long)r.stats.steps, r.outputs_written);
  } catch (const floodmra::ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  } catch (const floodmra::ParseError& e) {
    std::fprintf(stderr, "parse error: %s\n", e.what());
    return 3;
  } catch (const floodmra::IoError& e) {
    std::fprintf(stderr, "I/O error: %s\n", e.what());
    return 3;
  } catch (const floodmra::BlowUpError& e) {
    std::fprintf(stderr, "blow-up at t=%.17g: %s\n", e.t, e.what());
    return 4;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
