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

#include <cstdio>
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
  if (argc != 4 || (std::strcmp(argv[1], "ref") && std::strcmp(argv[1], "gpu"))) {
    std::fprintf(stderr, "usage: %s ref|gpu CONFIG OUTPUT_DIR\n", argv[0]);
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
