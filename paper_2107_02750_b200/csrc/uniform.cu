// Uniform-raster DG2/FV1/ACC (solver_uniform.cpp) on the device.
#include "fm_device.cuh"
#include "fm_sim.hpp"

namespace fmh {

void uniform_init(Sim&, const fm_sim_desc*, const fm_raster*) {
  throw Error(FM_ERR_OTHER, "uniform solvers: not built yet");
}
void un_launch_step(Sim&, bool, double, int*) { throw Error(FM_ERR_OTHER, "uniform: not built"); }
void un_launch_reduce_init(Sim&) { throw Error(FM_ERR_OTHER, "uniform: not built"); }

}  // namespace fmh
