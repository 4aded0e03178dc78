// Dynamically adaptive MWDG2 / HWFV1 on the device (solver_adaptive.cpp).
#include "fm_device.cuh"
#include "fm_sim.hpp"

namespace fmh {

struct AdaptState {};

void adaptive_destroy(AdaptState* a) { delete a; }

void adaptive_init(Sim&, const fm_sim_desc*, const fm_raster*) {
  throw Error(FM_ERR_OTHER, "adaptive solvers: not built yet");
}
void adaptive_adapt(Sim&, double) { throw Error(FM_ERR_OTHER, "adaptive solvers: not built yet"); }

}  // namespace fmh
