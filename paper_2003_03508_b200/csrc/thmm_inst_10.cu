// Explicit instantiations of the kernels for 10 padded/head 8-state tiles.
#define THMM_DEFINE_LAUNCHERS
#include "thmm_launch.cuh"

namespace thmm {
THMM_INSTANTIATE_NT(10)

THMM_INSTANTIATE_RUNS(10, false, 0)
THMM_INSTANTIATE_RUNS(10, true, 0)
}  // namespace thmm
