// Explicit instantiations of the kernels for 4 padded/head 8-state tiles.
#define THMM_DEFINE_LAUNCHERS
#include "thmm_launch.cuh"

namespace thmm {
THMM_INSTANTIATE_NT(4)
THMM_INSTANTIATE_TAILS(4)
THMM_INSTANTIATE_RUNS(4, false, 1)
THMM_INSTANTIATE_RUNS(4, false, 2)
THMM_INSTANTIATE_RUNS(4, false, 3)
THMM_INSTANTIATE_RUNS(4, false, 4)
}  // namespace thmm
