// Explicit instantiations of the kernels for 9 padded/head 8-state tiles.
#define THMM_DEFINE_LAUNCHERS
#include "thmm_launch.cuh"

namespace thmm {
THMM_INSTANTIATE_NT(9)
THMM_INSTANTIATE_TAILS(9)
THMM_INSTANTIATE_RUNS(9, false, 0)
THMM_INSTANTIATE_RUNS(9, true, 0)
THMM_INSTANTIATE_RUNS(9, false, 1)
THMM_INSTANTIATE_RUNS(9, false, 2)
THMM_INSTANTIATE_RUNS(9, false, 3)
THMM_INSTANTIATE_RUNS(9, false, 4)
}  // namespace thmm
