// Explicit instantiations of the kernels for 5 padded/head 8-state tiles.
#define THMM_DEFINE_LAUNCHERS
#include "thmm_launch.cuh"

namespace thmm {
THMM_INSTANTIATE_NT(5)
THMM_INSTANTIATE_TAILS(5)
THMM_INSTANTIATE_RUNS(5, false, 0)
THMM_INSTANTIATE_RUNS(5, true, 0)
THMM_INSTANTIATE_RUNS(5, false, 1)
THMM_INSTANTIATE_RUNS(5, false, 2)
THMM_INSTANTIATE_RUNS(5, false, 3)
THMM_INSTANTIATE_RUNS(5, false, 4)
}  // namespace thmm
