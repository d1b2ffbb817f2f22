// Explicit instantiations of the kernels for 7 padded/head 8-state tiles.
#define THMM_DEFINE_LAUNCHERS
#include "thmm_launch.cuh"

namespace thmm {
THMM_INSTANTIATE_NT(7)
THMM_INSTANTIATE_TAILS(7)
THMM_INSTANTIATE_RUNS(7, false, 0)
THMM_INSTANTIATE_RUNS(7, true, 0)
THMM_INSTANTIATE_RUNS(7, false, 1)
THMM_INSTANTIATE_RUNS(7, false, 2)
THMM_INSTANTIATE_RUNS(7, false, 3)
THMM_INSTANTIATE_RUNS(7, false, 4)
}  // namespace thmm
