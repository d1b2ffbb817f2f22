// Explicit instantiations of the kernels for 1 padded/head 8-state tiles.
#define THMM_DEFINE_LAUNCHERS
#include "thmm_launch.cuh"

namespace thmm {
THMM_INSTANTIATE_NT(1)
THMM_INSTANTIATE_TAILS(1)
}  // namespace thmm
