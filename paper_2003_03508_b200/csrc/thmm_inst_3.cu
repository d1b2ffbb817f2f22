// Explicit instantiations of the kernels for 3 padded/head 8-state tiles.
#define THMM_DEFINE_LAUNCHERS
#include "thmm_launch.cuh"

namespace thmm {
THMM_INSTANTIATE_NT(3)
THMM_INSTANTIATE_TAILS(3)
}  // namespace thmm
