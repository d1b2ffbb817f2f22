// Explicit instantiations of the kernels for 5 padded/head 8-state tiles.
#define THMM_DEFINE_LAUNCHERS
#include "thmm_launch.cuh"

namespace thmm {
THMM_INSTANTIATE_NT(5)
THMM_INSTANTIATE_TAILS(5)
}  // namespace thmm
