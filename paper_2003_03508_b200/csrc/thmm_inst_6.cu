// Explicit instantiations of the kernels for 6 padded/head 8-state tiles.
#define THMM_DEFINE_LAUNCHERS
#include "thmm_launch.cuh"

namespace thmm {
THMM_INSTANTIATE_NT(6)
THMM_INSTANTIATE_TAILS(6)
}  // namespace thmm
