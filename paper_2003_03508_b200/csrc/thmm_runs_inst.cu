// Explicit instantiations of the run-absorbing FP64 chain (thmm_runs.cuh) for
// 1..4 padded 8-state tiles (K <= 32: the table of powers fits next to two
// CTAs per SM).
#define THMM_DEFINE_LAUNCHERS
#include "thmm_launch.cuh"

namespace thmm {
THMM_INSTANTIATE_RUNS(1, false)
THMM_INSTANTIATE_RUNS(1, true)
THMM_INSTANTIATE_RUNS(2, false)
THMM_INSTANTIATE_RUNS(2, true)
THMM_INSTANTIATE_RUNS(3, false)
THMM_INSTANTIATE_RUNS(3, true)
THMM_INSTANTIATE_RUNS(4, false)
THMM_INSTANTIATE_RUNS(4, true)
}  // namespace thmm
