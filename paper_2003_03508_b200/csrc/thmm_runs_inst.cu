// Explicit instantiations of the run-absorbing FP64 chain (thmm_runs.cuh) and
// of the row-stacked vector kernels that share its column split
// (thmm_vec.cuh: stitched chain, collapse continuation) for padded K <= 32:
// plain variants of 1..4 padded tiles, head/tail variants of 1..3 head tiles
// with 1..4 tail states.
#define THMM_DEFINE_LAUNCHERS
#include "thmm_launch.cuh"

namespace thmm {
THMM_INSTANTIATE_RUNS(1, false, 0)
THMM_INSTANTIATE_RUNS(1, true, 0)
THMM_INSTANTIATE_RUNS(2, false, 0)
THMM_INSTANTIATE_RUNS(2, true, 0)
THMM_INSTANTIATE_RUNS(3, false, 0)
THMM_INSTANTIATE_RUNS(3, true, 0)
THMM_INSTANTIATE_RUNS(4, false, 0)
THMM_INSTANTIATE_RUNS(4, true, 0)
THMM_INSTANTIATE_RUNS(1, false, 1)
THMM_INSTANTIATE_RUNS(1, false, 2)
THMM_INSTANTIATE_RUNS(1, false, 3)
THMM_INSTANTIATE_RUNS(1, false, 4)
THMM_INSTANTIATE_RUNS(2, false, 1)
THMM_INSTANTIATE_RUNS(2, false, 2)
THMM_INSTANTIATE_RUNS(2, false, 3)
THMM_INSTANTIATE_RUNS(2, false, 4)
THMM_INSTANTIATE_RUNS(3, false, 1)
THMM_INSTANTIATE_RUNS(3, false, 2)
THMM_INSTANTIATE_RUNS(3, false, 3)
THMM_INSTANTIATE_RUNS(3, false, 4)
}  // namespace thmm
