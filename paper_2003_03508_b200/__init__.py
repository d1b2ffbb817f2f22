"""B200-native parallel HMM forward log-likelihood (arXiv 2003.03508).

Drop-in for the likelihood engine of the reference package ``tremorhmm``:
the same public names as ``tremorhmm.engine`` (and the core types it needs),
backed by hand-written sm_100a FP64 tensor-core kernels through the C-ABI in
include/thmm.h.  See DESIGN.md.
"""

from .engine import (
    MAX_PARALLEL_STATES,
    DeviceObservations,
    EngineConfig,
    SegmentProduct,
    batch_emissions,
    combine_segments,
    default_device,
    fold_nodes,
    padded_states,
    parallel_loglik,
    parallel_loglik_batch,
    scale_by_emission,
    segment_bounds,
    segment_chain_product,
    set_default_device,
    _parallel_loglik_arrays,
)
from .model import (
    LOG_2PI,
    HmmParams,
    Observation,
    ScaledMatrix,
    StateEmission,
    observation_arrays,
    pack_params,
)

__version__ = "0.1.0"

__all__ = [name for name in dir() if not name.startswith("_")] + ["_parallel_loglik_arrays"]
