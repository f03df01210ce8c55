"""B200-native lower-bound collection for the bin_packing feasibility check
(arXiv 2402.14821).  Drop-in for the reference's bound engine
(/root/reference/pkg/src/binpack/bounds.py, parallel.py): the sweeps run in
libbplb.so (hand-written sm_100a CUDA behind a C ABI, include/bplb.h)."""

from .bounds import (
    DEFAULT_DFF_ORDER,
    VB2_ACCUMULATOR_MAX,
    BoundResult,
    DffKind,
    L2Partition,
    LambdaRange,
    dff_bound,
    dff_bound_batch,
    dff_value,
    l1,
    l2,
    l2_partition,
    l2_value,
    lambda_range,
    lower_bound_seq,
)
from .instances import ArrayReducedInstance, ReducedInstance, reduce_packing_arrays
from .parallel import (GpuBoundEngine, ParallelBoundEngine, SharedMax, default_workers, lower_bound_multi,
                       lower_bound_par)
from .batch import (csr_from_lists, lower_bound_batch, lower_bound_batch_assign, lower_bound_batch_multi, open_marker,
                    reduce_packing_batch)

from .knapsack import KnapsackBatch, install_knapsack_gpu, knapsack_bins

__version__ = "0.1.0"

__all__ = [
    "ArrayReducedInstance",
    "KnapsackBatch",
    "install_knapsack_gpu",
    "knapsack_bins",
    "BoundResult",
    "DEFAULT_DFF_ORDER",
    "DffKind",
    "GpuBoundEngine",
    "L2Partition",
    "LambdaRange",
    "ParallelBoundEngine",
    "ReducedInstance",
    "SharedMax",
    "VB2_ACCUMULATOR_MAX",
    "csr_from_lists",
    "default_workers",
    "dff_bound",
    "dff_bound_batch",
    "dff_value",
    "l1",
    "l2",
    "l2_partition",
    "l2_value",
    "lambda_range",
    "lower_bound_batch",
    "lower_bound_batch_assign",
    "lower_bound_batch_multi",
    "open_marker",
    "reduce_packing_batch",
    "lower_bound_par",
    "lower_bound_multi",
    "lower_bound_seq",
    "reduce_packing_arrays",
    "__version__",
]
