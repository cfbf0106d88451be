"""B200-native K-means Lloyd engine — drop-in for the hot path of the
reference package ``kmeans-regimes`` (arxiv/paper_1402_3788).

Same entry points and result layout as the reference
(assign_step / update_step / converged / iterate / KmeansConfig / KmeansResult,
float64 centres, int64 counts and labels); the arithmetic runs in hand-written
sm_100a CUDA (paper_1402_3788_b200/csrc) behind a C ABI (include/kmeans_b200.h).
There is no CPU fallback: without the built library or an sm_100 device every
compute entry point raises DeviceUnavailableError.
"""

from .engine import (
    DiameterResult,
    KmeansConfig,
    KmeansResult,
    assign_step,
    converged,
    diameter,
    global_centroid_of,
    init_centers,
    iterate,
    run_b200,
    scan_rows,
    update_step,
)
from .estimator import RegimeKMeans
from .exceptions import (
    CapacityExceededError,
    ClusteringError,
    ContractViolationError,
    DataFormatError,
    DegenerateDataError,
    DeviceLostError,
    DeviceUnavailableError,
    DoubleCollectError,
    EmptyClusterError,
    InsufficientDataError,
    NonFiniteValueError,
    OutputMismatchError,
    ParseError,
    RaggedRowsError,
    RegimeNotAllowedError,
    UnknownTicketError,
    ValidationFailureError,
)
from .model import (
    DEFAULT_BLOCK,
    Assignment,
    ClusterModel,
    Dataset,
    Point,
    block_bounds,
    centroid_of,
    distance,
    fold_blocks,
    wcss,
)

__version__ = "0.1.0"

__all__ = [
    "RegimeKMeans", "diameter", "init_centers", "scan_rows",
    "Assignment", "CapacityExceededError", "ClusterModel", "ClusteringError", "ContractViolationError",
    "DataFormatError", "Dataset", "DEFAULT_BLOCK", "DegenerateDataError", "DeviceLostError",
    "DeviceUnavailableError", "DiameterResult", "DoubleCollectError", "EmptyClusterError",
    "InsufficientDataError", "KmeansConfig", "KmeansResult", "NonFiniteValueError", "OutputMismatchError",
    "ParseError", "Point", "RaggedRowsError", "RegimeNotAllowedError", "UnknownTicketError",
    "ValidationFailureError", "assign_step", "block_bounds", "centroid_of", "converged", "distance",
    "fold_blocks", "global_centroid_of", "iterate", "run_b200", "update_step", "wcss",
]
