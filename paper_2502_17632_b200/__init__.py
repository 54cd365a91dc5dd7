"""paper_2502_17632_b200: B200-native GiFt initial-placement hot path.

A drop-in for the hot path of the reference `giftplace` package (arXiv
2502.17632): netlist -> clique graph -> degrees / augmented normalisation ->
multi-resolution SpMM filter bank -> re-pin / clamp, all in hand-written
sm_100a CUDA (libgiftb200.so, C ABI in include/gift_b200.h).  Same names,
argument meaning and exception classes as `giftplace/__init__.py:26-38`.
"""

from .bookshelf import aux_files, parse_design, read_design
from .errors import (
    DanglingPinError,
    DeviceError,
    DimensionMismatchError,
    DuplicateCellError,
    MalformedLineError,
    MissingFileError,
    GiftPlaceError,
    IsolatedNodeError,
    NonSymmetricError,
    TooLargeForDenseError,
    ZeroSignalError,
)
from .gift import (
    DEFAULT_TERMS,
    JITTER_REGION_FRACTION,
    GiftConfig,
    gift_filter,
    gift_place,
    gift_place_arrays,
    initial_signal,
)
from .graph import (
    DENSE_LIMIT,
    FilterTerm,
    SparseSymMatrix,
    apply_operator_power,
    as_device_matrix,
    build_clique_graph,
    from_coo,
    normalized_augmented_adjacency,
)
from .metrics import hpwl, laplacian, quadratic_wirelength, rayleigh_smoothness
from .netlist import Cell, Design, FlatDesign, Net, Pin, Region, Row
from .plio import PL_PRECISION, format_placement, write_placement
from ._lib import set_tiled_policy

__version__ = "0.1.0"

__all__ = [
    "DEFAULT_TERMS", "DENSE_LIMIT", "PL_PRECISION", "format_placement", "write_placement",
    "DanglingPinError", "DuplicateCellError", "MalformedLineError", "MissingFileError", "aux_files",
    "parse_design", "read_design", "JITTER_REGION_FRACTION", "Cell", "Design", "DeviceError",
    "DimensionMismatchError", "FilterTerm", "FlatDesign", "GiftConfig", "GiftPlaceError", "IsolatedNodeError",
    "Net", "NonSymmetricError", "Pin", "Region", "Row", "SparseSymMatrix", "TooLargeForDenseError",
    "apply_operator_power", "as_device_matrix", "build_clique_graph", "from_coo", "gift_filter", "gift_place",
    "gift_place_arrays", "hpwl", "initial_signal", "laplacian", "normalized_augmented_adjacency",
    "quadratic_wirelength", "rayleigh_smoothness", "ZeroSignalError", "set_tiled_policy",
]
