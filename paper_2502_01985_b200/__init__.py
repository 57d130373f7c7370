"""B200-native factorized learning over normalized (DI-metadata) matrices.

Drop-in for the hot path of the reference package `factorlearn`
(arXiv 2502.01985, "Ilargi"): the `TargetHandle` operator surface
(`pkg/src/factorlearn/ops.py:147-328`) and the GD trainers
(`pkg/src/factorlearn/trainers.py`), re-implemented as hand-written sm_100a
CUDA kernels behind a C ABI (`include/fl_b200.h`).  There is no CPU fallback.
"""

from .metadata import (JOIN_TYPES, FactorizedTable, IndicatorMatrix,
                       MappingMatrix, MetadataError, ValidationReport,
                       block_mapping, fk_indicator, redundancy_stats)
from .ops import OpError, TargetHandle, export_trace_csv
from .sparse import OpTrace, ShapeError, SparseMatrix, SparseStructureError, as_dense
from . import costmodel, formats
from .trainers import (ConfigError, DivergenceError, TrainConfig, TrainResult,
                       gaussian_nmf, kmeans, linear_regression,
                       logistic_regression, train)

__version__ = "0.1.0"


def materialize(ft, *, threads: int = 1, trace: OpTrace | None = None, check: bool = True,
                device: int = 0) -> SparseMatrix:
    """The join result T = sum_k I_k S_k M_k^T (reference `metadata.py:215-225`,
    same signature), computed on the device; values are exact copies of the
    sources.  `threads` is accepted for API parity (the GPU ignores it); the
    join's work is recorded into `trace` when one is given."""
    h = TargetHandle.factorized(ft, threads=threads, check=check, device=device)
    out = h.materialize_target(traced=trace is not None)
    if trace is not None:
        trace.merge(h.trace)
    return out


__all__ = ["as_dense", "costmodel", "formats", "ConfigError", "DivergenceError", "FactorizedTable", "IndicatorMatrix",
           "JOIN_TYPES", "MappingMatrix", "MetadataError", "OpError", "OpTrace",
           "ShapeError", "SparseMatrix", "SparseStructureError", "TargetHandle",
           "TrainConfig", "TrainResult", "ValidationReport", "block_mapping",
           "export_trace_csv", "fk_indicator", "gaussian_nmf", "kmeans",
           "linear_regression", "logistic_regression", "materialize",
           "redundancy_stats", "train"]
