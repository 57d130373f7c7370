"""CPU oracle for the factorized-learning hot path -- TEST INFRASTRUCTURE ONLY.

This package is a float64 numpy restatement of the reference's algorithm
(`/root/reference/pkg/src/factorlearn/{ops,trainers,metadata}.py`).  Each
function cites the reference file:line it follows.  It is pinned against the
golden vectors in `tests/golden/` that were produced by running the real
reference (`tests/golden/make_golden.py`, run in the build container where
`/root/reference` exists).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline`
leg and `--impl reference`) may import this package, and only as the checker
or the timed CPU baseline -- never as the product path.  The product path
(`paper_2502_01985_b200`) never imports it and fails loudly when its CUDA
library is missing.
"""

from .reference_ops import (OracleTable, build_selectors, col_sum, elementwise,
                            lmm, materialize, rmm, row_sum, transpose_lmm)
from .reference_trainers import (gaussian_nmf, kmeans, linear_regression,
                                 logistic_regression, safe_learning_rate,
                                 train)

__all__ = ["OracleTable", "build_selectors", "col_sum", "elementwise",
           "gaussian_nmf", "kmeans", "linear_regression", "lmm",
           "logistic_regression", "materialize", "rmm", "row_sum",
           "safe_learning_rate", "train", "transpose_lmm"]
