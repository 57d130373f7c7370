"""Training data for the reference's factorize-vs-materialize estimator,
regenerated from B200 timings (BASELINE.json configs[4]).

The reference decides per (dataset, model, hardware) whether to train on the
factorized or the materialized target with a gradient-boosted classifier over
a fixed 33-entry feature vector (reference `features.py:22-45`), trained on a
corpus of `LabeledRun`s written as CSV (`estimator.py:54-61`).  This module
restates exactly what is needed to emit that corpus from our own B200
timings, so the reference's estimator (or any user of its corpus format)
retrains on B200 data unchanged:

* the analytic operator-cost model (`cost.py:116-244`: visit counts of the
  row-times-column multiply with dense bounds for iteration operands, bytes
  = 8 * visits * 1.5 read and 8 * output written, per-model operator
  manifests), restated here as plain arithmetic;
* `extract_features` (`features.py:88-121`) in the reference's order;
* the TR&FR baseline decision recorded with every run
  (`estimator.py:148-166`);
* `write_corpus` with the reference header (`estimator.py:54-61`).

Hardware group: `parallelism` = streaming multiprocessors x GPUs (the unit of
parallel work on the device, where the reference counts CPU threads) and
`memory_bandwidth` = the measured HBM copy bandwidth in bytes/s.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass

import numpy as np

ELEMENT_SIZE = 8          # cost.py:20
INDEX_OVERHEAD = 1.5      # cost.py:21
MODELS = ("linreg", "logreg", "kmeans", "gnmf")          # cost.py:23
JOIN_TYPES = ("inner", "left", "outer", "union")          # metadata.py:22
TUPLE_RATIO_THRESHOLD = 5.0                               # estimator.py:22
FEATURE_RATIO_THRESHOLD = 1.0                             # estimator.py:23

FEATURE_NAMES = (                                         # features.py:22-41
    "r_T", "c_T", "n_sources", "sum_r_k", "sum_c_k", "sparsity_T",
    "tuple_ratio_min", "tuple_ratio_max",
    "feature_ratio_min", "feature_ratio_max", "rho_c",
    "join_inner", "join_left", "join_outer", "join_union",
    "complexity_ratio", "o_materialized", "o_factorized",
    "bytes_read_mat", "bytes_written_mat",
    "bytes_read_fact", "bytes_written_fact",
    "iterations",
    "model_linreg", "model_logreg", "model_kmeans", "model_gnmf",
    "parallelism", "memory_bandwidth",
    "o_mat_per_thread", "o_fact_per_thread",
    "bytes_mat_over_bw", "bytes_fact_over_bw",
)
N_FEATURES = len(FEATURE_NAMES)
assert N_FEATURES == 33


class CostModelError(ValueError):
    pass


@dataclass(frozen=True)
class Source:
    rows: int
    cols: int
    nnz: int


@dataclass(frozen=True)
class Profile:
    """Shape summary of a factorized target (reference `DatasetProfile`,
    features.py:53-66): target extents, sources, join type, redundancy."""

    r_t: int
    c_t: int
    m_t: int
    sources: tuple
    join_type: str
    tuple_ratios: tuple
    feature_ratios: tuple
    sparsity: float
    rho_c: float
    replicated: tuple = ()    # (tuple ratio, feature ratio) of sources with fanout > 1

    @classmethod
    def from_table(cls, ft) -> "Profile":
        """From a `metadata.FactorizedTable` (host arithmetic on metadata)."""
        from .metadata import redundancy_stats
        st = redundancy_stats(ft)
        srcs = tuple(Source(s.n_rows, s.n_cols, s.nnz) for s in ft.sources)
        rep = tuple((ft.r_T / s.n_rows, ft.c_T / s.n_cols)
                    for s, ind in zip(ft.sources, ft.indicators)
                    if ind.fanout().max(initial=0) > 1)
        return cls(ft.r_T, ft.c_T, ft.target_nnz(), srcs, ft.join_type, st.tuple_ratios,
                   st.feature_ratios, st.sparsity_target, st.rho_c, rep)

    @classmethod
    def star(cls, r_fact: int, c_fact: int, dims) -> "Profile":
        """Dense inner-join star: fact r_fact x c_fact (1:1) plus dimensions
        [(rows, cols)] each referenced by every fact row."""
        c_t = c_fact + sum(c for _, c in dims)
        srcs = (Source(r_fact, c_fact, r_fact * c_fact),) + tuple(
            Source(r, c, r * c) for r, c in dims)
        m_t = r_fact * c_t
        rep = tuple((r_fact / r, c_t / c) for r, c in dims if r < r_fact)
        return cls(r_fact, c_t, m_t, srcs, "inner",
                   tuple(r_fact / s.rows for s in srcs), tuple(c_t / s.cols for s in srcs),
                   1.0 - m_t / (r_fact * c_t), sum(s.cols for s in srcs) / c_t, rep)


# ---------------------------------------------------------------------------
# analytic cost model (cost.py:116-244)
# ---------------------------------------------------------------------------
_UNARY = ("elementwise", "rowsum", "colsum")


def op_cost(op: str, p: Profile, r_x: int = 0, c_x: int = 0, *, mat: bool) -> int:
    """Visit count of one operator (cost.py:116-141)."""
    m_x = r_x * c_x
    if op in _UNARY:
        return p.m_t if mat else sum(s.nnz for s in p.sources)
    if op == "lmm":
        return (c_x * p.m_t + p.r_t * m_x) if mat else sum(c_x * s.nnz + s.rows * m_x
                                                          for s in p.sources)
    if op == "rmm":
        return (r_x * p.m_t + p.c_t * m_x) if mat else sum(r_x * s.nnz + s.cols * m_x
                                                          for s in p.sources)
    if op == "transpose_lmm":
        return (c_x * p.m_t + p.c_t * m_x) if mat else sum(c_x * s.nnz + s.cols * m_x
                                                          for s in p.sources)
    raise CostModelError(f"unknown operator tag {op!r}")


def _output_size(op: str, p: Profile, r_x: int, c_x: int, mat: bool) -> int:
    """cost.py:144-159."""
    if op == "lmm":
        return p.r_t * c_x
    if op == "rmm":
        return r_x * p.c_t
    if op == "transpose_lmm":
        return p.c_t * c_x
    if op == "elementwise":
        return p.m_t if mat else sum(s.nnz for s in p.sources)
    if op == "rowsum":
        return p.r_t
    if op == "colsum":
        return p.c_t
    raise CostModelError(f"unknown operator tag {op!r}")


def model_sequence(model: str, p: Profile, iterations: int, k: int, rank: int):
    """The operator manifest of each trainer (cost.py:176-200)."""
    r_t, c_t = p.r_t, p.c_t
    if model in ("linreg", "logreg"):
        return [(("lmm", c_t, 1), iterations), (("transpose_lmm", r_t, 1), iterations)]
    if model == "kmeans":
        return [(("rmm", k, r_t), 1), (("elementwise", 0, 0), 1), (("rowsum", 0, 0), 1),
                (("lmm", c_t, k), iterations), (("transpose_lmm", r_t, k), iterations)]
    if model == "gnmf":
        return [(("rowsum", 0, 0), 1), (("rmm", rank, r_t), iterations),
                (("lmm", c_t, rank), iterations)]
    raise CostModelError(f"unknown model {model!r}; one of {MODELS}")


@dataclass
class Cost:
    o_mat: int
    o_fact: int
    read_mat: float
    written_mat: float
    read_fact: float
    written_fact: float

    @property
    def complexity_ratio(self) -> float:          # cost.py:94-98
        if self.o_fact == 0:
            return float("inf") if self.o_mat else 1.0
        return self.o_mat / self.o_fact


def model_cost(model: str, p: Profile, iterations: int, k: int, rank: int) -> Cost:
    """cost.py:203-228 (op costs summed per operator tag, then over tags, in
    manifest order -- the same integer totals)."""
    seq = model_sequence(model, p, iterations, k, rank)
    out = []
    for mat in (True, False):
        by_op: dict = {}
        reads = writes = 0.0
        for (op, r_x, c_x), times in seq:
            visits = op_cost(op, p, r_x, c_x, mat=mat)
            by_op[op] = by_op.get(op, 0) + times * visits
            reads += times * ELEMENT_SIZE * INDEX_OVERHEAD * visits
            writes += times * ELEMENT_SIZE * _output_size(op, p, r_x, c_x, mat)
        out.append((sum(by_op.values()), reads, writes))
    (om, rm, wm), (of, rf, wf) = out
    return Cost(om, of, rm, wm, rf, wf)


def extract_features(p: Profile, model: str, iterations: int, k: int, rank: int,
                     parallelism: int, memory_bandwidth: float) -> np.ndarray:
    """The 33-entry vector in FEATURE_NAMES order (features.py:88-121)."""
    if model not in MODELS:
        raise CostModelError(f"unknown model {model!r}")
    if p.join_type not in JOIN_TYPES:
        raise CostModelError(f"unknown join type {p.join_type!r}")
    cp = model_cost(model, p, iterations, k, rank)
    bytes_mat = cp.read_mat + cp.written_mat
    bytes_fact = cp.read_fact + cp.written_fact
    v = [
        float(p.r_t), float(p.c_t), float(len(p.sources)),
        float(sum(s.rows for s in p.sources)), float(sum(s.cols for s in p.sources)),
        p.sparsity, min(p.tuple_ratios), max(p.tuple_ratios),
        min(p.feature_ratios), max(p.feature_ratios), p.rho_c,
        *(1.0 if p.join_type == j else 0.0 for j in JOIN_TYPES),
        cp.complexity_ratio, float(cp.o_mat), float(cp.o_fact),
        cp.read_mat, cp.written_mat, cp.read_fact, cp.written_fact,
        float(iterations),
        *(1.0 if model == m else 0.0 for m in MODELS),
        float(parallelism), float(memory_bandwidth),
        cp.o_mat / parallelism, cp.o_fact / parallelism,
        bytes_mat / memory_bandwidth, bytes_fact / memory_bandwidth,
    ]
    out = np.asarray(v, dtype=np.float64)
    if not np.all(np.isfinite(out)):
        raise CostModelError("non-finite feature value (empty or degenerate table?)")
    return out


def tr_fr_decision(p: Profile) -> str:
    """TR&FR baseline over the replicated sources (estimator.py:128-166):
    factorize iff min TR > 5 and min FR > 1; no replicated source ->
    materialize."""
    if not p.replicated:
        return "materialize"
    trs = [t for t, _ in p.replicated]
    frs = [f for _, f in p.replicated]
    if min(trs) > TUPLE_RATIO_THRESHOLD and min(frs) > FEATURE_RATIO_THRESHOLD:
        return "factorize"
    return "materialize"


def write_corpus(path, runs) -> None:
    """runs: iterable of (features, t_fact, t_mat, tr_fr); label = t_fact <
    t_mat.  The reference's corpus format (estimator.py:54-61), readable by
    its `read_corpus`."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(list(FEATURE_NAMES) + ["label", "t_fact", "t_mat", "tr_fr"])
        for f, t_fact, t_mat, tr_fr in runs:
            w.writerow([repr(float(v)) for v in f]
                       + [int(t_fact < t_mat), repr(float(t_fact)), repr(float(t_mat)), tr_fr])


__all__ = ["FEATURE_NAMES", "MODELS", "CostModelError", "Profile", "Source", "extract_features",
           "model_cost", "op_cost", "tr_fr_decision", "write_corpus"]
