"""Generate golden fixtures by running the REAL reference (factorlearn).

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src,
builds tables whose values are float32-representable (so the fp32 device
storage is exact), runs the reference's own TargetHandle operators, selector
derivation and trainers, and writes small .npz fixtures next to this script.
The fixtures travel with the repo; nothing on the GPU box reads
/root/reference.

Tables:
  two_source   conftest.py:12-31 (golden literal, 4x4)
  outer        conftest.py:34-50 (golden literal, 5x4 with padding row)
  gen_<join>_<n>_<seed>   datagen.generate(GenSpec(...)), values rounded to fp32
  star         2-source star: fact 3000x6 + dim 30x5, permuted round-robin FK
  star3        3-source star: fact 2400x5 + dims 40x7, 8x3
  clusters     planted well-separated clusters (K-means assignment parity)
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from factorlearn import ops as rops  # noqa: E402
from factorlearn.datagen import GenError, GenSpec, generate  # noqa: E402
from factorlearn.metadata import (FactorizedTable, IndicatorMatrix,  # noqa: E402
                                  MappingMatrix, materialize)
from factorlearn.ops import TargetHandle  # noqa: E402
from factorlearn.sparse import SparseMatrix  # noqa: E402
from factorlearn.trainers import TrainConfig, train  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def round_table(ft):
    """Same structure, source values rounded to float32 (exactly representable)."""
    srcs = []
    for s in ft.sources:
        srcs.append(SparseMatrix(s.n_rows, s.n_cols, s.indptr, s.indices,
                                 f32(s.data)))
    return FactorizedTable(srcs, ft.mappings, ft.indicators, ft.join_type,
                           ft.r_T, ft.c_T)


def two_source():
    s1 = SparseMatrix.from_dense([[1, 2], [3, 4], [5, 6], [7, 8]])
    s2 = SparseMatrix.from_dense([[10, 0], [30, 40]])
    m1 = MappingMatrix(SparseMatrix.from_dense([[1, 0], [0, 1], [0, 0], [0, 0]]))
    m2 = MappingMatrix(SparseMatrix.from_dense([[0, 0], [0, 0], [1, 0], [0, 1]]))
    i1 = IndicatorMatrix(SparseMatrix.identity(4))
    i2 = IndicatorMatrix(SparseMatrix.from_dense([[1, 0], [1, 0], [0, 1], [0, 1]]))
    return FactorizedTable([s1, s2], [m1, m2], [i1, i2], "inner", 4, 4)


def outer():
    s1 = SparseMatrix.from_dense([[1, 2], [3, 4], [5, 6], [7, 8]])
    s2 = SparseMatrix.from_dense([[10, 0], [30, 40]])
    m1 = MappingMatrix(SparseMatrix.from_dense([[1, 0], [0, 1], [0, 0], [0, 0]]))
    m2 = MappingMatrix(SparseMatrix.from_dense([[0, 0], [0, 0], [1, 0], [0, 1]]))
    i1 = IndicatorMatrix(SparseMatrix.from_dense(
        [[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1], [0, 0, 0, 0]]))
    i2 = IndicatorMatrix(SparseMatrix.from_dense([[1, 0], [1, 0], [0, 1], [0, 1], [0, 0]]))
    return FactorizedTable([s1, s2], [m1, m2], [i1, i2], "outer", 5, 4)


def star(seed, r_fact, dims, c_fact, value_fn=None):
    """Star schema built from the reference's own types, as SURVEY.md §7
    step 1 prescribes: identity fact indicator, permuted round-robin FKs."""
    rng = np.random.default_rng(seed)
    c_t = c_fact + sum(c for _, c in dims)
    vals = value_fn(rng) if value_fn else None
    srcs, maps, inds = [], [], []
    fact = f32(rng.random((r_fact, c_fact))) if vals is None else vals[0]
    srcs.append(SparseMatrix.from_dense(fact))
    maps.append(MappingMatrix(SparseMatrix.from_coo(
        c_t, c_fact, np.arange(c_fact), np.arange(c_fact), np.ones(c_fact))))
    inds.append(IndicatorMatrix(SparseMatrix.identity(r_fact)))
    off = c_fact
    for d, (r_d, c_d) in enumerate(dims):
        dim = f32(rng.random((r_d, c_d))) if vals is None else vals[1 + d]
        fk = rng.permutation(np.arange(r_fact) % r_d)
        srcs.append(SparseMatrix.from_dense(dim))
        maps.append(MappingMatrix(SparseMatrix.from_coo(
            c_t, c_d, off + np.arange(c_d), np.arange(c_d), np.ones(c_d))))
        inds.append(IndicatorMatrix(SparseMatrix.from_coo(
            r_fact, r_d, np.arange(r_fact), fk, np.ones(r_fact))))
        off += c_d
    return FactorizedTable(srcs, maps, inds, "inner", r_fact, c_t)


def clusters(seed=5, r_fact=1200, k=4):
    """Planted clusters: each fact row belongs to cluster (row % k); the
    fact source and the dim rows carry well-separated centres."""
    rng = np.random.default_rng(seed)
    c_fact, r_d, c_d = 4, 24, 3
    centres_f = rng.random((k, c_fact)) * 10
    lab = rng.permutation(np.arange(r_fact) % k)
    fact = f32(centres_f[lab] + 0.01 * rng.standard_normal((r_fact, c_fact)) + 20)
    # dim rows are grouped so that every dim row serves exactly one cluster
    dim_cluster = np.arange(r_d) % k
    centres_d = rng.random((k, c_d)) * 10
    dim = f32(centres_d[dim_cluster] + 0.01 * rng.standard_normal((r_d, c_d)) + 20)
    fk = np.empty(r_fact, dtype=np.int64)
    for c in range(k):
        rows = np.nonzero(lab == c)[0]
        cand = np.nonzero(dim_cluster == c)[0]
        fk[rows] = cand[np.arange(rows.size) % cand.size]
    c_t = c_fact + c_d
    srcs = [SparseMatrix.from_dense(fact), SparseMatrix.from_dense(dim)]
    maps = [MappingMatrix(SparseMatrix.from_coo(c_t, c_fact, np.arange(c_fact),
                                                np.arange(c_fact), np.ones(c_fact))),
            MappingMatrix(SparseMatrix.from_coo(c_t, c_d, c_fact + np.arange(c_d),
                                                np.arange(c_d), np.ones(c_d)))]
    inds = [IndicatorMatrix(SparseMatrix.identity(r_fact)),
            IndicatorMatrix(SparseMatrix.from_coo(r_fact, r_d, np.arange(r_fact),
                                                  fk, np.ones(r_fact)))]
    return FactorizedTable(srcs, maps, inds, "inner", r_fact, c_t)


def table_arrays(ft):
    """Plain-array form + the reference's own selector derivation."""
    out = {}
    sels = rops._build_selectors(ft)
    for k, (s, sel) in enumerate(zip(ft.sources, sels)):
        out[f"src{k}"] = s.to_dense()
        out[f"ind_sel{k}"] = sel.ind_sel
        out[f"group_indptr{k}"] = sel.group_indptr
        out[f"group_rows{k}"] = sel.group_rows
        out[f"map_sel{k}"] = sel.map_sel
        out[f"map_sel_t{k}"] = sel.map_sel_t
    out["materialized"] = materialize(ft).to_dense()
    return out


def ops_case(ft, seed):
    rng = np.random.default_rng(seed)
    h = TargetHandle.factorized(ft)
    x = f32(rng.random((ft.c_T, 3)))
    w = f32(rng.random((2, ft.r_T)))
    y = f32(rng.random((ft.r_T, 2)))
    out = {"op_x": x, "op_w": w, "op_y": y}
    out["lmm"] = h.lmm(SparseMatrix.from_dense(x)).to_dense()
    out["rmm"] = h.rmm(SparseMatrix.from_dense(w)).to_dense()
    out["tlmm"] = h.transpose_lmm(SparseMatrix.from_dense(y)).to_dense()
    out["row_sum"] = h.row_sum().to_dense()
    out["col_sum"] = h.col_sum().to_dense()
    out["sq_materialized"] = h.elementwise("square").materialize_target().to_dense()
    out["abs_lmm"] = h.elementwise("abs").lmm(SparseMatrix.from_dense(x)).to_dense()
    # the rest of the registered maps (sparse.py:298-307): the mapped join and
    # one product over the mapped table each
    for func, scalar in EW_CASES:
        m = h.elementwise(func, scalar)
        out[f"ew_{func}_materialized"] = m.materialize_target().to_dense()
        out[f"ew_{func}_lmm"] = m.lmm(SparseMatrix.from_dense(x)).to_dense()
    return out


EW_CASES = (("scale", 2.5), ("divide", 3.0), ("expm1", None), ("logistic_centered", None))


def trainer_case(ft, seed, models, iterations, k=3, rank=2):
    rng = np.random.default_rng(seed)
    h = TargetHandle.factorized(ft)
    td = materialize(ft).to_dense()
    gamma = 1.0 / max(np.abs(td).sum(axis=1).max() * np.abs(td).sum(axis=0).max(), 1e-12)
    y_lin = f32(rng.random((ft.r_T, 1)))
    y_log = rng.integers(0, 2, (ft.r_T, 1)).astype(np.float64)
    out = {"y_lin": y_lin, "y_log": y_log, "gamma": np.array(gamma)}
    meta = {}
    for model in models:
        cfg = TrainConfig(iterations=iterations, learning_rate=gamma,
                          k_clusters=k, rank=rank, seed=seed % 1000)
        y = {"linreg": y_lin, "logreg": y_log}.get(model)
        res = train(model, h, cfg, SparseMatrix.from_dense(y) if y is not None else None)
        out[f"{model}_loss"] = np.asarray(res.loss_history)
        for name, val in res.parameters.items():
            out[f"{model}_{name}"] = np.asarray(val)
        meta[model] = {"iterations": iterations, "learning_rate": gamma,
                       "k_clusters": k, "rank": rank, "seed": seed % 1000}
    return out, meta


def save(name, ft, extra, meta):
    arrays = table_arrays(ft)
    arrays.update(extra)
    info = {"name": name, "r_T": ft.r_T, "c_T": ft.c_T, "join_type": ft.join_type,
            "n_sources": ft.n_sources,
            "source_shapes": [list(s.shape) for s in ft.sources]}
    info.update(meta)
    arrays["meta"] = np.array(json.dumps(info))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    print("wrote", name, info["r_T"], "x", info["c_T"], "sources", info["n_sources"])


def main():
    ft = two_source()
    ops = ops_case(ft, 1)
    tr, meta = trainer_case(ft, 3, ("linreg", "logreg", "kmeans", "gnmf"), 6, k=2, rank=2)
    ops.update(tr)
    save("two_source", ft, ops, {"trainers": meta})

    ft = outer()
    save("outer", ft, ops_case(ft, 2), {})

    for join in ("inner", "left", "outer", "union"):
        for n_src in (2, 3):
            for seed in range(2):
                rho = 1.0 if join == "union" else 0.7
                sparsity = 0.75 if join == "union" else 0.5
                try:
                    g, _ = generate(GenSpec(r_t=180, n_sources=n_src, c_min=3, c_max=9,
                                            sparsity=sparsity, rho_c=rho, join_type=join,
                                            seed=100 + 10 * n_src + seed))
                except GenError:
                    continue
                g = round_table(g)
                extra = ops_case(g, 7 + seed)
                models = ("linreg", "logreg", "kmeans") if seed == 0 else ("linreg", "logreg")
                tr, meta = trainer_case(g, 11 + seed, models, 5, k=3)
                extra.update(tr)
                save(f"gen_{join}_{n_src}_{seed}", g, extra, {"trainers": meta})

    ft = star(21, 3000, [(30, 5)], 6)
    extra = ops_case(ft, 4)
    tr, meta = trainer_case(ft, 23, ("linreg", "logreg", "kmeans"), 10, k=4)
    extra.update(tr)
    # GNMF on the same (non-negative) table
    tr2, meta2 = trainer_case(ft, 29, ("gnmf",), 6, rank=3)
    extra.update({k: v for k, v in tr2.items() if k.startswith("gnmf")})
    meta.update(meta2)
    save("star", ft, extra, {"trainers": meta})

    ft = star(31, 2400, [(40, 7), (8, 3)], 5)
    extra = ops_case(ft, 5)
    tr, meta = trainer_case(ft, 37, ("linreg", "logreg", "kmeans", "gnmf"), 6, k=3, rank=2)
    extra.update(tr)
    save("star3", ft, extra, {"trainers": meta})

    ft = clusters()
    tr, meta = trainer_case(ft, 41, ("kmeans",), 8, k=4)
    save("clusters", ft, tr, {"trainers": meta})


if __name__ == "__main__":
    main()
