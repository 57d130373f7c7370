"""Config-scale golden fixtures made by the REAL reference (factorlearn).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_configs.py [c1 c3 c4]

Inputs come from tests/golden/configs.py (deterministic numpy generators the
GPU tests call too); only the reference's outputs are stored:

  cfg_c1.npz  BASELINE configs[0] exactly: 1M x 20 + 10K x 50, factorized
              linear regression, 100 GD iterations at the reference bench's
              safe learning rate (bench.py:112-123) -> w, loss_history, and
              SHA-256 digests of the reference's selectors (ops.py:55-74) and
              of the materialized join (metadata.py:215-225) for bit-exact
              comparison without shipping 1M-row arrays
  cfg_c3.npz  configs[2] shape at 1M rows, K-means k = 16, 10 iterations,
              training seed = first seed whose seed rows hit 16 distinct
              planted clusters -> assignments (uint8), centroids, losses
  cfg_c4.npz  configs[3] shape at 1M rows, GNMF rank 32, 5 iterations ->
              H, losses, W column sums and every 997th row of W
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import configs  # noqa: E402
from factorlearn import ops as rops  # noqa: E402
from factorlearn.bench import _safe_learning_rate  # noqa: E402
from factorlearn.metadata import (FactorizedTable, IndicatorMatrix,  # noqa: E402
                                  MappingMatrix, materialize)
from factorlearn.ops import TargetHandle  # noqa: E402
from factorlearn.sparse import SparseMatrix  # noqa: E402
from factorlearn.trainers import TrainConfig, train  # noqa: E402


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def ref_table(srcs, sels, maps, r_t, c_t):
    S, M, I = [], [], []
    for s, sel, mp in zip(srcs, sels, maps):
        S.append(SparseMatrix.from_dense(s))
        c_k = s.shape[1]
        M.append(MappingMatrix(SparseMatrix.from_coo(c_t, c_k, np.asarray(mp), np.arange(c_k),
                                                     np.ones(c_k))))
        sel = np.asarray(sel)
        ok = sel >= 0
        I.append(IndicatorMatrix(SparseMatrix.from_coo(r_t, s.shape[0], np.nonzero(ok)[0],
                                                       sel[ok], np.ones(int(ok.sum())))))
    return FactorizedTable(S, M, I, "inner", r_t, c_t)


def save(name, arrays, meta):
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    print("wrote", name, meta, flush=True)


def make_c1():
    srcs, sels, maps, r_t, c_t, y = configs.c1_arrays()
    ft = ref_table(srcs, sels, maps, r_t, c_t)
    t0 = time.perf_counter()
    target = materialize(ft)
    gamma = _safe_learning_rate(target)
    sel = rops._build_selectors(ft)
    dense_digest = digest(target.to_dense())
    del target
    h = TargetHandle.factorized(ft)
    res = train("linreg", h, TrainConfig(iterations=100, learning_rate=gamma),
                SparseMatrix.from_dense(y.reshape(-1, 1)))
    meta = {"iterations": 100, "learning_rate": gamma,
            "reference_seconds": time.perf_counter() - t0,
            "reference_wall_time": res.wall_time,
            "join_sha256": dense_digest,
            "selectors_sha256": [digest(s.ind_sel, s.group_indptr, s.group_rows, s.map_sel,
                                        s.map_sel_t) for s in sel]}
    save("cfg_c1", {"w": res.parameters["w"].ravel(),
                    "loss": np.asarray(res.loss_history)}, meta)


def make_c3():
    srcs, sels, maps, r_t, c_t, lab = configs.c3_arrays()
    seed = configs.c3_seed(lab=lab)
    ft = ref_table(srcs, sels, maps, r_t, c_t)
    t0 = time.perf_counter()
    h = TargetHandle.factorized(ft)
    res = train("kmeans", h, TrainConfig(iterations=10, k_clusters=16, seed=seed))
    a = np.asarray(res.parameters["assignments"])
    meta = {"iterations": 10, "k_clusters": 16, "seed": seed,
            "reference_seconds": time.perf_counter() - t0,
            "reference_wall_time": res.wall_time}
    save("cfg_c3", {"assignments": a.astype(np.uint8), "centroids": res.parameters["centroids"],
                    "loss": np.asarray(res.loss_history)}, meta)


def make_c4():
    srcs, sels, maps, r_t, c_t = configs.c4_arrays()
    ft = ref_table(srcs, sels, maps, r_t, c_t)
    t0 = time.perf_counter()
    h = TargetHandle.factorized(ft)
    res = train("gnmf", h, TrainConfig(iterations=5, rank=32, seed=4))
    w = res.parameters["w"]
    meta = {"iterations": 5, "rank": 32, "seed": 4,
            "reference_seconds": time.perf_counter() - t0,
            "reference_wall_time": res.wall_time}
    save("cfg_c4", {"h": res.parameters["h"], "loss": np.asarray(res.loss_history),
                    "w_colsum": w.sum(axis=0), "w_rows": w[::997]}, meta)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c3", "c4"]
    for n in which:
        {"c1": make_c1, "c3": make_c3, "c4": make_c4}[n]()
