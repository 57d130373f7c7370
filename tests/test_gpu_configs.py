"""Parity at the BASELINE.json config shapes (GPU vs the REAL reference).

Inputs are regenerated from seeds by tests/golden/configs.py; the expected
outputs were produced by running the unmodified reference on exactly those
inputs (tests/golden/make_golden_configs.py -> cfg_*.npz).

  C1 (configs[0], full size: 1M x 20 + 10K x 50, linreg, 100 iterations):
     selectors and join bit-exact (SHA-256 of the reference's arrays), w and
     every loss within 1e-4 relative
  C3 shape at 1M rows (K-means k = 16, planted clusters, 10 iterations):
     assignments identical, centroids / losses within 1e-4
  C4 shape at 1M rows (GNMF rank 32, 5 iterations): H, losses, W column
     sums and sampled W rows within 1e-4
  plus: a one-row dimension under 10M fact rows (fanout 1e7) against the
  oracle, and GNMF run-to-run bit identity.
"""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN_DIR

sys.path.insert(0, GOLDEN_DIR)
import configs  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = 1e-4


def max_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def digest(*arrays) -> str:
    """Same digest as make_golden_configs.digest (dtype, shape, bytes)."""
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def golden(name):
    raw = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    g = {k: raw[k] for k in raw.files}
    g["meta"] = json.loads(str(g["meta"]))
    return g


def product_table(fl, srcs, sels, maps, r_t, c_t):
    from paper_2502_01985_b200.metadata import fk_indicator
    from paper_2502_01985_b200.sparse import SparseMatrix
    S, M, I = [], [], []
    for s, sel, mp in zip(srcs, sels, maps):
        c_k = s.shape[1]
        S.append(fl.SparseMatrix.from_dense(s))
        M.append(fl.MappingMatrix(SparseMatrix.from_coo(c_t, c_k, np.asarray(mp), np.arange(c_k),
                                                        np.ones(c_k))))
        I.append(fk_indicator(r_t, s.shape[0], np.asarray(sel)))
    return fl.FactorizedTable(S, M, I, "inner", r_t, c_t)


@pytest.fixture(scope="module")
def fl():
    import paper_2502_01985_b200 as fl
    return fl


def test_c1_full_config_matches_reference(fl):
    g = golden("cfg_c1")
    m = g["meta"]
    srcs, sels, maps, r_t, c_t, y = configs.c1_arrays()
    ft = product_table(fl, srcs, sels, maps, r_t, c_t)
    h = fl.TargetHandle.factorized(ft)
    # selectors: the device-derived arrays hash to the reference's
    for k, s in enumerate(h.selectors):
        got = digest(*(np.asarray(a, dtype=np.int64) for a in
                       (s.ind_sel, s.group_indptr, s.group_rows, s.map_sel, s.map_sel_t)))
        assert got == m["selectors_sha256"][k], f"selectors of source {k}"
    # the join, bit-exact (fp32 copies widened to the reference's float64)
    assert digest(h.materialize_dense().astype(np.float64)) == m["join_sha256"]
    res = fl.train("linreg", h, fl.TrainConfig(iterations=m["iterations"],
                                               learning_rate=m["learning_rate"]),
                   y.reshape(-1, 1))
    assert len(res.loss_history) == 100
    assert max_rel(res.loss_history, g["loss"]) < TOL
    assert max_rel(res.parameters["w"].ravel(), g["w"]) < TOL


def test_c3_shape_kmeans_matches_reference(fl):
    g = golden("cfg_c3")
    m = g["meta"]
    srcs, sels, maps, r_t, c_t, _ = configs.c3_arrays()
    h = fl.TargetHandle.from_arrays(srcs, sels, maps, r_t, c_t)
    res = fl.train("kmeans", h, fl.TrainConfig(iterations=m["iterations"],
                                               k_clusters=m["k_clusters"], seed=m["seed"]))
    a = res.parameters["assignments"]
    assert a.dtype == np.int64
    assert np.array_equal(a, g["assignments"].astype(np.int64))
    assert max_rel(res.parameters["centroids"], g["centroids"]) < TOL
    assert max_rel(res.loss_history, g["loss"]) < TOL


def test_c4_shape_gnmf_matches_reference(fl):
    g = golden("cfg_c4")
    m = g["meta"]
    srcs, sels, maps, r_t, c_t = configs.c4_arrays()
    h = fl.TargetHandle.from_arrays(srcs, sels, maps, r_t, c_t)
    res = fl.train("gnmf", h, fl.TrainConfig(iterations=m["iterations"], rank=m["rank"],
                                             seed=m["seed"]))
    w = res.parameters["w"]
    assert max_rel(res.loss_history, g["loss"]) < TOL
    assert max_rel(res.parameters["h"], g["h"]) < TOL
    assert max_rel(w.sum(axis=0), g["w_colsum"]) < TOL
    assert max_rel(w[::997], g["w_rows"]) < TOL


def test_gnmf_run_to_run_bit_identical(fl):
    """Z_d = I_d^T W and every other reduction are fixed-order: two fits on
    the same inputs give identical bits (W, H, losses)."""
    srcs, sels, maps, r_t, c_t = configs.c4_arrays(rows=400_000)
    h = fl.TargetHandle.from_arrays(srcs, sels, maps, r_t, c_t)
    cfg = fl.TrainConfig(iterations=4, rank=32, seed=9)
    a = fl.train("gnmf", h, cfg)
    b = fl.train("gnmf", h, cfg)
    assert np.array_equal(a.parameters["w"], b.parameters["w"])
    assert np.array_equal(a.parameters["h"], b.parameters["h"])
    assert a.loss_history == b.loss_history


@pytest.mark.parametrize("model", ["linreg", "logreg"])
def test_fanout_1e7_one_row_dimension(fl, model):
    """A one-row dimension under 10M fact rows: one I_d^T segment spans the
    whole pass (every warp's carry), compared with the oracle."""
    import oracle
    from oracle import reference_trainers as rt
    srcs, sels, maps, r_t, c_t, y = configs.fanout_arrays()
    if model == "logreg":
        y = (y > 0.5).astype(np.float64)
    h = fl.TargetHandle.from_arrays(srcs, sels, maps, r_t, c_t)
    tab = oracle.OracleTable(srcs, [np.asarray(s) for s in sels],
                             [np.asarray(mp, dtype=np.int64) for mp in maps], r_t, c_t)
    lr = rt.safe_learning_rate(tab)
    want = rt.train(model, tab, iterations=4, learning_rate=lr, y=y)
    res = fl.train(model, h, fl.TrainConfig(iterations=4, learning_rate=lr), y.reshape(-1, 1))
    assert max_rel(res.loss_history, want["loss_history"]) < TOL
    assert max_rel(res.parameters["w"], want["parameters"]["w"]) < TOL
    # the dimension's gradient is the full-column sum: check it on its own
    wd, wd_ref = res.parameters["w"].ravel()[8:], want["parameters"]["w"].ravel()[8:]
    assert max_rel(wd, wd_ref) < TOL
