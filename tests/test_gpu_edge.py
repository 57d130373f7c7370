"""GPU parity on edge-shaped tables: a single target row, row counts that are
not multiples of the 256-row tile or the 32/64-row warp units, a dimension
no fact row matches (left join), a one-row dimension (fanout = r_T), and an
injective "dimension" larger than the fact table (it joins the stream block
through the inverted indicator).  Join bit-exact; operators, GLM weights /
losses, K-means and GNMF results against the oracle (1e-4 relative, K-means
assignments identical)."""

import numpy as np
import pytest

import oracle
from oracle import reference_trainers as rt

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def fl():
    import paper_2502_01985_b200 as fl
    return fl


def _table(seed, r_fact, c_fact, dims):
    """dims: list of (r_d, c_d, fk_kind) with fk_kind in
    'random' | 'none' (all -1) | 'one' (r_d = 1) | 'inject' (injective)."""
    rng = np.random.default_rng(seed)
    srcs = [rng.random((r_fact, c_fact)).astype(np.float32)]
    sels = [None]
    for r_d, c_d, kind in dims:
        srcs.append(rng.random((r_d, c_d)).astype(np.float32))
        if kind == "random":
            fk = rng.integers(0, r_d, r_fact)
        elif kind == "none":
            fk = np.full(r_fact, -1)
        elif kind == "one":
            fk = np.zeros(r_fact, dtype=np.int64)
        else:   # injective into a larger source
            fk = rng.permutation(r_d)[:r_fact]
        sels.append(fk.astype(np.int32))
    maps, off = [], 0
    for s in srcs:
        maps.append(np.arange(s.shape[1], dtype=np.int32) + off)
        off += s.shape[1]
    return srcs, sels, maps, r_fact, off


def _oracle(srcs, sels, maps, r, c):
    ind = [np.arange(r) if s is None else np.asarray(s, dtype=np.int64) for s in sels]
    return oracle.OracleTable([s.astype(np.float64) for s in srcs], ind,
                              [m.astype(np.int64) for m in maps], r, c)


def _rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-12))


CASES = {
    "single_row": (1, 3, [(1, 2, "one")]),
    "ragged_257_unmatched_dim": (257, 5, [(3, 5, "none"), (11, 2, "random")]),
    "one_row_dim": (1000, 4, [(1, 6, "one")]),
    "injective_dim": (777, 6, [(5000, 3, "inject"), (40, 5, "random")]),
    "ragged_4097": (4097, 20, [(97, 13, "random")]),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_edge_tables_operators(fl, name):
    r, c_f, dims = CASES[name]
    srcs, sels, maps, r_t, c_t = _table(11, r, c_f, dims)
    tab = _oracle(srcs, sels, maps, r_t, c_t)
    h = fl.TargetHandle.from_arrays(srcs, sels, maps, r_t, c_t)
    assert np.array_equal(h.materialize_dense().astype(np.float64), oracle.materialize(tab))
    rng = np.random.default_rng(3)
    x = rng.random((c_t, 2)).astype(np.float32)
    assert _rel(h.lmm(x), oracle.lmm(tab, x)) < 1e-5
    y = rng.random((r_t, 3)).astype(np.float32)
    assert _rel(h.transpose_lmm(y), oracle.transpose_lmm(tab, y)) < 1e-5


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("model", ["linreg", "logreg"])
def test_edge_tables_glm(fl, name, model):
    r, c_f, dims = CASES[name]
    srcs, sels, maps, r_t, c_t = _table(12, r, c_f, dims)
    tab = _oracle(srcs, sels, maps, r_t, c_t)
    h = fl.TargetHandle.from_arrays(srcs, sels, maps, r_t, c_t)
    rng = np.random.default_rng(4)
    y = (rng.integers(0, 2, r_t) if model == "logreg" else rng.random(r_t)).astype(np.float64)
    lr = rt.safe_learning_rate(tab)
    ref = rt.train(model, tab, iterations=6, learning_rate=lr, y=y)
    res = fl.train(model, h, fl.TrainConfig(iterations=6, learning_rate=lr), y.reshape(-1, 1))
    assert _rel(res.loss_history, ref["loss_history"]) < TOL
    assert _rel(res.parameters["w"], ref["parameters"]["w"]) < TOL


@pytest.mark.parametrize("name", ["ragged_257_unmatched_dim", "one_row_dim", "injective_dim",
                                  "ragged_4097"])
def test_edge_tables_kmeans(fl, name):
    r, c_f, dims = CASES[name]
    srcs, sels, maps, r_t, c_t = _table(13, r, c_f, dims)
    tab = _oracle(srcs, sels, maps, r_t, c_t)
    h = fl.TargetHandle.from_arrays(srcs, sels, maps, r_t, c_t)
    k = 3
    ref = rt.kmeans(tab, 4, k, 5)
    res = fl.train("kmeans", h, fl.TrainConfig(iterations=4, k_clusters=k, seed=5))
    assert np.array_equal(res.parameters["assignments"], ref["parameters"]["assignments"])
    assert _rel(res.loss_history, ref["loss_history"]) < TOL


@pytest.mark.parametrize("name", ["ragged_257_unmatched_dim", "one_row_dim", "injective_dim",
                                  "ragged_4097"])
def test_edge_tables_gnmf(fl, name):
    r, c_f, dims = CASES[name]
    srcs, sels, maps, r_t, c_t = _table(14, r, c_f, dims)
    tab = _oracle(srcs, sels, maps, r_t, c_t)
    h = fl.TargetHandle.from_arrays(srcs, sels, maps, r_t, c_t)
    ref = rt.gaussian_nmf(tab, 4, 3, 2)
    res = fl.train("gnmf", h, fl.TrainConfig(iterations=4, rank=3, seed=2))
    assert _rel(res.loss_history, ref["loss_history"]) < TOL
    assert _rel(res.parameters["h"], ref["parameters"]["h"]) < TOL
    assert _rel(res.parameters["w"], ref["parameters"]["w"]) < TOL
