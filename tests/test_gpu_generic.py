"""GPU parity of the width-general paths (csrc/generic.cu, ops.cu do_lmm_many):
K-means past k = 32 / 124 streamed columns / 8 gathered sources, GNMF past
rank 32 / 60 streamed columns, and the GLMs and operators over more than 8
gathered sources -- every shape the reference trains (trainers.py:198-307),
against the reference goldens and the CPU oracle.  Tolerance as elsewhere:
1e-4 relative; K-means assignments identical on well-separated data."""

import numpy as np
import pytest

import oracle
from oracle import reference_trainers as rt
from conftest import golden_names, load_golden, star_table
from test_gpu_trainers import _cfg, max_rel, planted_star

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def fl():
    import paper_2502_01985_b200 as fl
    return fl


def _cases(model):
    out = []
    for name in golden_names():
        g = load_golden(name)
        if model in g.meta.get("trainers", {}):
            out.append(name)
    return out


def planted_seeded(seed, r_fact, dims, c_fact, k, train_seed, noise=0.01):
    """planted_star with the reference's K-means seed rows (trainers.py:209-
    210: sorted rng.choice of k target rows) placed one per planted cluster,
    so Lloyd converges to the planted clusters and every row's nearest and
    second-nearest centroids are far apart (assignments are then identical
    for any correct implementation, fp32 or fp64)."""
    from paper_2502_01985_b200.metadata import FactorizedTable, block_mapping, fk_indicator
    from paper_2502_01985_b200.sparse import SparseMatrix
    rng = np.random.default_rng(seed)
    lab = rng.integers(0, k, r_fact)
    pick = np.sort(np.random.default_rng(train_seed).choice(r_fact, size=k, replace=False))
    lab[pick] = np.arange(k)
    c_t = c_fact + sum(c for _, c in dims)
    cen = rng.random((k, c_fact))
    fact = (cen[lab] + noise * rng.standard_normal((r_fact, c_fact))).astype(np.float32)
    srcs = [SparseMatrix.from_dense(fact.astype(np.float64))]
    maps = [block_mapping(c_t, c_fact, 0)]
    inds = [fk_indicator(r_fact, r_fact, np.arange(r_fact))]
    off = c_fact
    for r_d, c_d in dims:
        dlab = np.arange(r_d) % k
        dim = (rng.random((k, c_d))[dlab] + noise * rng.standard_normal((r_d, c_d))).astype(np.float32)
        fk = np.empty(r_fact, dtype=np.int64)
        for j in range(k):
            rows = np.nonzero(dlab == j)[0]
            mine = np.nonzero(lab == j)[0]
            fk[mine] = rows[rng.integers(0, rows.size, mine.size)]
        srcs.append(SparseMatrix.from_dense(dim.astype(np.float64)))
        maps.append(block_mapping(c_t, c_d, off))
        inds.append(fk_indicator(r_fact, r_d, fk))
        off += c_d
    return FactorizedTable(srcs, maps, inds, "inner", r_fact, c_t)


def _km_path(fl, ft, k):
    from paper_2502_01985_b200.trainers import KMeansSession, kmeans_init
    h = fl.TargetHandle.factorized(ft)
    s = KMeansSession(h, k, kmeans_init(h, k, 0))
    try:
        return s.path
    finally:
        s.close()


def _gn_path(fl, ft, rank):
    from paper_2502_01985_b200.trainers import GnmfSession
    h = fl.TargetHandle.factorized(ft)
    r_t, c_t = h.shape
    s = GnmfSession(h, rank, np.ones((r_t, rank)), np.ones((rank, c_t)), 1.0)
    try:
        return s.path
    finally:
        s.close()


# ---------------------------------------------------------------------------
# K-means
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", _cases("kmeans"))
def test_kmeans_generic_forced_matches_reference(fl, name, monkeypatch):
    monkeypatch.setenv("FL_KM_GENERIC", "1")
    g = load_golden(name)
    m = g.meta["trainers"]["kmeans"]
    res = fl.train("kmeans", fl.TargetHandle.factorized(g.ft), _cfg(fl, m))
    assert len(res.loss_history) == m["iterations"]
    assert np.array_equal(res.parameters["assignments"], g["kmeans_assignments"])
    assert max_rel(res.loss_history, g["kmeans_loss"]) < TOL
    assert max_rel(res.parameters["centroids"], g["kmeans_centroids"]) < TOL


@pytest.mark.parametrize("k,dims,c_fact", [
    (40, [(3000, 30), (200, 5)], 20),           # k > 32
    (12, [(400, 9)], 150),                      # 150 streamed columns (> 124)
    (6, [(60 + 7 * i, 3 + i % 4) for i in range(10)], 8),   # 10 gathered sources (> 8)
    (48, [(500, 300)], 12),                     # k > 32 and a 300-column dimension
])
def test_kmeans_width_general_vs_oracle(fl, k, dims, c_fact):
    ft = planted_seeded(23, 30_000, dims, c_fact, k, 4)
    assert _km_path(fl, ft, k) == "generic"
    tab = oracle.OracleTable.from_ft(ft)
    want = rt.kmeans(tab, 5, k, 4)
    res = fl.train("kmeans", fl.TargetHandle.factorized(ft),
                   fl.TrainConfig(iterations=5, k_clusters=k, seed=4))
    assert np.array_equal(res.parameters["assignments"], want["parameters"]["assignments"])
    assert max_rel(res.loss_history, want["loss_history"]) < TOL
    assert max_rel(res.parameters["centroids"], want["parameters"]["centroids"]) < TOL


def test_kmeans_generic_deterministic(fl):
    ft = planted_seeded(29, 20_000, [(700, 13)], 10, 36, 2)
    h = fl.TargetHandle.factorized(ft)
    cfg = fl.TrainConfig(iterations=4, k_clusters=36, seed=2)
    a = fl.train("kmeans", h, cfg)
    b = fl.train("kmeans", h, cfg)
    assert np.array_equal(a.parameters["centroids"], b.parameters["centroids"])
    assert a.loss_history == b.loss_history


# ---------------------------------------------------------------------------
# Gaussian NMF
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", _cases("gnmf"))
def test_gnmf_generic_forced_matches_reference(fl, name, monkeypatch):
    monkeypatch.setenv("FL_GN_GENERIC", "1")
    g = load_golden(name)
    m = g.meta["trainers"]["gnmf"]
    res = fl.train("gnmf", fl.TargetHandle.factorized(g.ft), _cfg(fl, m))
    assert len(res.loss_history) == m["iterations"]
    assert max_rel(res.loss_history, g["gnmf_loss"]) < TOL
    assert max_rel(res.parameters["h"], g["gnmf_h"]) < TOL
    assert max_rel(res.parameters["w"], g["gnmf_w"]) < TOL


@pytest.mark.parametrize("rank,dims,c_fact", [
    (48, [(2000, 50)], 20),                     # rank > 32
    (10, [(300, 7)], 150),                      # 150 streamed columns (> 60)
    (6, [(50 + 9 * i, 2 + i % 3) for i in range(10)], 6),   # 10 gathered sources
])
def test_gnmf_width_general_vs_oracle(fl, rank, dims, c_fact):
    ft = star_table(41, 20_000, dims, c_fact)
    assert _gn_path(fl, ft, rank) == "generic"
    tab = oracle.OracleTable.from_ft(ft)
    want = rt.gaussian_nmf(tab, 5, rank, 6)
    res = fl.train("gnmf", fl.TargetHandle.factorized(ft),
                   fl.TrainConfig(iterations=5, rank=rank, seed=6))
    assert max_rel(res.loss_history, want["loss_history"]) < TOL
    assert max_rel(res.parameters["h"], want["parameters"]["h"]) < TOL
    assert max_rel(res.parameters["w"], want["parameters"]["w"]) < TOL


def test_gnmf_generic_materialized_wide(fl):
    """The C4-style materialized baseline: a 70-column dense T (pitch 76 >
    60) trains through the width-general session and agrees with the
    factorized fit."""
    ft = star_table(43, 15_000, [(300, 50)], 20)
    tab = oracle.OracleTable.from_ft(ft)
    dense = oracle.materialize(tab)
    mh = fl.TargetHandle.materialized(fl.SparseMatrix.from_dense(dense))
    want = rt.gaussian_nmf(tab, 4, 32, 3)
    res = fl.train("gnmf", mh, fl.TrainConfig(iterations=4, rank=32, seed=3))
    assert max_rel(res.loss_history, want["loss_history"]) < TOL
    assert max_rel(res.parameters["w"], want["parameters"]["w"]) < TOL


def test_gnmf_generic_deterministic_and_monotone(fl, monkeypatch):
    monkeypatch.setenv("FL_GN_GENERIC", "1")
    ft = star_table(47, 12_000, [(400, 9)], 10)
    h = fl.TargetHandle.factorized(ft)
    cfg = fl.TrainConfig(iterations=8, rank=6, seed=1)
    a = fl.train("gnmf", h, cfg)
    b = fl.train("gnmf", h, cfg)
    assert np.array_equal(a.parameters["w"], b.parameters["w"])
    assert a.loss_history == b.loss_history
    lh = np.asarray(a.loss_history)
    assert np.all(np.diff(lh) <= 1e-6 * np.abs(lh[:-1]))


# ---------------------------------------------------------------------------
# GLMs and operators over more than 8 gathered sources
# ---------------------------------------------------------------------------
MANY = [(40 + 11 * i, 2 + i % 5) for i in range(11)]


@pytest.mark.parametrize("model", ["linreg", "logreg"])
def test_glm_many_sources_vs_oracle(fl, model):
    ft = star_table(53, 25_000, MANY, 9)
    tab = oracle.OracleTable.from_ft(ft)
    rng = np.random.default_rng(2)
    y = (rng.random(ft.r_T) if model == "linreg" else rng.integers(0, 2, ft.r_T)).astype(np.float64)
    lr = rt.safe_learning_rate(tab)
    want = rt.train(model, tab, iterations=6, learning_rate=lr, y=y)
    res = fl.train(model, fl.TargetHandle.factorized(ft),
                   fl.TrainConfig(iterations=6, learning_rate=lr), y.reshape(-1, 1))
    assert max_rel(res.loss_history, want["loss_history"]) < TOL
    assert max_rel(res.parameters["w"], want["parameters"]["w"]) < TOL


def test_operators_many_sources_vs_oracle(fl):
    ft = star_table(59, 18_000, MANY, 7)
    tab = oracle.OracleTable.from_ft(ft)
    h = fl.TargetHandle.factorized(ft)
    rng = np.random.default_rng(5)
    c_t = ft.c_T
    x = rng.random((c_t, 3)).astype(np.float32)
    want = oracle.lmm(tab, x)
    got = h.lmm(x)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-5
    y = rng.random((ft.r_T, 2)).astype(np.float32)
    want_t = oracle.transpose_lmm(tab, y)
    got_t = h.transpose_lmm(y)
    assert np.linalg.norm(got_t - want_t) / np.linalg.norm(want_t) < 1e-5
    assert np.array_equal(h.materialize_dense().astype(np.float64), oracle.materialize(tab))
