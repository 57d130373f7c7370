"""GPU parity of the tcgen05 fact passes with MN-major row-contraction
operands (csrc/kmeans_t5.cuh): the K-means screen Z = F C_F^T and the sums
[F_hi | F_lo]^T one-hot as tcgen05 MMAs from shared memory into TMEM, the
one-hot / F operand tiles read MN-major in the 128B / 32-byte-atom swizzle.
Same bar as the other fused passes: assignments identical, losses and
centroids within 1e-4 relative; bit-identical run to run."""

import numpy as np
import pytest

import oracle
from oracle import reference_trainers as rt
from conftest import golden_names, load_golden
from test_gpu_generic import planted_seeded
from test_gpu_trainers import _cfg, max_rel

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def fl():
    import paper_2502_01985_b200 as fl
    return fl


@pytest.fixture
def t5(monkeypatch):
    monkeypatch.setenv("FL_KM_T5", "1")


def _km_cases():
    return [n for n in golden_names() if "kmeans" in load_golden(n).meta.get("trainers", {})]


@pytest.mark.parametrize("name", _km_cases())
def test_kmeans_t5_matches_reference(fl, t5, name):
    g = load_golden(name)
    m = g.meta["trainers"]["kmeans"]
    res = fl.train("kmeans", fl.TargetHandle.factorized(g.ft), _cfg(fl, m))
    assert np.array_equal(res.parameters["assignments"], g["kmeans_assignments"])
    assert max_rel(res.loss_history, g["kmeans_loss"]) < TOL
    assert max_rel(res.parameters["centroids"], g["kmeans_centroids"]) < TOL


@pytest.mark.parametrize("k,dims,c_fact,rows", [(16, [(3000, 30), (200, 5)], 20, 60_000),
                                                (4, [(500, 9)], 12, 40_001),
                                                (24, [(4000, 7)], 5, 30_000),
                                                (32, [(600, 60)], 28, 50_000),
                                                (9, [], 20, 20_000),
                                                (16, [(60 + 7 * i, 3) for i in range(4)], 8, 25_000)])
def test_kmeans_t5_planted_vs_oracle(fl, t5, k, dims, c_fact, rows):
    from paper_2502_01985_b200.trainers import KMeansSession, kmeans_init
    ft = planted_seeded(21, rows, dims, c_fact, k, 3)
    h = fl.TargetHandle.factorized(ft)
    s = KMeansSession(h, k, kmeans_init(h, k, 3))
    assert s.path == "tcgen05_mn"
    s.close()
    tab = oracle.OracleTable.from_ft(ft)
    want = rt.kmeans(tab, 6, k, 3)
    res = fl.train("kmeans", h, fl.TrainConfig(iterations=6, k_clusters=k, seed=3))
    assert np.array_equal(res.parameters["assignments"], want["parameters"]["assignments"])
    assert max_rel(res.loss_history, want["loss_history"]) < TOL
    assert max_rel(res.parameters["centroids"], want["parameters"]["centroids"]) < TOL


@pytest.mark.parametrize("k,noise", [(16, 0.35), (8, 1.0)])
def test_kmeans_t5_overlapping_clusters_certified(fl, t5, k, noise):
    """Overlapping clusters: the screen's near-ties go through the exact
    certification; one iteration from identical seeds."""
    from test_gpu_trainers import planted_star
    ft = planted_star(5, 40_000, [(2000, 24), (300, 6)], 20, k, noise=noise)
    tab = oracle.OracleTable.from_ft(ft)
    want = rt.kmeans(tab, 1, k, 7)
    res = fl.train("kmeans", fl.TargetHandle.factorized(ft),
                   fl.TrainConfig(iterations=1, k_clusters=k, seed=7))
    diff = np.count_nonzero(res.parameters["assignments"] != want["parameters"]["assignments"])
    assert diff <= 2
    assert max_rel(res.loss_history, want["loss_history"]) < TOL


def test_kmeans_t5_deterministic_and_matches_mma_pass(fl, monkeypatch):
    ft = planted_seeded(31, 70_000, [(2000, 24), (100, 4)], 20, 16, 5)
    h = fl.TargetHandle.factorized(ft)
    cfg = fl.TrainConfig(iterations=5, k_clusters=16, seed=5)
    monkeypatch.setenv("FL_KM_T5", "1")
    a = fl.train("kmeans", h, cfg)
    b = fl.train("kmeans", h, cfg)
    assert np.array_equal(a.parameters["centroids"], b.parameters["centroids"])
    assert a.loss_history == b.loss_history
    monkeypatch.setenv("FL_KM_T5", "0")
    c = fl.train("kmeans", h, cfg)
    assert np.array_equal(a.parameters["assignments"], c.parameters["assignments"])
    assert max_rel(a.parameters["centroids"], c.parameters["centroids"]) < 1e-6
    assert max_rel(a.loss_history, c.loss_history) < 1e-6


# ---------------------------------------------------------------------------
# GNMF (csrc/gnmf_t5.cuh)
# ---------------------------------------------------------------------------
@pytest.fixture
def g5(monkeypatch):
    monkeypatch.setenv("FL_GN_T5", "1")


def _gn_cases():
    return [n for n in golden_names() if "gnmf" in load_golden(n).meta.get("trainers", {})]


@pytest.mark.parametrize("name", _gn_cases())
def test_gnmf_t5_matches_reference(fl, g5, name):
    g = load_golden(name)
    m = g.meta["trainers"]["gnmf"]
    res = fl.train("gnmf", fl.TargetHandle.factorized(g.ft), _cfg(fl, m))
    assert max_rel(res.loss_history, g["gnmf_loss"]) < TOL
    assert max_rel(res.parameters["h"], g["gnmf_h"]) < TOL
    assert max_rel(res.parameters["w"], g["gnmf_w"]) < TOL


@pytest.mark.parametrize("rank,dims,c_fact,rows", [(32, [(2000, 50)], 20, 40_000),
                                                   (20, [(700, 9)], 28, 30_001),
                                                   (25, [], 28, 20_000),
                                                   (17, [(5000, 20)], 3, 25_000)])
def test_gnmf_t5_vs_oracle(fl, g5, rank, dims, c_fact, rows):
    from conftest import star_table
    from paper_2502_01985_b200.trainers import GnmfSession
    ft = star_table(37, rows, dims, c_fact)
    h = fl.TargetHandle.factorized(ft)
    s = GnmfSession(h, rank, np.ones((ft.r_T, rank)), np.ones((rank, ft.c_T)), 1.0)
    assert s.path == "tcgen05_mn"
    s.close()
    tab = oracle.OracleTable.from_ft(ft)
    want = rt.gaussian_nmf(tab, 5, rank, 9)
    res = fl.train("gnmf", h, fl.TrainConfig(iterations=5, rank=rank, seed=9))
    assert max_rel(res.loss_history, want["loss_history"]) < TOL
    assert max_rel(res.parameters["h"], want["parameters"]["h"]) < TOL
    assert max_rel(res.parameters["w"], want["parameters"]["w"]) < TOL


def test_gnmf_t5_deterministic_and_matches_mma_pass(fl, monkeypatch):
    from conftest import star_table
    ft = star_table(39, 60_000, [(800, 30)], 20)
    h = fl.TargetHandle.factorized(ft)
    cfg = fl.TrainConfig(iterations=6, rank=32, seed=2)
    monkeypatch.setenv("FL_GN_T5", "1")
    a = fl.train("gnmf", h, cfg)
    b = fl.train("gnmf", h, cfg)
    assert np.array_equal(a.parameters["w"], b.parameters["w"])
    assert a.loss_history == b.loss_history
    monkeypatch.setenv("FL_GN_T5", "0")
    c = fl.train("gnmf", h, cfg)
    assert max_rel(a.parameters["w"], c.parameters["w"]) < 1e-5
    assert max_rel(a.loss_history, c.loss_history) < 1e-6
