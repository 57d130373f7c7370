"""GPU parity of the fused trainers vs the reference's golden runs and the
CPU oracle.  Tolerance (north star): 1e-4 relative on weights, losses and
centroids; K-means assignments identical on well-separated data."""

import numpy as np
import pytest

import oracle
from oracle import reference_trainers as rt
from conftest import golden_names, load_golden, star_table

pytestmark = pytest.mark.gpu

TOL = 1e-4


def max_rel(a, b, floor=1e-12):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(np.max(np.abs(b)), floor)
    return float(np.max(np.abs(a - b)) / scale)


@pytest.fixture(scope="module")
def fl():
    import paper_2502_01985_b200 as fl
    return fl


def _cases(models):
    out = []
    for name in golden_names():
        g = load_golden(name)
        for m in g.meta.get("trainers", {}):
            if m in models:
                out.append((name, m))
    return out


@pytest.mark.parametrize("name,model", _cases(("linreg", "logreg")))
def test_glm_matches_reference(fl, name, model):
    g = load_golden(name)
    m = g.meta["trainers"][model]
    h = fl.TargetHandle.factorized(g.ft)
    y = g["y_lin"] if model == "linreg" else g["y_log"]
    cfg = fl.TrainConfig(iterations=m["iterations"], learning_rate=m["learning_rate"],
                         k_clusters=m["k_clusters"], rank=m["rank"], seed=m["seed"])
    res = fl.train(model, h, cfg, fl.SparseMatrix.from_dense(y))
    assert len(res.loss_history) == m["iterations"]
    assert max_rel(res.loss_history, g[f"{model}_loss"]) < TOL
    assert max_rel(res.parameters["w"], g[f"{model}_w"]) < TOL


@pytest.mark.parametrize("model", ["linreg", "logreg"])
@pytest.mark.parametrize("dims", [[(2000, 17)], [(900, 11), (40, 3)], [(30000, 6)]])
def test_glm_random_star_vs_oracle(fl, model, dims):
    ft = star_table(11, 120_000, dims, 20)
    tab = oracle.OracleTable.from_ft(ft)
    rng = np.random.default_rng(3)
    if model == "linreg":
        y = rng.random(ft.r_T).astype(np.float32).astype(np.float64)
    else:
        y = rng.integers(0, 2, ft.r_T).astype(np.float64)
    lr = rt.safe_learning_rate(tab)
    want = rt.train(model, tab, iterations=8, learning_rate=lr, y=y)
    h = fl.TargetHandle.factorized(ft)
    res = fl.train(model, h, fl.TrainConfig(iterations=8, learning_rate=lr), y.reshape(-1, 1))
    assert max_rel(res.loss_history, want["loss_history"]) < TOL
    assert max_rel(res.parameters["w"], want["parameters"]["w"]) < TOL


@pytest.mark.parametrize("name,model", _cases(("linreg", "logreg")))
def test_glm_csr_pass_matches_reference(fl, name, model, monkeypatch):
    """The sparse fact pass (CSR copy of the stream block, FL_GLM_SPARSE=1
    forces it) against the reference goldens."""
    monkeypatch.setenv("FL_GLM_SPARSE", "1")
    g = load_golden(name)
    m = g.meta["trainers"][model]
    h = fl.TargetHandle.factorized(g.ft)
    y = g["y_lin"] if model == "linreg" else g["y_log"]
    cfg = fl.TrainConfig(iterations=m["iterations"], learning_rate=m["learning_rate"],
                         k_clusters=m["k_clusters"], rank=m["rank"], seed=m["seed"])
    res = fl.train(model, h, cfg, fl.SparseMatrix.from_dense(y))
    assert max_rel(res.loss_history, g[f"{model}_loss"]) < TOL
    assert max_rel(res.parameters["w"], g[f"{model}_w"]) < TOL


def sparse_star(seed, r_fact, dims, c_fact, density):
    """star_table with the fact values zeroed at random (kept fp32-exact)."""
    from paper_2502_01985_b200.metadata import FactorizedTable
    ft = star_table(seed, r_fact, dims, c_fact)
    rng = np.random.default_rng(seed + 100)
    f = ft.sources[0].to_dense()
    f[rng.random(f.shape) >= density] = 0.0
    return FactorizedTable([fl_sparse(f)] + list(ft.sources[1:]), ft.mappings, ft.indicators,
                           ft.join_type, ft.r_T, ft.c_T)


def fl_sparse(a):
    from paper_2502_01985_b200.sparse import SparseMatrix
    return SparseMatrix.from_dense(a)


@pytest.mark.parametrize("model", ["linreg", "logreg"])
@pytest.mark.parametrize("dims,density", [([(2000, 17)], 0.1), ([(900, 11), (40, 3)], 0.05),
                                          ([(30000, 6)], 0.2)])
def test_glm_sparse_star_auto_csr_vs_oracle(fl, model, dims, density, monkeypatch):
    """Sparse fact tables on the CSR pass match the oracle; the session is
    deterministic run to run."""
    from paper_2502_01985_b200.trainers import GlmSession
    monkeypatch.setenv("FL_GLM_SPARSE", "1")
    ft = sparse_star(13, 100_003, dims, 20, density)
    tab = oracle.OracleTable.from_ft(ft)
    rng = np.random.default_rng(3)
    y = (rng.random(ft.r_T).astype(np.float32).astype(np.float64) if model == "linreg"
         else rng.integers(0, 2, ft.r_T).astype(np.float64))
    lr = rt.safe_learning_rate(tab)
    want = rt.train(model, tab, iterations=8, learning_rate=lr, y=y)
    h = fl.TargetHandle.factorized(ft)
    s = GlmSession(h, model, y, lr)
    try:
        path, dens = s.path
    finally:
        s.close()
    assert path == "csr" and dens < 0.25
    res = fl.train(model, h, fl.TrainConfig(iterations=8, learning_rate=lr), y.reshape(-1, 1))
    assert max_rel(res.loss_history, want["loss_history"]) < TOL
    assert max_rel(res.parameters["w"], want["parameters"]["w"]) < TOL
    again = fl.train(model, h, fl.TrainConfig(iterations=8, learning_rate=lr), y.reshape(-1, 1))
    assert np.array_equal(res.parameters["w"], again.parameters["w"])


def test_glm_deterministic(fl):
    ft = star_table(12, 90_000, [(500, 9)], 12)
    y = np.random.default_rng(1).random((ft.r_T, 1))
    h = fl.TargetHandle.factorized(ft)
    cfg = fl.TrainConfig(iterations=5, learning_rate=1e-6)
    a = fl.train("linreg", h, cfg, y)
    b = fl.train("linreg", h, cfg, y)
    assert np.array_equal(a.parameters["w"], b.parameters["w"])
    assert a.loss_history == b.loss_history


def test_first_loss_and_one_step(fl):
    """test_trainers.py:112-119, :151-160: loss_0 = 1/2||y||^2; one step from
    w0 = 0 lands at lr T^T y."""
    g = load_golden("two_source")
    h = fl.TargetHandle.factorized(g.ft)
    y = np.random.default_rng(4).standard_normal((4, 1))
    res = fl.train("linreg", h, fl.TrainConfig(iterations=1, learning_rate=1e-3), y)
    assert res.loss_history[0] == pytest.approx(0.5 * float((y ** 2).sum()), rel=1e-6)
    want = 1e-3 * (g["materialized"].T @ y)
    assert max_rel(res.parameters["w"], want) < 1e-6


def test_divergence_raises(fl):
    g = load_golden("two_source")
    h = fl.TargetHandle.factorized(g.ft)
    y = np.random.default_rng(5).standard_normal((4, 1))
    with pytest.raises(fl.DivergenceError) as exc:
        fl.train("linreg", h, fl.TrainConfig(iterations=200, learning_rate=1e3), y)
    assert exc.value.iteration > 0


def test_logreg_label_check(fl):
    g = load_golden("two_source")
    h = fl.TargetHandle.factorized(g.ft)
    with pytest.raises(fl.ConfigError, match="0/1"):
        fl.train("logreg", h, fl.TrainConfig(), np.array([[2.0], [0.0], [1.0], [0.0]]))


def test_materialized_path_agrees(fl):
    g = load_golden("star")
    m = g.meta["trainers"]["linreg"]
    cfg = fl.TrainConfig(iterations=m["iterations"], learning_rate=m["learning_rate"])
    mh = fl.TargetHandle.materialized(fl.SparseMatrix.from_dense(g["materialized"]))
    res = fl.train("linreg", mh, cfg, g["y_lin"])
    assert max_rel(res.loss_history, g["linreg_loss"]) < TOL


# ---------------------------------------------------------------------------
# K-means (trainers.py:198-246)
# ---------------------------------------------------------------------------
def _cfg(fl, m):
    return fl.TrainConfig(iterations=m["iterations"], learning_rate=m["learning_rate"],
                          k_clusters=m["k_clusters"], rank=m["rank"], seed=m["seed"])


@pytest.mark.parametrize("name,model", _cases(("kmeans",)))
def test_kmeans_matches_reference(fl, name, model):
    g = load_golden(name)
    m = g.meta["trainers"]["kmeans"]
    res = fl.train("kmeans", fl.TargetHandle.factorized(g.ft), _cfg(fl, m))
    assert len(res.loss_history) == m["iterations"]
    assert np.array_equal(res.parameters["assignments"], g["kmeans_assignments"])
    assert max_rel(res.loss_history, g["kmeans_loss"]) < TOL
    assert max_rel(res.parameters["centroids"], g["kmeans_centroids"]) < TOL


def planted_star(seed, r_fact, dims, c_fact, k, noise=0.01):
    """Star schema with planted, well-separated clusters: every dimension row
    and every fact row carries a cluster label; a fact row only references
    dimension rows of its own cluster, so T's rows cluster cleanly."""
    from paper_2502_01985_b200.metadata import FactorizedTable, block_mapping, fk_indicator
    from paper_2502_01985_b200.sparse import SparseMatrix
    rng = np.random.default_rng(seed)
    lab = rng.integers(0, k, r_fact)
    c_t = c_fact + sum(c for _, c in dims)
    cen = rng.random((k, c_fact))
    fact = (cen[lab] + noise * rng.standard_normal((r_fact, c_fact))).astype(np.float32)
    srcs = [SparseMatrix.from_dense(fact.astype(np.float64))]
    maps = [block_mapping(c_t, c_fact, 0)]
    inds = [fk_indicator(r_fact, r_fact, np.arange(r_fact))]
    off = c_fact
    for r_d, c_d in dims:
        dlab = np.arange(r_d) % k
        dcen = rng.random((k, c_d))
        dim = (dcen[dlab] + noise * rng.standard_normal((r_d, c_d))).astype(np.float32)
        # fact row i -> a random dim row with the same label
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


@pytest.mark.parametrize("k,dims,c_fact", [(16, [(3000, 30), (200, 5)], 20),
                                           (4, [(500, 9)], 12),
                                           (24, [(4000, 7)], 5),
                                           # wide dimensions: two work items per thread and
                                           # 3 / 5 prefetch slots in k_km_dim_sums
                                           (16, [(600, 150)], 10),
                                           (24, [(400, 70)], 6)])
def test_kmeans_planted_star_vs_oracle(fl, k, dims, c_fact):
    ft = planted_star(21, 60_000, dims, c_fact, k)
    tab = oracle.OracleTable.from_ft(ft)
    want = rt.kmeans(tab, 6, k, 3)
    res = fl.train("kmeans", fl.TargetHandle.factorized(ft),
                   fl.TrainConfig(iterations=6, k_clusters=k, seed=3))
    assert np.array_equal(res.parameters["assignments"], want["parameters"]["assignments"])
    assert max_rel(res.loss_history, want["loss_history"]) < TOL
    assert max_rel(res.parameters["centroids"], want["parameters"]["centroids"]) < TOL


@pytest.mark.parametrize("k,noise", [(16, 0.35), (8, 1.0)])
def test_kmeans_overlapping_clusters_certified(fl, k, noise):
    """Heavily overlapping clusters: many rows have a runner-up inside the
    tf32 screen's error bound, so the exact certification path decides them.
    One iteration (identical initial centroids): assignments may differ from
    the fp64 oracle only on true fp32-level ties."""
    ft = planted_star(5, 40_000, [(2000, 24), (300, 6)], 20, k, noise=noise)
    tab = oracle.OracleTable.from_ft(ft)
    want = rt.kmeans(tab, 1, k, 7)
    res = fl.train("kmeans", fl.TargetHandle.factorized(ft),
                   fl.TrainConfig(iterations=1, k_clusters=k, seed=7))
    diff = np.count_nonzero(res.parameters["assignments"] != want["parameters"]["assignments"])
    assert diff <= 2
    assert max_rel(res.loss_history, want["loss_history"]) < TOL


def test_kmeans_tie_and_empty_cluster(fl):
    """test_trainers.py:261-270: [[0],[0],[10]], k=3 -> [0, 0, 2], loss 0 and
    the empty cluster keeps its centroid."""
    from paper_2502_01985_b200.metadata import FactorizedTable, block_mapping, fk_indicator
    s = fl.SparseMatrix.from_dense([[0.0], [0.0], [10.0]])
    ft = FactorizedTable([s], [block_mapping(1, 1, 0)], [fk_indicator(3, 3, [0, 1, 2])],
                         "inner", 3, 1)
    res = fl.train("kmeans", fl.TargetHandle.factorized(ft),
                   fl.TrainConfig(iterations=3, k_clusters=3, seed=0))
    assert list(res.parameters["assignments"]) == [0, 0, 2]
    assert res.parameters["centroids"][1, 0] == 0.0
    assert res.loss_history[-1] == 0.0


def test_kmeans_k1_is_global_mean(fl):
    """test_trainers.py:272-277."""
    g = load_golden("star")
    res = fl.train("kmeans", fl.TargetHandle.factorized(g.ft),
                   fl.TrainConfig(iterations=2, k_clusters=1))
    want = g["materialized"].mean(axis=0)
    assert max_rel(res.parameters["centroids"][0], want) < 1e-6


def test_kmeans_materialized_and_deterministic(fl):
    g = load_golden("star3")
    m = g.meta["trainers"]["kmeans"]
    mh = fl.TargetHandle.materialized(fl.SparseMatrix.from_dense(g["materialized"]))
    res = fl.train("kmeans", mh, _cfg(fl, m))
    assert np.array_equal(res.parameters["assignments"], g["kmeans_assignments"])
    assert max_rel(res.loss_history, g["kmeans_loss"]) < TOL
    h = fl.TargetHandle.factorized(g.ft)
    a = fl.train("kmeans", h, _cfg(fl, m))
    b = fl.train("kmeans", h, _cfg(fl, m))
    assert np.array_equal(a.parameters["centroids"], b.parameters["centroids"])
    assert a.loss_history == b.loss_history


# ---------------------------------------------------------------------------
# Gaussian NMF (trainers.py:256-307)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,model", _cases(("gnmf",)))
def test_gnmf_matches_reference(fl, name, model):
    g = load_golden(name)
    m = g.meta["trainers"]["gnmf"]
    res = fl.train("gnmf", fl.TargetHandle.factorized(g.ft), _cfg(fl, m))
    assert len(res.loss_history) == m["iterations"]
    assert max_rel(res.loss_history, g["gnmf_loss"]) < TOL
    assert max_rel(res.parameters["h"], g["gnmf_h"]) < TOL
    assert max_rel(res.parameters["w"], g["gnmf_w"]) < TOL


@pytest.mark.parametrize("rank,dims,c_fact", [(32, [(2000, 50)], 20),
                                              (5, [(900, 11), (40, 3)], 12),
                                              (12, [(30000, 6)], 7),
                                              # wide dimensions: two work items per thread and
                                              # 3 / 9 prefetch slots in k_gnmf_dim_p
                                              (32, [(800, 90)], 10),
                                              (16, [(500, 220)], 8)])
def test_gnmf_random_star_vs_oracle(fl, rank, dims, c_fact):
    ft = star_table(31, 40_000, dims, c_fact)
    tab = oracle.OracleTable.from_ft(ft)
    want = rt.gaussian_nmf(tab, 6, rank, 5)
    res = fl.train("gnmf", fl.TargetHandle.factorized(ft),
                   fl.TrainConfig(iterations=6, rank=rank, seed=5))
    assert max_rel(res.loss_history, want["loss_history"]) < TOL
    assert max_rel(res.parameters["h"], want["parameters"]["h"]) < TOL
    assert max_rel(res.parameters["w"], want["parameters"]["w"]) < TOL


@pytest.mark.parametrize("rank,dims,c_fact,tc", [(32, [(2000, 50)], 20, "1"),
                                                 (32, [(2000, 50)], 20, "0"),
                                                 (20, [(700, 9), (60, 4)], 28, "1"),
                                                 (25, [], 32, "1"),
                                                 (17, [(5000, 20)], 3, "1")])
def test_gnmf_fact_pass_variants_vs_oracle(fl, rank, dims, c_fact, tc, monkeypatch):
    """Both fact passes: tcgen05 (FL_GN_TC=1, csrc/gnmf_tc.cuh; rank tiles of
    32, <= 32 streamed columns, several / no gathered sources, ragged last
    tile) and the mma.sync pass (FL_GN_TC=0)."""
    monkeypatch.setenv("FL_GN_TC", tc)
    ft = star_table(37, 30_001, dims, c_fact)
    tab = oracle.OracleTable.from_ft(ft)
    want = rt.gaussian_nmf(tab, 5, rank, 9)
    res = fl.train("gnmf", fl.TargetHandle.factorized(ft),
                   fl.TrainConfig(iterations=5, rank=rank, seed=9))
    assert max_rel(res.loss_history, want["loss_history"]) < TOL
    assert max_rel(res.parameters["h"], want["parameters"]["h"]) < TOL
    assert max_rel(res.parameters["w"], want["parameters"]["w"]) < TOL


def test_gnmf_materialized_agrees(fl):
    g = load_golden("star3")
    m = g.meta["trainers"]["gnmf"]
    mh = fl.TargetHandle.materialized(fl.SparseMatrix.from_dense(g["materialized"]))
    res = fl.train("gnmf", mh, _cfg(fl, m))
    assert max_rel(res.loss_history, g["gnmf_loss"]) < TOL
    assert max_rel(res.parameters["w"], g["gnmf_w"]) < TOL


def test_gnmf_config_errors(fl):
    g = load_golden("two_source")
    h = fl.TargetHandle.factorized(g.ft)
    with pytest.raises(fl.ConfigError):
        fl.train("gnmf", h, fl.TrainConfig(rank=5))
    neg = fl.TargetHandle.factorized(star_table(3, 300, [(10, 3)], 4, nonneg=False))
    with pytest.raises(fl.ConfigError, match="non-negative"):
        fl.train("gnmf", neg, fl.TrainConfig(rank=2))


def test_gnmf_monotone_loss(fl):
    """Acceptance C5 (test_acceptance.py:229-250): MU-NMF loss is monotone."""
    ft = star_table(8, 20_000, [(500, 9)], 10)
    res = fl.train("gnmf", fl.TargetHandle.factorized(ft), fl.TrainConfig(iterations=15, rank=8))
    lh = np.asarray(res.loss_history)
    assert np.all(np.diff(lh) <= 1e-6 * np.abs(lh[:-1]))


@pytest.mark.parametrize("name", ["clusters", "star", "star3"])
def test_kmeans_tcgen05_variant_matches_reference(fl, name, monkeypatch):
    """The opt-in tcgen05 fact pass (FL_KM_TC=1, csrc/kmeans_tc.cuh) against
    the reference goldens."""
    monkeypatch.setenv("FL_KM_TC", "1")
    g = load_golden(name)
    m = g.meta["trainers"]["kmeans"]
    res = fl.train("kmeans", fl.TargetHandle.factorized(g.ft), _cfg(fl, m))
    assert np.array_equal(res.parameters["assignments"], g["kmeans_assignments"])
    assert max_rel(res.loss_history, g["kmeans_loss"]) < TOL
    assert max_rel(res.parameters["centroids"], g["kmeans_centroids"]) < TOL


@pytest.mark.parametrize("name,model", [("star", "linreg"), ("star3", "logreg"),
                                        ("gen_outer_3_0", "linreg"), ("gen_left_2_1", "logreg")])
def test_glm_width_general_path_matches_reference(fl, name, model, monkeypatch):
    """The generic-operator GLM iteration (used for tables too wide for the
    fused passes), forced on the golden tables."""
    monkeypatch.setenv("FL_GLM_UNFUSED", "1")
    g = load_golden(name)
    m = g.meta["trainers"][model]
    y = g["y_lin"] if model == "linreg" else g["y_log"]
    res = fl.train(model, fl.TargetHandle.factorized(g.ft), _cfg(fl, m), fl.SparseMatrix.from_dense(y))
    assert max_rel(res.loss_history, g[f"{model}_loss"]) < TOL
    assert max_rel(res.parameters["w"], g[f"{model}_w"]) < TOL


@pytest.mark.parametrize("model", ["linreg", "logreg"])
def test_glm_wide_tables_vs_oracle(fl, model):
    """Widths past the fused passes: a 300-column fact table with a 260-column
    dimension, factorized and materialized."""
    ft = star_table(17, 6_000, [(60, 260)], 300)
    tab = oracle.OracleTable.from_ft(ft)
    rng = np.random.default_rng(8)
    y = (rng.random(ft.r_T) if model == "linreg" else rng.integers(0, 2, ft.r_T)).astype(np.float64)
    lr = rt.safe_learning_rate(tab)
    want = rt.train(model, tab, iterations=5, learning_rate=lr, y=y)
    for h in (fl.TargetHandle.factorized(ft),
              fl.TargetHandle.materialized(fl.SparseMatrix.from_dense(oracle.materialize(tab)))):
        res = fl.train(model, h, fl.TrainConfig(iterations=5, learning_rate=lr), y.reshape(-1, 1))
        assert max_rel(res.loss_history, want["loss_history"]) < TOL
        assert max_rel(res.parameters["w"], want["parameters"]["w"]) < TOL


def test_glm_pdl_launch_is_bit_identical(tmp_path):
    """The GLM iteration kernels are launched with programmatic dependent
    launch (prologues overlap the previous kernel's tail).  The same fit with
    FL_NO_PDL=1 (plain stream order) must give bit-identical weights and
    losses: nothing before a kernel's griddepcontrol.wait may touch its
    predecessor's outputs."""
    import os
    import subprocess
    import sys
    script = tmp_path / "fit.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.abspath(__file__))!r})\n"
        "import paper_2502_01985_b200 as fl\n"
        "from conftest import star_table\n"
        "ft = star_table(21, 20_000, [(700, 9), (30, 4)], 11)\n"
        "h = fl.TargetHandle.factorized(ft)\n"
        "y = np.random.default_rng(2).integers(0, 2, 20_000).astype(np.float64).reshape(-1, 1)\n"
        "r = fl.train('logreg', h, fl.TrainConfig(iterations=20, learning_rate=1e-4), y)\n"
        "np.save(sys.argv[1], np.concatenate([r.parameters['w'].ravel(), np.asarray(r.loss_history)]))\n")
    outs = []
    for flag in (None, "1"):
        env = dict(os.environ)
        env.pop("FL_NO_PDL", None)
        if flag:
            env["FL_NO_PDL"] = flag
        out = tmp_path / f"r{flag}.npy"
        subprocess.run([sys.executable, str(script), str(out)], check=True, env=env, timeout=300)
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("model", ["linreg", "logreg"])
@pytest.mark.parametrize("dims,rows", [([(1000, 50)], 100_000), ([(30, 7)], 70_000),
                                       ([(60_000, 13)], 120_000)])
def test_glm_solo_iteration_vs_three_kernel_path(fl, model, dims, rows, monkeypatch):
    """The one-kernel GLM iteration (sort source only: q_d staged per CTA,
    the dimension gradient from the segment sums, reduction + update by the
    last CTA) against the three-kernel path and the oracle."""
    from paper_2502_01985_b200.trainers import GlmSession
    ft = star_table(71, rows, dims, 20)
    tab = oracle.OracleTable.from_ft(ft)
    rng = np.random.default_rng(4)
    y = (rng.random(ft.r_T) if model == "linreg" else rng.integers(0, 2, ft.r_T)).astype(np.float64)
    lr = rt.safe_learning_rate(tab)
    want = rt.train(model, tab, iterations=9, learning_rate=lr, y=y)
    h = fl.TargetHandle.factorized(ft)
    got = {}
    for solo in ("1", "0"):
        monkeypatch.setenv("FL_GLM_SOLO", solo)
        s = GlmSession(h, model, y, lr)
        s.run(9)
        got[solo] = s.result(9)
        s.close()
        w, loss = got[solo]
        assert max_rel(loss, want["loss_history"]) < TOL
        assert max_rel(w, want["parameters"]["w"].ravel()) < TOL
    assert max_rel(got["1"][0], got["0"][0]) < 1e-5
    monkeypatch.setenv("FL_GLM_SOLO", "1")
    a = fl.train(model, h, fl.TrainConfig(iterations=5, learning_rate=lr), y.reshape(-1, 1))
    b = fl.train(model, h, fl.TrainConfig(iterations=5, learning_rate=lr), y.reshape(-1, 1))
    assert np.array_equal(a.parameters["w"], b.parameters["w"]) and a.loss_history == b.loss_history
