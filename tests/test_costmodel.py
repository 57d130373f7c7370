"""Cost-estimator corpus: the restated analytic cost
model and 33-entry feature vector against the REAL reference's
`extract_features` / TR&FR decision (tests/golden/features.npz, made by
tests/golden/make_features_golden.py), and the corpus format."""

import csv
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, load_golden, star_table
from paper_2502_01985_b200 import costmodel as cm

FEAT = np.load(os.path.join(GOLDEN_DIR, "features.npz"))


@pytest.mark.parametrize("name", [str(n) for n in FEAT["names"]])
def test_features_match_reference(name):
    g = load_golden(name)
    prof = cm.Profile.from_table(g.ft)
    want = FEAT[f"{name}__features"]
    got = []
    for it, k, rank in FEAT["cfgs"]:
        for par, bw in FEAT["hws"]:
            for m in cm.MODELS:
                got.append(cm.extract_features(prof, m, int(it), min(int(k), g.ft.r_T),
                                               min(int(rank), g.ft.r_T, g.ft.c_T),
                                               int(par), float(bw)))
    got = np.stack(got)
    assert got.shape == want.shape == (len(got), cm.N_FEATURES)
    np.testing.assert_array_equal(got, want)
    assert cm.tr_fr_decision(prof) == str(FEAT[f"{name}__tr_fr"])


def test_star_profile_equals_table_profile():
    ft = star_table(4, 5000, [(50, 7), (5000, 3)], 6)
    a = cm.Profile.from_table(ft)
    b = cm.Profile.star(5000, 6, [(50, 7), (5000, 3)])
    for f in ("r_t", "c_t", "m_t", "sources", "join_type", "tuple_ratios",
              "feature_ratios", "sparsity", "rho_c", "replicated"):
        assert getattr(a, f) == getattr(b, f), f
    assert cm.tr_fr_decision(b) == "factorize"          # TR 100 > 5, FR 16/7 > 1
    assert cm.tr_fr_decision(cm.Profile.star(100, 6, [(100, 3)])) == "materialize"


def test_corpus_format(tmp_path):
    p = cm.Profile.star(1000, 20, [(10, 50)])
    runs = [(cm.extract_features(p, m, 10, 8, 8, 148, 6.5e12), 1e-3, 2e-3, cm.tr_fr_decision(p))
            for m in cm.MODELS]
    path = tmp_path / "corpus.csv"
    cm.write_corpus(path, runs)
    rows = list(csv.reader(open(path)))
    assert rows[0] == list(cm.FEATURE_NAMES) + ["label", "t_fact", "t_mat", "tr_fr"]
    assert len(rows) == 5
    for r, (f, tf, tm, d) in zip(rows[1:], runs):
        assert np.array_equal(np.array([float(v) for v in r[:cm.N_FEATURES]]), f)
        assert r[cm.N_FEATURES] == "1" and r[-1] == d


def test_cost_model_errors():
    p = cm.Profile.star(10, 2, [(5, 2)])
    with pytest.raises(cm.CostModelError):
        cm.extract_features(p, "svm", 1, 1, 1, 1, 1.0)
    with pytest.raises(cm.CostModelError):
        cm.op_cost("hadamard", p, mat=True)
