"""Pin the CPU oracle at the BASELINE config shapes against the real
reference's outputs (tests/golden/cfg_*.npz, make_golden_configs.py).  No
GPU needed; ~30 s in total."""

import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN_DIR

sys.path.insert(0, GOLDEN_DIR)
import configs  # noqa: E402

import oracle  # noqa: E402
from oracle import reference_trainers as rt  # noqa: E402


def golden(name):
    raw = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    g = {k: raw[k] for k in raw.files}
    g["meta"] = json.loads(str(g["meta"]))
    return g


def table(srcs, sels, maps, r_t, c_t):
    return oracle.OracleTable(list(srcs), [np.asarray(s, dtype=np.int64) for s in sels],
                              [np.asarray(m, dtype=np.int64) for m in maps], r_t, c_t)


def max_rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def test_oracle_c1_full_config():
    g = golden("cfg_c1")
    srcs, sels, maps, r_t, c_t, y = configs.c1_arrays()
    tab = table(srcs, sels, maps, r_t, c_t)
    assert rt.safe_learning_rate(tab) == pytest.approx(g["meta"]["learning_rate"], rel=1e-12)
    want = rt.train("linreg", tab, iterations=100, learning_rate=g["meta"]["learning_rate"], y=y)
    assert max_rel(want["loss_history"], g["loss"]) < 1e-10
    assert max_rel(want["parameters"]["w"].ravel(), g["w"]) < 1e-10


def test_oracle_c3_shape_kmeans():
    g = golden("cfg_c3")
    m = g["meta"]
    srcs, sels, maps, r_t, c_t, lab = configs.c3_arrays()
    assert configs.c3_seed(lab=lab, start=m["seed"]) == m["seed"]
    tab = table(srcs, sels, maps, r_t, c_t)
    want = rt.kmeans(tab, m["iterations"], m["k_clusters"], m["seed"])
    assert np.array_equal(want["parameters"]["assignments"], g["assignments"].astype(np.int64))
    assert max_rel(want["parameters"]["centroids"], g["centroids"]) < 1e-10
    assert max_rel(want["loss_history"], g["loss"]) < 1e-10


def test_oracle_c4_shape_gnmf():
    g = golden("cfg_c4")
    m = g["meta"]
    srcs, sels, maps, r_t, c_t = configs.c4_arrays()
    tab = table(srcs, sels, maps, r_t, c_t)
    want = rt.gaussian_nmf(tab, m["iterations"], m["rank"], m["seed"])
    assert max_rel(want["loss_history"], g["loss"]) < 1e-10
    assert max_rel(want["parameters"]["h"], g["h"]) < 1e-10
    w = want["parameters"]["w"]
    assert max_rel(w.sum(axis=0), g["w_colsum"]) < 1e-10
    assert max_rel(w[::997], g["w_rows"]) < 1e-10
