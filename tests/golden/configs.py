"""Deterministic numpy generators of the BASELINE.json config shapes used by
the config-scale parity tests (tests/test_gpu_configs.py) and by the script
that runs the REAL reference on them (tests/golden/make_golden_configs.py).

Both sides call the same functions, so the GPU box regenerates bit-identical
inputs from a seed and only the reference's outputs travel as fixtures.
Values are float32-representable (fp32 device storage is exact).

  c1_arrays   BASELINE configs[0] exactly: fact 1,000,000 x 20 + dim
              10,000 x 50, U(0,1); FK = round-robin then permuted (tuple
              ratio 100, reference datagen.py:133-135); y ~ U(0,1)
  c3_arrays   configs[2] shape at 1M rows: fact 1,000,000 x 20 + dim A
              10,000 x 60 (TR 100) + dim B 1,000 x 5 (TR 1000); 16 planted
              clusters with noise sigma 0.01 (dimension row r has cluster
              r mod 16; a fact row references dimension rows of its own
              cluster only)
  c4_arrays   configs[3] shape at 1M rows: fact 1,000,000 x 20 + dim
              10,000 x 50, U(0,1) (non-negative), for GNMF rank 32
"""

from __future__ import annotations

import numpy as np


def _f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def _rr_fk(rng, rows, r_d):
    return rng.permutation(np.arange(rows, dtype=np.int64) % r_d)


def c1_arrays(seed=0, rows=1_000_000):
    """(sources, ind_sels, col_maps, r_T, c_T, y) -- fact + one dimension."""
    rng = np.random.default_rng(seed)
    fact = _f32(rng.random((rows, 20)))
    dim = _f32(rng.random((rows // 100, 50)))
    fk = _rr_fk(rng, rows, rows // 100)
    y = _f32(rng.random(rows))
    maps = [np.arange(20), 20 + np.arange(50)]
    return [fact, dim], [np.arange(rows), fk], maps, rows, 70, y


def c3_arrays(seed=3, rows=1_000_000, k=16, sigma=0.01):
    rng = np.random.default_rng(seed)
    r_a, r_b = rows // 100, rows // 1000
    fk_a = _rr_fk(rng, rows, r_a)
    lab = fk_a % k
    cen_f = rng.random((k, 20))
    cen_a = rng.random((k, 60))
    cen_b = rng.random((k, 5))
    fact = _f32(cen_f[lab] + sigma * rng.standard_normal((rows, 20)))
    dim_a = _f32(cen_a[np.arange(r_a) % k] + sigma * rng.standard_normal((r_a, 60)))
    dim_b = _f32(cen_b[np.arange(r_b) % k] + sigma * rng.standard_normal((r_b, 5)))
    fk_b = lab + k * rng.integers(0, r_b // k, rows)
    maps = [np.arange(20), 20 + np.arange(60), 80 + np.arange(5)]
    return [fact, dim_a, dim_b], [np.arange(rows), fk_a, fk_b], maps, rows, 85, lab


def c3_seed(rows=1_000_000, k=16, lab=None, start=0):
    """Smallest training seed >= start whose K-means seed rows (trainers.py:
    209-210: sorted rng.choice of k distinct rows) fall in k distinct planted
    clusters -- the well-separated case the north star requires identical
    assignments on (no planted cluster is split between two centroids)."""
    if lab is None:
        lab = c3_arrays(rows=rows, k=k)[5]
    s = start
    while True:
        pick = np.random.default_rng(s).choice(rows, size=k, replace=False)
        if np.unique(lab[pick]).size == k:
            return s
        s += 1


def c4_arrays(seed=4, rows=1_000_000):
    rng = np.random.default_rng(seed)
    fact = _f32(rng.random((rows, 20)))
    dim = _f32(rng.random((rows // 100, 50)))
    fk = _rr_fk(rng, rows, rows // 100)
    maps = [np.arange(20), 20 + np.arange(50)]
    return [fact, dim], [np.arange(rows), fk], maps, rows, 70


def fanout_arrays(seed=5, rows=10_000_000):
    """One-row dimension under `rows` fact rows (fanout = rows): the GLM
    segmented scan carries one segment across every warp of the pass."""
    rng = np.random.default_rng(seed)
    fact = _f32(rng.random((rows, 8)))
    dim = _f32(rng.random((1, 6)))
    maps = [np.arange(8), 8 + np.arange(6)]
    y = _f32(rng.random(rows))
    return [fact, dim], [np.arange(rows), np.zeros(rows, dtype=np.int64)], maps, rows, 14, y
