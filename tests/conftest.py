"""Shared fixtures: golden-vector loader and table builders.

Golden fixtures in tests/golden/*.npz were produced by the REAL reference
(tests/golden/make_golden.py).  `load_golden(name)` returns the arrays plus a
product-side FactorizedTable built from them (fp32-representable values) and
the oracle's plain-array table.
"""

from __future__ import annotations

import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device")


def pytest_collection_modifyitems(config, items):
    """Skip gpu-marked tests on a host without a usable CUDA device."""
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden_names():
    return sorted(os.path.basename(p)[:-4]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                  if os.path.basename(p) != "features.npz"
                  and not os.path.basename(p).startswith("cfg_"))


class Golden(dict):
    pass


def load_golden(name):
    from paper_2502_01985_b200.metadata import (FactorizedTable,
                                                IndicatorMatrix,
                                                MappingMatrix, fk_indicator)
    from paper_2502_01985_b200.sparse import SparseMatrix

    raw = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    g = Golden({k: raw[k] for k in raw.files})
    meta = json.loads(str(g["meta"]))
    g.meta = meta
    r_t, c_t = meta["r_T"], meta["c_T"]
    srcs, maps, inds = [], [], []
    for k in range(meta["n_sources"]):
        s = g[f"src{k}"]
        srcs.append(SparseMatrix.from_dense(s))
        mst = g[f"map_sel_t{k}"]
        ok = mst >= 0
        maps.append(MappingMatrix(SparseMatrix.from_coo(
            c_t, s.shape[1], mst[ok], np.nonzero(ok)[0], np.ones(int(ok.sum())))))
        inds.append(fk_indicator(r_t, s.shape[0], g[f"ind_sel{k}"]))
    g.ft = FactorizedTable(srcs, maps, inds, meta["join_type"], r_t, c_t)
    return g


@pytest.fixture(params=golden_names())
def golden(request):
    return load_golden(request.param)


def star_table(seed, r_fact, dims, c_fact, *, nonneg=True, sort_fk=False):
    """Synthetic star schema as (FactorizedTable, dense fact, [(dim, fk)]).
    Values are float32-representable uniform(0,1)."""
    from paper_2502_01985_b200.metadata import (FactorizedTable,
                                                block_mapping, fk_indicator)
    from paper_2502_01985_b200.sparse import SparseMatrix

    rng = np.random.default_rng(seed)
    c_t = c_fact + sum(c for _, c in dims)
    fact = rng.random((r_fact, c_fact)).astype(np.float32).astype(np.float64)
    if not nonneg:
        fact -= 0.5
    srcs = [SparseMatrix.from_dense(fact)]
    maps = [block_mapping(c_t, c_fact, 0)]
    inds = [fk_indicator(r_fact, r_fact, np.arange(r_fact))]
    off = c_fact
    for r_d, c_d in dims:
        dim = rng.random((r_d, c_d)).astype(np.float32).astype(np.float64)
        fk = rng.permutation(np.arange(r_fact) % r_d)
        if sort_fk:
            fk = np.sort(fk)
        srcs.append(SparseMatrix.from_dense(dim))
        maps.append(block_mapping(c_t, c_d, off))
        inds.append(fk_indicator(r_fact, r_d, fk))
        off += c_d
    return FactorizedTable(srcs, maps, inds, "inner", r_fact, c_t)


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
