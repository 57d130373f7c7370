"""Several sessions alive on one table with different launch plans (the solo
one-kernel GLM iteration with its shared-memory plan, and the three-kernel
iteration): creating the second must not break the first's launches (the
per-kernel dynamic shared-memory limit is process-wide and only raised), and
every variant of the solo tail reaches the same weights."""

import os

import numpy as np
import pytest

from conftest import star_table

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fl():
    import paper_2502_01985_b200 as fl
    return fl


def _session(fl, h, y, env):
    from paper_2502_01985_b200.trainers import GlmSession
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return GlmSession(h, "linreg", y, 1e-7)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_sessions_with_different_plans_coexist(fl):
    # C1-like shape: one sort-source dimension, fanout 100 -> the solo path
    ft = star_table(5, 200_000, [(2000, 50)], 20)
    h = fl.TargetHandle.factorized(ft)
    y = np.random.default_rng(0).random(200_000).astype(np.float32)
    variants = [{}, {"FL_GLM_SOLO_S0": "0"}, {"FL_GLM_SOLO": "0"}]
    sess = [_session(fl, h, y, v) for v in variants]
    assert sess[0].path[0] == "solo" and sess[2].path[0] != "solo"
    out = []
    for s in sess:   # the first sessions launch after the later ones were planned
        s.run(7)
        s.kernel_times(2)   # direct (non-graph) launches
        out.append(s.result(7))
    w0, l0 = out[0]
    w1, l1 = out[1]   # S_d span via L2: same sums, identical results
    assert np.array_equal(w1, w0) and np.array_equal(l1, l0)
    w3, l3 = out[2]
    assert np.max(np.abs(w3 - w0)) <= 1e-5 * np.max(np.abs(w0))
    assert np.max(np.abs(l3 - l0) / np.abs(l0)) <= 1e-5


def test_staged_host_copies_match_direct(fl):
    """Pageable host buffers of >= 128 MB go through the pinned staging ring
    (GNMF W_0 upload, W read-back): bit-identical to the driver's copies."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from conftest import star_table
import paper_2502_01985_b200 as fl
from paper_2502_01985_b200.trainers import GnmfSession
ft = star_table(9, 1_100_000, [(11_000, 12)], 20)
h = fl.TargetHandle.factorized(ft)
rng = np.random.default_rng(4)
w0 = rng.random((1_100_000, 32)) * 0.1     # 282 MB, pageable
h0 = rng.random((32, 32)) * 0.1
s = GnmfSession(h, 32, w0, h0, 1.0)
s.run(2)
w, hh, loss = s.result(2)
np.save(sys.argv[1], w)
'''
    import os
    import tempfile
    here = os.path.dirname(os.path.abspath(__file__))
    outs = []
    with tempfile.TemporaryDirectory() as td:
        for env in ({}, {"FL_NO_STAGED_COPY": "1"}):
            p = os.path.join(td, f"w{len(outs)}.npy")
            e = dict(os.environ, **env)
            r = subprocess.run([sys.executable, "-c", code, p], cwd=here, env=e,
                               capture_output=True, text=True, timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            outs.append(np.load(p))
    assert outs[0].shape == (1_100_000, 32)
    assert np.array_equal(outs[0], outs[1])


def test_pageable_table_upload_staged_bit_exact(fl):
    """A >= 128 MB pageable fact block is uploaded through the pinned staging
    ring (fl_table_finalize): the join is still bit-exact."""
    rng = np.random.default_rng(12)
    r, cf, rd, cd = 2_000_000, 20, 20_000, 6
    fact = rng.random((r, cf), dtype=np.float32)          # 160 MB, numpy-owned (pageable)
    dim = rng.random((rd, cd), dtype=np.float32)
    fk = rng.permutation(np.arange(r) % rd).astype(np.int32)
    maps = [np.arange(cf, dtype=np.int32), cf + np.arange(cd, dtype=np.int32)]
    h = fl.TargetHandle.from_arrays([fact, dim], [None, fk], maps, r, cf + cd)
    got = h.materialize_dense()
    assert np.array_equal(got[:, :cf], fact)
    assert np.array_equal(got[:, cf:], dim[fk])
