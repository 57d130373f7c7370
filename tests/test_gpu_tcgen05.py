"""Known-answer tests of the tcgen05 operand layouts (csrc/tc05.cuh) through
`fl_tc_selftest`: tf32-exact inputs (small integers), so D must be exact."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run(mode, K, N, seed=0):
    from paper_2502_01985_b200 import _lib
    rng = np.random.default_rng(seed)
    A = rng.integers(-4, 5, (128, K)).astype(np.float32)
    B = rng.integers(-4, 5, (K, N)).astype(np.float32)
    D = np.empty((128, N), dtype=np.float32)
    _lib.call("fl_tc_selftest", mode, A.ctypes.data_as(C.c_void_p), B.ctypes.data_as(C.c_void_p),
              D.ctypes.data_as(C.c_void_p), K, N, None)
    return A, B, D


@pytest.mark.parametrize("mode,K,N", [(0, 24, 16), (0, 128, 64), (2, 32, 32)])
def test_layouts_exact(mode, K, N):
    A, B, D = run(mode, K, N)
    assert np.array_equal(D, A @ B)


@pytest.mark.parametrize("K,N", [(128, 16), (128, 32), (64, 48)])
def test_padded_transposed_tiles(K, N):
    """The F^T / one-hot^T tiles: 32 stored rows, padded K-chunk stride."""
    A, B, D = run(1, K, N)
    assert np.array_equal(D[:32], A[:32] @ B)
