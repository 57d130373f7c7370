#!/usr/bin/env python
"""Probe the MN-major tf32 tcgen05 operand layout on the B200 (fl_tc_probe)
and how kind::tf32 treats fp32 operand bits below the tf32 mantissa
(fl_tc_selftest mode 0 with non-tf32 inputs).  Prints a report; run with
`python tools/tc_probe.py` on the GPU box."""

import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_01985_b200 import _lib  # noqa: E402


def ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def tf32_trunc(x):
    return (x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def tf32_round(x):
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x1000) & 0xFFFFE000      # round half away (magnitude)
    return u.astype(np.uint32).view(np.float32)


def main():
    lib = _lib.load()
    print("== mode 0: TMA 128B/32B-atom swizzle layout of a 32 x 32 fp32 tile")
    tile = np.arange(1024, dtype=np.float32)
    dump = np.zeros(1024, dtype=np.float32)
    _lib.call("fl_tc_probe", 0, ptr(tile), None, None, ptr(dump), 0, 0, None)
    d = dump.astype(np.int64)
    for r in range(10):
        row = d[r * 32:(r + 1) * 32]
        src_rows = row // 32
        src_cols = row % 32
        print(f" smem row {r}: src row {sorted(set(src_rows.tolist()))} cols "
              f"{src_cols.tolist()}")

    rng = np.random.default_rng(0)
    for K in (16, 32):
        A = (rng.integers(-8, 9, (128, K)) / 4).astype(np.float32)
        for mode, N in ((1, 32), (1, 64), (2, 32), (2, 64)):
            B = (rng.integers(-8, 9, (K, N)) / 4).astype(np.float32)
            want = A.astype(np.float64) @ B.astype(np.float64)
            cands = [(K * 128, 1024, 1), (1024, K * 128, 1), (16, 1024, 1), (K * 128, 1024, 2),
                     (1024, K * 128, 2)]
            for lbo, sbo, lay in cands:
                D = np.zeros((128, N), dtype=np.float32)
                prm = np.array([lbo, sbo, lay], dtype=np.int32)
                try:
                    _lib.call("fl_tc_probe", mode, ptr(A), ptr(B), ptr(D), None, K, N, ptr(prm))
                except Exception as e:      # noqa: BLE001
                    print(f" mode {mode} K {K} N {N} lbo {lbo} sbo {sbo} layout {lay}: ERROR {e}")
                    continue
                err = float(np.max(np.abs(D - want)))
                print(f" mode {mode} K {K} N {N} lbo {lbo} sbo {sbo} layout {lay}: "
                      f"max err {err:.3g} {'OK' if err == 0 else ''}")

    print("== kind::tf32 treatment of fp32 operand bits (selftest mode 0)")
    K, N = 32, 32
    A = rng.random((128, K)).astype(np.float32) + 1.0
    Bm = np.eye(K, N, dtype=np.float32)
    D = np.zeros((128, N), dtype=np.float32)
    _lib.call("fl_tc_selftest", 0, ptr(A), ptr(Bm), ptr(D), K, N, None)
    print(" exact fp32:", float(np.max(np.abs(D - A))),
          " truncated:", float(np.max(np.abs(D - tf32_trunc(A)))),
          " rounded:", float(np.max(np.abs(D - tf32_round(A)))))


if __name__ == "__main__":
    main()
