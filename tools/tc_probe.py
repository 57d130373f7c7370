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


def one(mode, K, N, lbo, sbo, lay):
    """one MN-major MMA check (run in its own process: a bad descriptor
    faults and poisons the CUDA context)"""
    rng = np.random.default_rng(K * 1000 + N)
    A = (rng.integers(-8, 9, (128, K)) / 4).astype(np.float32)
    B = (rng.integers(-8, 9, (K, N)) / 4).astype(np.float32)
    want = A.astype(np.float64) @ B.astype(np.float64)
    D = np.zeros((128, N), dtype=np.float32)
    prm = np.array([lbo, sbo, lay], dtype=np.int32)
    _lib.call("fl_tc_probe", mode, ptr(A), ptr(B), ptr(D), None, K, N, ptr(prm))
    err = float(np.max(np.abs(D - want)))
    print(f" mode {mode} K {K} N {N} lbo {lbo} sbo {sbo} layout {lay}: max err {err:.3g}"
          f" {'OK' if err == 0 else ''}", flush=True)


def truncation():
    rng = np.random.default_rng(5)
    K, N = 32, 32
    A = rng.random((128, K)).astype(np.float32) + 1.0
    Bm = np.eye(K, N, dtype=np.float32)
    D = np.zeros((128, N), dtype=np.float32)
    _lib.call("fl_tc_selftest", 0, ptr(A), ptr(Bm), ptr(D), K, N, None)
    print(" exact fp32:", float(np.max(np.abs(D - A))),
          " truncated:", float(np.max(np.abs(D - tf32_trunc(A)))),
          " rounded:", float(np.max(np.abs(D - tf32_round(A)))), flush=True)


def timing():
    """cycles per kind::tf32 MMA (M x N x 8) issued back to back, K-major vs
    MN-major operands, 1 CTA and one CTA per SM; then the same chain spread
    round-robin over 1-8 independent accumulators"""
    _lib.load()
    print(f"{'M':>4} {'N':>4} {'A':>3} {'B':>3} {'1 CTA':>8} {'148 CTAs':>9}  cycles / MMA, one "
          f"accumulator", flush=True)
    lay = {0: "K", 1: "MN"}
    for M in (64, 128):
        for N in (32, 64, 128, 256):
            for a_mn, b_mn in ((0, 0), (1, 1), (1, 0), (0, 1)):
                out = []
                for ctas in (1, 148):
                    c = C.c_double()
                    _lib.call("fl_tc_timing", M, N, a_mn, b_mn, 200, ctas, 1, C.byref(c))
                    out.append(c.value)
                print(f"{M:>4} {N:>4} {lay[a_mn]:>3} {lay[b_mn]:>3} {out[0]:8.1f} {out[1]:9.1f}"
                      f"   floor max(M,128) N / 256 = {max(M, 128) * N / 256:.0f}", flush=True)
    print("independent accumulators (148 CTAs, MN-major A and B):", flush=True)
    for M, N in ((64, 32), (128, 32), (128, 64), (128, 128)):
        row = []
        for nacc in (1, 2, 4, 8):
            if N * nacc > 512:
                row.append("   -")
                continue
            c = C.c_double()
            _lib.call("fl_tc_timing", M, N, 1, 1, 200, 148, nacc, C.byref(c))
            row.append(f"{c.value:6.1f}")
        print(f" M {M:>3} N {N:>3}: nacc 1 / 2 / 4 / 8 -> " + " ".join(row), flush=True)
    print("kind::f16 (bf16 operands, K = 16 per MMA), 148 CTAs, one accumulator:", flush=True)
    for M in (64, 128):
        row = []
        for N in (32, 64, 96, 128, 256):
            c = C.c_double()
            _lib.call("fl_tc_timing", M, N, 0, 0, 200, 148, 1 | 256, C.byref(c))
            row.append(f"N {N}: {c.value:6.1f}")
        print(f" M {M:>3}: " + "  ".join(row), flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "timing":
        timing()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one(*(int(v) for v in sys.argv[2:8]))
        return
    if len(sys.argv) > 1 and sys.argv[1] == "trunc":
        truncation()
        return
    import subprocess
    print("== kind::tf32 treatment of fp32 operand bits (selftest mode 0)", flush=True)
    subprocess.run([sys.executable, __file__, "trunc"], timeout=120)
    print("== MN-major candidates", flush=True)
    for K in (16, 32):
        for mode, N in ((1, 32), (2, 32), (1, 64), (2, 64)):
            grp = K * 128
            for lbo, sbo in ((grp, 512), (512, grp), (grp, 1024), (1024, grp), (grp, 128),
                             (128, grp), (grp, 256), (256, grp)):
                subprocess.run([sys.executable, __file__, "one", str(mode), str(K), str(N),
                                str(lbo), str(sbo), "1"], timeout=120)
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

if __name__ == "__main__":
    main()
