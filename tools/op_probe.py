"""Time the generic operators (lmm / transpose_lmm) at a bench workload's size.

Usage: python tools/op_probe.py [workload]   (default c2)

Compares the narrow thread-per-row lmm kernel against the generic one
(FL_NO_NARROW_LMM=1) for 1-3 operand columns: outputs must be identical,
times are CUDA-event medians over 10 calls.
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2502_01985_b200 as fl  # noqa: E402


def timed(fn, reps=10):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    fn()
    torch.cuda.synchronize()
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))


def main():
    wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    dev = torch.device("cuda")
    sh = bench.make_shard(torch, wl, 0, 1, dev)
    h = bench.build_handle(fl, wl, sh)
    del sh
    torch.cuda.empty_cache()
    r, c = h.shape
    g = torch.Generator(device=dev).manual_seed(0)
    for cx in (1, 2, 3):
        x = torch.rand((c, cx), device=dev, generator=g)
        os.environ["FL_NO_NARROW_LMM"] = "1"
        ref = h.lmm(x, traced=False).clone()
        t_main = timed(lambda: h.lmm(x, traced=False))
        os.environ.pop("FL_NO_NARROW_LMM")
        out = h.lmm(x, traced=False)
        same = bool(torch.equal(out, ref))
        t_nar = timed(lambda: h.lmm(x, traced=False))
        y = torch.rand((r, cx), device=dev, generator=g)
        t_tl = timed(lambda: h.transpose_lmm(y, traced=False))
        print(f"rows {r} cols {c} c_x {cx}: lmm generic {t_main:.3f} ms, narrow {t_nar:.3f} ms "
              f"(identical={same}); transpose_lmm {t_tl:.3f} ms", flush=True)




def wide(wl_name="c2"):
    """Wider operands (generic kernels): lmm / transpose_lmm / rmm at 8 and 32 columns."""
    wl = bench.WORKLOADS[wl_name]
    dev = torch.device("cuda")
    sh = bench.make_shard(torch, wl, 0, 1, dev)
    h = bench.build_handle(fl, wl, sh)
    del sh
    torch.cuda.empty_cache()
    r, c = h.shape
    for k in [int(v) for v in os.environ.get("OP_KS", "8,32").split(",")]:
        x = torch.rand((c, k), device=dev)
        y = torch.rand((r, k), device=dev)
        w = torch.rand((k, r), device=dev)
        print(f"k {k}: lmm {timed(lambda: h.lmm(x, traced=False), 3):.2f} ms, "
              f"transpose_lmm {timed(lambda: h.transpose_lmm(y, traced=False), 3):.2f} ms, "
              f"rmm {timed(lambda: h.rmm(w, traced=False), 3):.2f} ms", flush=True)


def crossprod(wl_name="c2"):
    """Factorized T^T T at a workload's size: CUDA-event time (median of 5)
    and the check against the dense product of the device-joined T
    (fp64 torch matmul over 10M-row chunks)."""
    wl = bench.WORKLOADS[wl_name]
    dev = torch.device("cuda")
    sh = bench.make_shard(torch, wl, 0, 1, dev)
    h = bench.build_handle(fl, wl, sh)
    del sh
    torch.cuda.empty_cache()
    r, c = h.shape
    t_cp = timed(lambda: h.crossprod(traced=False), 5)
    got = torch.as_tensor(h.crossprod(traced=False), device=dev)
    T = torch.empty((r, c), device=dev, dtype=torch.float32)
    h.materialize_dense(out=T)
    want = torch.zeros((c, c), device=dev, dtype=torch.float64)
    for r0 in range(0, r, 10_000_000):
        blk = T[r0:r0 + 10_000_000].double()
        want += blk.T @ blk
    del T, blk
    torch.cuda.empty_cache()
    err = float((got - want).norm() / want.norm())
    print(f"crossprod {wl_name}: rows {r} cols {c}: {t_cp:.3f} ms, rel err vs dense "
          f"{err:.2e}", flush=True)


if __name__ == "__main__":
    if "--crossprod" in sys.argv:
        sys.argv.remove("--crossprod")
        for w in (sys.argv[1:] or ["c2", "c3"]):
            crossprod(w)
    elif "--wide" in sys.argv:
        sys.argv.remove("--wide")
        wide(sys.argv[1] if len(sys.argv) > 1 else "c2")
    else:
        main()
