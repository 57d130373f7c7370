"""Phase timings of one C4 (GNMF) end-to-end job through the public API, as
bench.py's e2e leg runs it: upload, t_sq (elementwise square + row_sum),
session creation (W_0 / H_0 upload), iterations, result read-back.

    python tools/e2e_c4_probe.py [--iters 100] [--jobs 3]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--jobs", type=int, default=3)
    ap.add_argument("--public", action="store_true",
                    help="time fl.train('gnmf') itself (reference-exact numpy init, pageable W_0)")
    args = ap.parse_args()
    import torch
    import paper_2502_01985_b200 as fl
    from paper_2502_01985_b200.sparse import as_dense
    from paper_2502_01985_b200.trainers import GnmfSession
    wl = dict(bench.WORKLOADS["c4"])
    dev = torch.device("cuda", 0)
    sh = bench.make_shard(torch, wl, 0, 1, dev)
    maps, c_t = bench.col_maps(wl)

    def pinned(t):
        p = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        p.copy_(t)
        return p

    host = [pinned(sh["fact"])] + [pinned(d) for d in sh["dims"]]
    fks = [pinned(f) for f in sh["fks"]]
    g = torch.Generator()
    g.manual_seed(7)
    w0_h = pinned(torch.rand((sh["rows"], wl["rank"]), generator=g, dtype=torch.float64) * 0.5)
    h0_h = pinned(torch.rand((wl["rank"], c_t), generator=g, dtype=torch.float64) * 0.5)
    del sh
    torch.cuda.synchronize()
    if args.public:
        h2 = fl.TargetHandle.from_arrays([t.numpy() for t in host],
                                         [None] + [f.numpy() for f in fks], maps, wl["rows"], c_t)
        for j in range(args.jobs):
            t0 = time.perf_counter()
            res = fl.train("gnmf", h2, fl.TrainConfig(iterations=args.iters, rank=wl["rank"], seed=3))
            t1 = time.perf_counter()
            print(f"public train('gnmf') job {j}: {t1 - t0:.2f} s, device iterations "
                  f"{res.wall_time:.2f} s, final loss {res.loss_history[-1]:.6e}", flush=True)
        return
    for j in range(args.jobs):
        ts = [("start", time.perf_counter())]

        def mark(name):
            torch.cuda.synchronize()
            ts.append((name, time.perf_counter()))

        h2 = fl.TargetHandle.from_arrays([t.numpy() for t in host],
                                         [None] + [f.numpy() for f in fks], maps, wl["rows"], c_t)
        mark("upload+layout")
        sq = h2.elementwise("square", traced=False)
        mark("elementwise square")
        from paper_2502_01985_b200.trainers import _rows_total
        t_sq = _rows_total(sq)
        mark("t_sq (device row sums)")
        del sq
        mark("free squared table")
        s2 = GnmfSession(h2, wl["rank"], w0_h.numpy(), h0_h.numpy(), t_sq)
        mark("session (W0/H0 upload)")
        s2.run(args.iters)
        mark(f"{args.iters} iterations")
        w, hh, losses = s2.result(args.iters)
        mark("result (W, H, losses to host)")
        s2.close()
        del h2
        torch.cuda.empty_cache()
        mark("close")
        print(f"job {j}: " + ", ".join(f"{n} {(t - ts[i][1]) * 1e3:.0f} ms"
                                        for i, (n, t) in enumerate(ts[1:])), flush=True)


if __name__ == "__main__":
    main()
