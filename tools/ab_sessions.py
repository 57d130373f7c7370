"""In-process A/B timing of session variants (env switches read at session
creation), interleaved so box-to-box and drift effects cancel.

    python tools/ab_sessions.py --workload c1 --variants "base:;red1:FL_GLM_SOLO_RED=1" \
        [--rounds 5] [--steps 50]

Each variant gets its own session on the SAME device table.  C1 steps are
timed like bench.py (L2 flushed -- written, then clean lines read -- before
each iteration, CUDA events around the iteration alone); other workloads time
`steps` back-to-back iterations.  Prints the median ms per step per variant.
"""
from __future__ import annotations

import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c1")
    ap.add_argument("--variants", required=True)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    import torch
    import paper_2502_01985_b200 as fl
    wl = dict(bench.WORKLOADS[args.workload])
    dev = torch.device("cuda", 0)
    sh = bench.make_shard(torch, wl, 0, 1, dev)
    h = bench.build_handle(fl, wl, sh)
    variants = []
    for spec in args.variants.split(";"):
        name, _, envs = spec.partition(":")
        env = dict(kv.split("=", 1) for kv in envs.split(",") if kv)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        sess, _ = bench.make_session(torch, fl, wl, h, sh, None)
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        sess.run(5)
        variants.append((name, sess))
    torch.cuda.synchronize()
    flush = args.workload == "c1"
    fb = torch.empty(64 << 20, dtype=torch.float32, device=dev) if flush else None
    fr = torch.ones(64 << 20, dtype=torch.float32, device=dev) if flush else None
    st = torch.cuda.current_stream(dev)
    res = {n: [] for n, _ in variants}
    for _ in range(args.rounds):
        for name, sess in variants:
            if flush:
                evs = []
                for _ in range(args.steps):
                    fb.fill_(1.0)
                    fr.sum()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    sess.run(1)
                    e1.record(st)
                    evs.append((e0, e1))
                torch.cuda.synchronize()
                ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
            else:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
                sess.run(args.steps)
                e1.record(st)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / args.steps
            res[name].append(ms)
    for name, sess in variants:
        kt = sess.kernel_times(5)
        v = res[name]
        print(f"{args.workload} {name:12s} median {statistics.median(v) * 1e3:9.2f} us/step  "
              f"min {min(v) * 1e3:9.2f}  all {[round(x * 1e3, 1) for x in v]}  "
              f"kernel_ms {[round(x, 4) for x in kt]}", flush=True)


if __name__ == "__main__":
    main()
