#!/usr/bin/env python
"""Headline benchmark: factorized GD iterations/sec on the B200.

Workload (BASELINE.json configs[1], "C2"): 2-source star schema, fact
100,000,000 x 20 + dimension 1,000,000 x 50 (tuple ratio 100), fp32 U(0,1)
values, FK = round-robin then permuted (reference datagen.py:133-135), labels
Bernoulli(0.5) (bench.py:107), factorized logistic regression, learning rate
= the reference's safe gamma (bench.py:112-123).  One step = one full GD
iteration (all fact rows).  Inputs (8.9 GB) are far larger than L2 (126 MB),
so no L2 flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun: fact rows are sharded by FK range of the dimension
(each rank holds 1/N of the fact rows and the matching 1/N of the dimension
rows), and the per-iteration gradient + loss (c_T + 1 doubles) is all-reduced
with NCCL.  Work is fixed in total ("strong" scaling): value = iterations/s of
the whole 100M-row job.

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "factorized GD iterations/sec (logistic regression, C2 star schema)"
UNIT = "iterations/s"
R_FACT, C_FACT, TR, C_DIM = 100_000_000, 20, 100, 50


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# synthetic C2 shard (device resident)
# ---------------------------------------------------------------------------
def make_shard(torch, rows: int, dim_rows: int, seed: int, device):
    """One rank's share of the star schema, generated on the device: fact rows
    (fp32 U(0,1)), the dimension slice they reference, a permuted round-robin
    FK (fanout exactly rows/dim_rows) and Bernoulli(0.5) uint8 labels."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    fact = torch.rand((rows, C_FACT), generator=g, device=device, dtype=torch.float32)
    dim = torch.rand((dim_rows, C_DIM), generator=g, device=device, dtype=torch.float32)
    perm = torch.randperm(rows, generator=g, device=device)
    fk = (torch.arange(rows, device=device, dtype=torch.int64) % dim_rows)[perm].to(torch.int32)
    del perm
    y = torch.randint(0, 2, (rows,), generator=g, device=device, dtype=torch.uint8)
    return fact, dim, fk, y


def build_handle(fl, fact, dim, fk):
    c_t = C_FACT + C_DIM
    return fl.TargetHandle.from_arrays(
        [fact, dim], [None, fk],
        [np.arange(C_FACT, dtype=np.int32), C_FACT + np.arange(C_DIM, dtype=np.int32)],
        fact.shape[0], c_t)


def safe_gamma(torch, h, dist=None):
    """bench.py:112-123 computed factorized on the device: 1 / (max row L1 *
    max col L1); values are non-negative so |T| = T."""
    r, c = h.shape
    ones_c = torch.ones((c, 1), device="cuda", dtype=torch.float32)
    ones_r = torch.ones((r, 1), device="cuda", dtype=torch.float32)
    row_max = h.lmm(ones_c, traced=False).max().double()
    col = h.transpose_lmm(ones_r, traced=False).reshape(-1)
    if dist is not None:
        dist.all_reduce(row_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(col)
    return float(1.0 / (row_max * col.max()).item())


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port on the host cores
# ---------------------------------------------------------------------------
def cpu_sample_tables(rows: int, seed: int = 0):
    import oracle
    rng = np.random.default_rng(seed)
    dim_rows = max(1, rows // TR)
    fact = rng.random((rows, C_FACT), dtype=np.float32).astype(np.float64)
    dim = rng.random((dim_rows, C_DIM), dtype=np.float32).astype(np.float64)
    fk = rng.permutation(np.arange(rows) % dim_rows)
    y = rng.integers(0, 2, rows).astype(np.float64).reshape(-1, 1)
    tab = oracle.OracleTable([fact, dim], [np.arange(rows), fk],
                             [np.arange(C_FACT), C_FACT + np.arange(C_DIM)], rows,
                             C_FACT + C_DIM)
    return tab, y


def cpu_step(tab, y, w, lr):
    """One logistic-regression GD iteration of the reference algorithm
    (trainers.py:179-190) on the oracle's factorized operators."""
    from oracle import reference_ops as ops
    z = ops.lmm(tab, w)
    p = 1.0 / (1.0 + np.exp(-z))
    pc = np.clip(p, 1e-12, 1.0 - 1e-12)
    loss = -(y.T @ np.log(pc) + (1.0 - y).T @ np.log1p(-pc)).item()
    grad = ops.transpose_lmm(tab, p - y)
    return w - lr * grad, loss


def cpu_measure(total_budget_s: float, n_steps: int, min_rows=200_000, max_rows=20_000_000):
    """Time n_steps GD iterations on a bounded sample sized to fit the budget;
    returns (seconds per iteration at the FULL 100M rows, sample description,
    per-step full-scale times)."""
    cal_rows = 1_000_000
    tab, y = cpu_sample_tables(cal_rows)
    w = np.zeros((C_FACT + C_DIM, 1))
    cpu_step(tab, y, w, 1e-9)
    t0 = time.perf_counter()
    cpu_step(tab, y, w, 1e-9)
    per_row = (time.perf_counter() - t0) / cal_rows
    rows = int(total_budget_s / max(n_steps, 1) / per_row)
    rows = int(min(max(rows, min_rows), max_rows)) // TR * TR
    tab, y = cpu_sample_tables(rows, seed=1)
    w = np.zeros((C_FACT + C_DIM, 1))
    times = []
    for _ in range(n_steps):
        t0 = time.perf_counter()
        w, _ = cpu_step(tab, y, w, 1e-9)
        times.append(time.perf_counter() - t0)
    scale = R_FACT / rows
    full = [t * scale for t in times]
    sample = (f"{rows} fact rows x {C_FACT} + {rows // TR} x {C_DIM} (1/{scale:g} of C2), "
              f"{n_steps} GD iterations timed, linear extrapolation to 100M rows")
    return float(np.median(full)), sample, full


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle  # noqa: F401
    cores = os.cpu_count() or 1
    budget = 150.0
    per_iter_full, sample, _ = cpu_measure(budget, args.warmup + args.steps)
    value = 1.0 / per_iter_full
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_iter_full * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 logistic regression, fact 100M x 20 + dim 1M x 50 (TR 100)",
                   "parallelism": f"cpu x{cores} (numpy/BLAS)"},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=R_FACT)
    ap.add_argument("--model", default="logreg", choices=["logreg", "linreg"])
    ap.add_argument("--e2e-iters", type=int, default=100)
    ap.add_argument("--no-materialized", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2502_01985_b200 as fl
    from paper_2502_01985_b200 import _lib
    from paper_2502_01985_b200.trainers import GlmSession

    dev = torch.device("cuda", local)
    info = _lib.device_info(local)
    R = args.rows
    dim_total = R // TR
    # FK-range sharding: rank r owns dim rows [d0, d1) and the fact rows that
    # reference them (exactly fanout TR each)
    d0 = dim_total * rank // world
    d1 = dim_total * (rank + 1) // world
    rows = (d1 - d0) * TR
    fact, dim, fk, y = make_shard(torch, rows, d1 - d0, 1234 + rank, dev)
    torch.cuda.synchronize()
    h = build_handle(fl, fact, dim, fk)
    gamma = safe_gamma(torch, h, dist)
    sess = GlmSession(h, args.model, y, gamma)
    stream0 = torch.cuda.default_stream(dev)

    def step_dist(n):
        buf_ptr, n_red = sess.reduce_buffer()
        red = torch.as_tensor(_DevArray(buf_ptr, n_red, local), device=dev)
        for _ in range(n):
            sess.partial()
            dist.all_reduce(red)
            sess.update()

    def run(n):
        if world == 1:
            sess.run(n)
        else:
            step_dist(n)

    run(args.warmup)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream0)
        run(args.steps)
        e1.record(stream0)
        torch.cuda.synchronize()
    ms_total = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms_total], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_per_step = ms_total / args.steps
    value = 1e3 / ms_per_step

    # per-kernel device times (events between the three kernels, library side)
    kt = sess.kernel_times(10)
    # algorithmic bytes: fact pass = rows * (4*20 + 4 fk + b_y)
    b_y = 1 if args.model == "logreg" else 4
    fact_bytes = rows * (4 * C_FACT + 4 + b_y)
    dim_bytes = (d1 - d0) * 4 * C_DIM
    iter_bytes = fact_bytes + 2 * dim_bytes
    peak, peak_src = measured_peaks()
    achieved = fact_bytes / (kt[1] * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_fact_pass.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            pj = json.load(fh)
        if pj.get("rows") == rows:
            traffic = pj.get("dram_bytes_per_launch")
    w_host, losses = sess.result(args.warmup + args.steps + 10)
    finite = bool(np.all(np.isfinite(losses)))

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 (fp64 reductions)", "data": "synthetic",
        "config": {
            "workload": ("C2: 2-source star, fact 100M x 20 + dim 1M x 50 (TR 100), "
                         f"factorized {'logistic' if args.model == 'logreg' else 'linear'} "
                         "regression GD"),
            "fact_rows": R, "dim_rows": dim_total, "c_T": C_FACT + C_DIM,
            "l2": "inputs 8.9 GB >> L2 126 MB (no flush needed)",
            "parallelism": f"dp{world} (fact rows sharded by FK range; NCCL all-reduce of c_T+1 doubles)"
                           if world > 1 else "single GPU",
            "sm_count": info["sm_count"],
        },
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "k_glm_fact (fact-row pass)",
                     "algorithmic_bytes_per_launch": fact_bytes, "kernel_ms": kt[1],
                     "peak_source": peak_src},
        "iteration": {"algorithmic_bytes": iter_bytes,
                      "achieved_gbs": iter_bytes / (ms_per_step * 1e-3) / 1e9,
                      "frac": iter_bytes / (ms_per_step * 1e-3) / 1e9 / peak,
                      "kernel_ms": {"dim_q": kt[0], "fact_pass": kt[1], "dim_t_update": kt[2]}},
        "gpu_launches": 3 * args.steps,
        "clocks": clk.summary(),
        "loss_finite": finite,
    }

    if world == 1 and not args.no_materialized:
        out["materialized"] = bench_materialized(torch, fl, GlmSession, h, y, gamma, args,
                                                 peak)
    del fact, dim
    torch.cuda.empty_cache()
    if world == 1 and not args.no_e2e:
        out["e2e"] = bench_e2e(torch, fl, GlmSession, h, fk, y, gamma, args, rows)
    if rank == 0 and world == 1 and not args.no_cpu:
        per_iter_full, sample, _ = cpu_measure(20.0, 3)
        out["cpu_baseline"] = {"value": 1.0 / per_iter_full, "unit": UNIT,
                               "cores": os.cpu_count() or 1, "kind": "port",
                               "sample": sample}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


class _DevArray:
    """__cuda_array_interface__ view of a library-owned fp64 device buffer."""

    def __init__(self, ptr, n, device):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                         "data": (ptr, False), "version": 3}


def bench_materialized(torch, fl, GlmSession, h, y, gamma, args, peak):
    """The materialized-T baseline (north star): dense T (100M x 70 fp32) in
    HBM, same fused GD kernels on a single streamed source."""
    r, c = h.shape
    T = torch.empty((r, c), device="cuda", dtype=torch.float32)
    h.materialize_dense(out=T)
    torch.cuda.synchronize()
    mh = fl.TargetHandle.from_arrays([T], [None], [np.arange(c, dtype=np.int32)], r, c)
    del T
    torch.cuda.empty_cache()
    ms = GlmSession(mh, args.model, y, gamma)
    ms.run(args.warmup)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    steps = max(10, args.steps // 4)
    e0.record()
    ms.run(steps)
    e1.record()
    torch.cuda.synchronize()
    mps = e0.elapsed_time(e1) / steps
    kt = ms.kernel_times(5)
    b_y = 1 if args.model == "logreg" else 4
    lay = mh.layout
    mat_bytes = r * (4 * c + b_y)
    res = {"value": 1e3 / mps, "unit": UNIT, "ms_per_step": mps,
           "stream_pitch": lay["stream_pitch"],
           "fact_pass_gbs": mat_bytes / (kt[1] * 1e-3) / 1e9,
           "fact_pass_frac": mat_bytes / (kt[1] * 1e-3) / 1e9 / peak,
           "note": "dense T 100M x 70 fp32 (pitch padded to an odd float4 count)"}
    ms.close()
    del mh
    torch.cuda.empty_cache()
    return res


def bench_e2e(torch, fl, GlmSession, h, fk_dev, y_dev, gamma, args, rows):
    """End to end through the public API from pinned HOST buffers: upload
    (fact, dim, FK, labels), device layout derivation, `--e2e-iters` GD
    iterations, and the read-back of w and the loss history."""
    # host copies of the inputs (untimed)
    r, c = h.shape
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(99)
    fact_h = torch.empty((rows, C_FACT), dtype=torch.float32, pin_memory=True)
    fact_h.copy_(torch.rand((rows, C_FACT), generator=g, device=dev))
    dim_h = torch.empty((rows // TR, C_DIM), dtype=torch.float32, pin_memory=True)
    dim_h.copy_(torch.rand((rows // TR, C_DIM), generator=g, device=dev))
    fk_h = torch.empty((rows,), dtype=torch.int32, pin_memory=True)
    fk_h.copy_(fk_dev)
    y_h = torch.empty((rows,), dtype=torch.uint8, pin_memory=True)
    y_h.copy_(y_dev)
    torch.cuda.synchronize()
    J = args.e2e_iters
    t0 = time.perf_counter()
    h2 = fl.TargetHandle.from_arrays(
        [fact_h.numpy(), dim_h.numpy()], [None, fk_h.numpy()],
        [np.arange(C_FACT, dtype=np.int32), C_FACT + np.arange(C_DIM, dtype=np.int32)],
        rows, C_FACT + C_DIM)
    s2 = GlmSession(h2, args.model, y_h.numpy(), gamma)
    s2.run(J)
    w, losses = s2.result(J)
    t1 = time.perf_counter()
    h2d = fact_h.numel() * 4 + dim_h.numel() * 4 + fk_h.numel() * 4 + y_h.numel()
    d2h = 8 * (c + J)
    s2.close()
    del h2
    return {"value": J / (t1 - t0), "unit": UNIT, "h2d_bytes_per_step": h2d / J,
            "d2h_bytes_per_step": d2h / J, "iterations_per_job": J,
            "job_seconds": t1 - t0,
            "note": ("one train() job from pinned host buffers per measurement: "
                     "H2D of all inputs + device layout (FK sort) + J iterations + D2H")}


if __name__ == "__main__":
    main()
