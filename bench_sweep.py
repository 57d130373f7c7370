#!/usr/bin/env python
"""C5 (BASELINE.json configs[4]): factorize-vs-materialize timings on the B200
over a tuple-ratio x feature-ratio grid -- the training data of the
reference's materialize/factorize cost estimator (features.py / estimator.py,
SURVEY.md §8 row f2), regenerated from B200 timings.

Grid: fact R x 20 (default R = 10M), one dimension table
with tuple ratio TR = R / r_dim in {1, 2, 5, 10, 20, 50, 100, 200, 500, 1000}
and feature ratio FR = c_dim / c_fact in {0.1, 0.2, 0.5, 1, 2, 5, 10}
(Morpheus' d_dim / d_fact; the reference's own `feature_ratio` is c_T / c_k,
metadata.py:239).  Per cell and model, the fused factorized session and the
same session on the materialized dense T (joined on the device) are timed
with CUDA events over `--iters` iterations after a warm-up.  Models whose
fused kernels do not cover a width (K-means / GNMF on very wide materialized
T) are recorded as unsupported.

Output: a CSV table (one row per cell x model: shape, TR, FR, model,
t_fact, t_mat per iteration, label = factorized faster), a JSON summary, and
`<out>_corpus.csv`: the same runs as the reference estimator's training
corpus (33-entry feature vectors of `paper_2502_01985_b200.costmodel`, which
reproduces the reference's `extract_features` bit for bit, label, t_fact /
t_mat of the whole `--iters`-iteration run, TR&FR decision; the reference's
`estimator.read_corpus` format).  Hardware group: parallelism = SMs,
memory bandwidth = MEASURED_PEAKS.json's HBM copy bandwidth.

    python bench_sweep.py [--rows 10000000] [--iters 10] [--out profiles/r01_c5_sweep]
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TRS = [1, 2, 5, 10, 20, 50, 100, 200, 500, 1000]
FRS = [0.1, 0.2, 0.5, 1, 2, 5, 10]
C_FACT = 20
MODELS = ["linreg", "logreg", "kmeans", "gnmf"]


def time_session(torch, make, iters):
    """(seconds per iteration, or None if the model does not cover the shape)."""
    from paper_2502_01985_b200 import _lib
    try:
        s = make()
    except (_lib.FlError, ValueError) as e:
        if "supports" in str(e) or "too wide" in str(e) or "budget" in str(e):
            return None
        raise
    try:
        s.run(2)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        s.run(iters)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3 / iters
    finally:
        s.close()


def sessions(torch, h, model, y_lin, y_log, rows):
    from paper_2502_01985_b200.trainers import (GlmSession, GnmfSession, KMeansSession,
                                                kmeans_init)
    if model == "linreg":
        return lambda: GlmSession(h, "linreg", y_lin, 1e-9)
    if model == "logreg":
        return lambda: GlmSession(h, "logreg", y_log, 1e-9)
    if model == "kmeans":
        return lambda: KMeansSession(h, 8, kmeans_init(h, 8, 0))
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    c = h.shape[1]

    def mk():
        w0 = torch.rand((rows, 8), generator=g, device="cuda", dtype=torch.float64)
        h0 = torch.rand((8, c), generator=g, device="cuda", dtype=torch.float64)
        return GnmfSession(h, 8, w0, h0, 1.0)
    return mk


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_c5_sweep"))
    ap.add_argument("--models", default=",".join(MODELS))
    args = ap.parse_args()
    import torch
    import paper_2502_01985_b200 as fl
    dev = torch.device("cuda")
    R = args.rows
    models = args.models.split(",")
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    fact = torch.rand((R, C_FACT), generator=g, device=dev)
    y_lin = torch.rand((R,), generator=g, device=dev)
    y_log = torch.randint(0, 2, (R,), generator=g, device=dev, dtype=torch.uint8)
    rows_out = []
    t_start = time.time()
    for tr in TRS:
        r_dim = max(1, R // tr)
        fk = (torch.arange(R, device=dev) % r_dim)[torch.randperm(R, generator=g, device=dev)]
        fk = fk.to(torch.int32)
        for fr in FRS:
            c_dim = max(1, int(round(fr * C_FACT)))
            dim = torch.rand((r_dim, c_dim), generator=g, device=dev)
            c_t = C_FACT + c_dim
            maps = [np.arange(C_FACT, dtype=np.int32), C_FACT + np.arange(c_dim, dtype=np.int32)]
            h = fl.TargetHandle.from_arrays([fact, dim], [None, fk], maps, R, c_t)
            T = torch.empty((R, c_t), device=dev)
            h.materialize_dense(out=T)
            torch.cuda.synchronize()
            hm = fl.TargetHandle.from_arrays([T], [None], [np.arange(c_t, dtype=np.int32)], R, c_t)
            del T
            torch.cuda.empty_cache()
            for model in models:
                tf = time_session(torch, sessions(torch, h, model, y_lin, y_log, R), args.iters)
                tm = time_session(torch, sessions(torch, hm, model, y_lin, y_log, R), args.iters)
                rows_out.append({"tuple_ratio": tr, "feature_ratio": fr, "r_T": R, "c_T": c_t,
                                 "r_dim": r_dim, "c_dim": c_dim, "model": model,
                                 "t_fact": tf, "t_mat": tm,
                                 "label": (tf is not None and tm is not None and tf < tm)})
            del h, hm, dim
            torch.cuda.empty_cache()
        del fk
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out + ".csv", "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(rows_out[0]))
        w.writeheader()
        for r in rows_out:
            w.writerow(r)
    sup = [r for r in rows_out if r["t_fact"] is not None and r["t_mat"] is not None]
    summary = {
        "grid": {"tuple_ratios": TRS, "feature_ratios": FRS, "fact_rows": R, "c_fact": C_FACT,
                 "iters": args.iters, "models": models},
        "cells": len(rows_out), "timed": len(sup),
        "factorized_faster": sum(1 for r in sup if r["label"]),
        "by_model": {m: {"fact_faster": sum(1 for r in sup if r["model"] == m and r["label"]),
                         "timed": sum(1 for r in sup if r["model"] == m),
                         "median_speedup_mat_over_fact": float(np.median(
                             [r["t_mat"] / r["t_fact"] for r in sup if r["model"] == m]))
                         if any(r["model"] == m for r in sup) else None}
                     for m in models},
        "seconds": time.time() - t_start,
    }
    # the estimator corpus (reference estimator.py:54-61 format)
    from paper_2502_01985_b200 import costmodel as cm
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    bw = 6650e9
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        with open(pk) as fh:
            bw = float(json.load(fh).get("hbm_gbs", 6650.0)) * 1e9
    corpus = []
    for r in sup:
        prof = cm.Profile.star(R, C_FACT, [(r["r_dim"], r["c_dim"])])
        f = cm.extract_features(prof, r["model"], args.iters, 8, 8, sms, bw)
        if r["t_fact"] * args.iters == r["t_mat"] * args.iters:
            continue   # exact tie: no label
        corpus.append((f, r["t_fact"] * args.iters, r["t_mat"] * args.iters,
                       cm.tr_fr_decision(prof)))
    cm.write_corpus(args.out + "_corpus.csv", corpus)
    summary["corpus"] = {"runs": len(corpus), "parallelism": sms, "memory_bandwidth": bw,
                         "path": os.path.basename(args.out) + "_corpus.csv"}
    with open(args.out + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
