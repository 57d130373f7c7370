"""World-size-2 gloo tests of the multi-GPU host logic (no GPU): the shard
plan, the rank-local tables and the all-reduce algebra of every trainer's
reduce buffer.  Per-rank partials are computed with the CPU oracle (test
infrastructure) on the rank-local tables `distributed.shard_arrays` builds;
the all-reduced sums must equal the single-process values."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import reference_ops as rops
from paper_2502_01985_b200 import distributed as D


def star(seed=3, r=3000, dims=((40, 5), (7, 3)), c_fact=6, left=False):
    rng = np.random.default_rng(seed)
    srcs = [rng.random((r, c_fact))]
    sels = [None]
    for r_d, c_d in dims:
        srcs.append(rng.random((r_d, c_d)))
        fk = rng.permutation(np.arange(r) % r_d)
        if left:
            fk[rng.random(r) < 0.1] = -1
        sels.append(fk)
    return srcs, sels


def oracle_table(srcs, sels):
    r = srcs[0].shape[0]
    maps, off = [], 0
    for s in srcs:
        maps.append(off + np.arange(s.shape[1]))
        off += s.shape[1]
    ind = [np.arange(r) if s is None else np.asarray(s, dtype=np.int64) for s in sels]
    return oracle.OracleTable([np.asarray(s, float) for s in srcs], ind, maps, r, off)


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("left", [False, True])
def test_plan_partitions_rows(world, left):
    srcs, sels = star(left=left)
    plans = D.plan_shards(sels[1], srcs[1].shape[0], world)
    allrows = np.concatenate([p.rows for p in plans])
    assert np.array_equal(np.sort(allrows), np.arange(srcs[0].shape[0]))
    sizes = [p.n_rows for p in plans]
    assert max(sizes) - min(sizes) <= 2 * 75 + 1     # within ~ one fanout
    for p in plans:          # each rank owns exactly the dim rows it references
        fk = np.asarray(sels[1])[p.rows]
        fk = fk[fk >= 0]
        assert np.all((fk >= p.dim_lo) & (fk < p.dim_hi))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    srcs, sels = star(left=True)
    full = oracle_table(srcs, sels)
    plan = D.plan_shards(sels[1], srcs[1].shape[0], world)[rank]
    ls, li = D.shard_arrays(srcs, sels, plan, shard_source=1)
    local = oracle_table(ls, li)
    rng = np.random.default_rng(0)
    out = {}
    # GLM: gradient + loss buffer (c_T + 1)
    w = rng.random((full.c_T, 1))
    y = rng.random((full.r_T, 1))
    r_loc = rops.lmm(local, w) - y[plan.rows]
    buf = torch.tensor(np.concatenate([rops.transpose_lmm(local, r_loc).ravel(),
                                       [0.5 * float((r_loc ** 2).sum())]]))
    D.all_reduce_(buf, dist)
    r_full = rops.lmm(full, w) - y
    want = np.concatenate([rops.transpose_lmm(full, r_full).ravel(),
                           [0.5 * float((r_full ** 2).sum())]])
    out["glm"] = float(np.max(np.abs(buf.numpy() - want)) / np.max(np.abs(want)))
    # K-means: seed rows gathered by slot, then sums + counts
    k = 5
    pick = D.kmeans_seed_rows(full.r_T, k, 7)
    slots, lrows = D.local_seed_slots(plan, pick)
    seed = torch.zeros((k, full.c_T), dtype=torch.float64)
    if slots.size:
        sel = np.zeros((slots.size, local.r_T))
        sel[np.arange(slots.size), lrows] = 1.0
        seed[torch.as_tensor(slots)] = torch.tensor(rops.rmm(local, sel))
    D.all_reduce_(seed, dist)
    fsel = np.zeros((k, full.r_T))
    fsel[np.arange(k), pick] = 1.0
    out["seed"] = float(np.max(np.abs(seed.numpy() - rops.rmm(full, fsel))))
    assign = rng.integers(0, k, full.r_T)
    oh = np.zeros((local.r_T, k))
    oh[np.arange(local.r_T), assign[plan.rows]] = 1.0
    kb = torch.tensor(np.concatenate([rops.transpose_lmm(local, oh).T.ravel(), oh.sum(0)]))
    D.all_reduce_(kb, dist)
    ohf = np.zeros((full.r_T, k))
    ohf[np.arange(full.r_T), assign] = 1.0
    kw = np.concatenate([rops.transpose_lmm(full, ohf).T.ravel(), ohf.sum(0)])
    out["kmeans"] = float(np.max(np.abs(kb.numpy() - kw)) / np.max(np.abs(kw)))
    # GNMF: [W^T T | W^T W]
    W = rng.random((full.r_T, 3))
    gb = torch.tensor(np.concatenate([rops.rmm(local, W[plan.rows].T).ravel(),
                                      (W[plan.rows].T @ W[plan.rows]).ravel()]))
    D.all_reduce_(gb, dist)
    gw = np.concatenate([rops.rmm(full, W.T).ravel(), (W.T @ W).ravel()])
    out["gnmf"] = float(np.max(np.abs(gb.numpy() - gw)) / np.max(np.abs(gw)))
    results[rank] = out
    dist.destroy_process_group()


def test_sharded_reduce_buffers_equal_single_process():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for rank in range(world):
        r = results[rank]
        assert r["glm"] < 1e-12 and r["kmeans"] < 1e-12 and r["gnmf"] < 1e-12
        assert r["seed"] == 0.0
