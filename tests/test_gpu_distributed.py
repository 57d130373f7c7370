"""The sharded (multi-GPU) trainer path on the device: two ranks share the
one GPU of the test box over gloo (CUDA tensors), each owns a shard from
`distributed.plan_shards` and steps partial -> all-reduce -> update through
the C ABI.  Results must match the single-process oracle within the north
star's tolerance (1e-4 relative; K-means assignments identical)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(seed=5, r=24_000, dims=((300, 7), (12, 3)), c_fact=9, clusters=0):
    rng = np.random.default_rng(seed)
    if clusters:
        lab = rng.integers(0, clusters, r)
        fact = rng.random((clusters, c_fact))[lab] + 0.01 * rng.standard_normal((r, c_fact))
    else:
        fact = rng.random((r, c_fact))
    srcs, sels = [fact.astype(np.float32).astype(np.float64)], [None]
    for r_d, c_d in dims:
        if clusters:
            dl = np.arange(r_d) % clusters
            dim = rng.random((clusters, c_d))[dl] + 0.01 * rng.standard_normal((r_d, c_d))
            fk = np.empty(r, dtype=np.int64)
            for j in range(clusters):
                cand = np.nonzero(dl == j)[0]
                mine = np.nonzero(lab == j)[0]
                fk[mine] = cand[rng.integers(0, cand.size, mine.size)]
        else:
            dim = rng.random((r_d, c_d))
            fk = rng.permutation(np.arange(r) % r_d)
        srcs.append(dim.astype(np.float32).astype(np.float64))
        sels.append(fk)
    maps, off = [], 0
    for s_ in srcs:
        maps.append(np.arange(s_.shape[1]) + off)
        off += s_.shape[1]
    return srcs, sels, maps, r, off


def _oracle_table(srcs, sels, maps, r, c):
    import oracle
    ind = [np.arange(r) if s is None else np.asarray(s, dtype=np.int64) for s in sels]
    return oracle.OracleTable(srcs, ind, [m.astype(np.int64) for m in maps], r, c)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import paper_2502_01985_b200 as fl
    from paper_2502_01985_b200 import distributed as D
    from paper_2502_01985_b200.trainers import GlmSession, GnmfSession, KMeansSession
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    res = {}
    # ---- GLM (linear + logistic)
    srcs, sels, maps, r, c = _data()
    plan = D.plan_shards(sels[1], srcs[1].shape[0], world)[rank]
    ls, li = D.shard_arrays(srcs, sels, plan, 1)
    h = fl.TargetHandle.from_arrays(ls, li, maps, plan.n_rows, c)
    rng = np.random.default_rng(2)
    ylin = rng.random(r).astype(np.float32).astype(np.float64)
    ylog = rng.integers(0, 2, r).astype(np.float64)
    for model, y in (("linreg", ylin), ("logreg", ylog)):
        s = GlmSession(h, model, y[plan.rows], 1e-6)
        D.run_sharded(s, 6, dist, dev)
        w, loss = s.result(6)
        res[model] = (w, loss)
        s.close()
    # ---- K-means (planted clusters)
    srcs, sels, maps, r, c = _data(seed=9, clusters=6)
    plan = D.plan_shards(sels[1], srcs[1].shape[0], world)[rank]
    ls, li = D.shard_arrays(srcs, sels, plan, 1)
    h = fl.TargetHandle.from_arrays(ls, li, maps, plan.n_rows, c)
    cents0 = D.sharded_kmeans_seed(h, plan, r, 6, 4, dist)
    s = KMeansSession(h, 6, cents0)
    D.run_sharded(s, 5, dist, dev)   # the last iteration writes its assignments
    cents, assign, loss = s.result(5)
    res["kmeans"] = (cents0, plan.rows, assign, cents, loss)
    s.close()
    # ---- GNMF
    srcs, sels, maps, r, c = _data(seed=11)
    plan = D.plan_shards(sels[1], srcs[1].shape[0], world)[rank]
    ls, li = D.shard_arrays(srcs, sels, plan, 1)
    h = fl.TargetHandle.from_arrays(ls, li, maps, plan.n_rows, c)
    rg = np.random.default_rng(3)
    w0 = rg.random((r, 4)) * 0.3
    h0 = rg.random((4, c)) * 0.3
    tab = _oracle_table(srcs, sels, maps, r, c)
    import oracle
    t_sq = float(oracle.row_sum(oracle.elementwise(tab, "square")).sum())
    s = GnmfSession(h, 4, w0[plan.rows], h0, t_sq)
    D.run_sharded(s, 5, dist, dev)
    W, H, loss = s.result(5)
    res["gnmf"] = (plan.rows, W, H, loss)
    s.close()
    out[rank] = res
    dist.destroy_process_group()


def test_sharded_trainers_match_oracle():
    import torch.multiprocessing as mp
    from oracle import reference_ops as rops
    from oracle import reference_trainers as rt
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    # GLM vs oracle
    srcs, sels, maps, r, c = _data()
    tab = _oracle_table(srcs, sels, maps, r, c)
    rng = np.random.default_rng(2)
    ylin = rng.random(r).astype(np.float32).astype(np.float64)
    ylog = rng.integers(0, 2, r).astype(np.float64)
    for model, y in (("linreg", ylin), ("logreg", ylog)):
        want = rt.train(model, tab, iterations=6, learning_rate=1e-6, y=y)
        for rank in range(world):
            w, loss = out[rank][model]
            ww = want["parameters"]["w"].ravel()
            assert np.max(np.abs(w - ww)) / np.max(np.abs(ww)) < TOL
            wl = np.asarray(want["loss_history"])
            assert np.max(np.abs(loss - wl) / np.abs(wl)) < TOL
    # K-means: seeds identical to the reference's; assignments identical
    srcs, sels, maps, r, c = _data(seed=9, clusters=6)
    tab = _oracle_table(srcs, sels, maps, r, c)
    want = rt.kmeans(tab, 5, 6, 4)
    pick = np.sort(np.random.default_rng(4).choice(r, size=6, replace=False))
    sel = np.zeros((6, r))
    sel[np.arange(6), pick] = 1.0
    for rank in range(world):
        cents0, rows, assign, cents, loss = out[rank]["kmeans"]
        assert np.array_equal(cents0, rops.rmm(tab, sel))
        cw = want["parameters"]["centroids"]
        assert np.max(np.abs(cents - cw)) / np.max(np.abs(cw)) < TOL
        wl = np.asarray(want["loss_history"])
        assert np.max(np.abs(np.asarray(loss) - wl) / np.abs(wl)) < TOL
    got = np.full(r, -1, dtype=np.int64)
    for rank in range(world):
        _, rows, assign, _, _ = out[rank]["kmeans"]
        got[rows] = assign
    # the final iteration's assignments, as the reference returns them
    assert np.array_equal(got, want["parameters"]["assignments"])
    # GNMF vs oracle with the same initial W, H
    srcs, sels, maps, r, c = _data(seed=11)
    tab = _oracle_table(srcs, sels, maps, r, c)
    rg = np.random.default_rng(3)
    w = rg.random((r, 4)) * 0.3
    hh = rg.random((4, c)) * 0.3
    t_sq = float(rops.row_sum(rops.elementwise(tab, "square")).sum())
    losses = []
    for it in range(5):
        p = rops.rmm(tab, w.T)
        if it > 0:
            losses.append(t_sq - 2 * float((p * hh).sum()) + float((w.T @ w * (hh @ hh.T)).sum()))
        hh = hh * p / (w.T @ w @ hh + 1e-12)
        q = rops.lmm(tab, hh.T)
        w = w * q / (w @ (hh @ hh.T) + 1e-12)
    p = rops.rmm(tab, w.T)
    losses.append(t_sq - 2 * float((p * hh).sum()) + float((w.T @ w * (hh @ hh.T)).sum()))
    for rank in range(world):
        rows, W, H, loss = out[rank]["gnmf"]
        assert np.max(np.abs(W - w[rows])) / np.max(np.abs(w)) < TOL
        assert np.max(np.abs(H - hh)) / np.max(np.abs(hh)) < TOL
        assert np.max(np.abs(np.asarray(loss) - losses) / np.abs(losses)) < TOL
