"""The library's own NCCL path (csrc/comm.cu, `distributed.NcclComm`) on the
one GPU of the test box: a 1-rank NCCL communicator attached to each session
makes run() execute partial -> ncclAllReduce -> update per iteration inside
the session's CUDA graphs.  NCCL code really executes (the all-reduce of one
rank is NCCL's copy), so the captured multi-GPU iteration is exercised before
an 8-GPU node exists.  With one rank the result must be BIT-IDENTICAL to the
unsharded fused run, and match the oracle within the north-star tolerance."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch
    import torch.distributed as dist
    import paper_2502_01985_b200 as fl
    from paper_2502_01985_b200 import distributed as D
    from paper_2502_01985_b200.trainers import (GlmSession, GnmfSession, KMeansSession,
                                                kmeans_init)
    from conftest import star_table
    from test_gpu_trainers import planted_star
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", 0))
    comm = D.NcclComm(dist, 0)
    res = {}
    ft = star_table(61, 50_000, [(700, 13), (40, 3)], 12)
    h = fl.TargetHandle.factorized(ft)
    rng = np.random.default_rng(1)
    y = rng.integers(0, 2, ft.r_T).astype(np.float64)
    for it in (3, 19):   # one graph of 8 plus a remainder
        pair = []
        for use in (False, True):
            s = GlmSession(h, "logreg", y, 1e-4)
            if use:
                D.run_sharded(s, it, dist, torch.device("cuda", 0), comm=comm)
            else:
                s.run(it)
            pair.append(s.result(it))
            s.close()
        res[f"logreg{it}"] = pair
    for k, kft in ((6, planted_star(3, 40_000, [(300, 9)], 10, 6)),
                   (40, planted_star(4, 30_000, [(900, 7)], 8, 40))):   # fused / generic
        hk = fl.TargetHandle.factorized(kft)
        c0 = kmeans_init(hk, k, 2)
        pair = []
        for use in (False, True):
            s = KMeansSession(hk, k, c0)
            path = s.path
            if use:
                D.run_sharded(s, 7, dist, torch.device("cuda", 0), comm=comm)
            else:
                s.run(7)
            pair.append(s.result(7) + (path,))
            s.close()
        res[f"kmeans{k}"] = pair
    ft_w = star_table(63, 30_000, [(500, 40)], 10)   # c_T = 50: room for rank 40
    for rank_, gft in ((5, ft), (40, ft_w)):   # fused / generic
        hg = fl.TargetHandle.factorized(gft)
        g = np.random.default_rng(7)
        w0 = g.random((gft.r_T, rank_)) * 0.2
        h0 = g.random((rank_, gft.c_T)) * 0.2
        t_sq = float((hg.materialize_dense().astype(np.float64) ** 2).sum())
        pair = []
        for use in (False, True):
            s = GnmfSession(hg, rank_, w0, h0, t_sq)
            path = s.path
            if use:
                D.run_sharded(s, 6, dist, torch.device("cuda", 0), comm=comm)
            else:
                s.run(6)
            pair.append(s.result(6) + (path,))
            s.close()
        res[f"gnmf{rank_}"] = pair
    comm.close()
    out[rank] = res
    dist.destroy_process_group()


def test_nccl_captured_iterations_bit_identical():
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(1, _free_port(), out), nprocs=1, join=True)
    res = out[0]
    for key in ("logreg3", "logreg19"):
        (w0, l0), (w1, l1) = res[key]
        assert np.array_equal(w0, w1) and np.array_equal(l0, l1), key
        assert len(l1) == int(key[6:])
    for k in (6, 40):
        (c0, a0, l0, p0), (c1, a1, l1, p1) = res[f"kmeans{k}"]
        assert p0 == p1 and (p0 == "generic") == (k == 40)
        assert np.array_equal(c0, c1) and np.array_equal(a0, a1) and np.array_equal(l0, l1)
        assert len(l1) == 7
    for r in (5, 40):
        (w0, h0, l0, p0), (w1, h1, l1, p1) = res[f"gnmf{r}"]
        assert p0 == p1 and (p0 == "generic") == (r == 40)
        assert np.array_equal(w0, w1) and np.array_equal(h0, h1) and np.array_equal(l0, l1)
        assert len(l1) == 6
