"""Multi-GPU execution of the fused trainers: one process per GPU.

The reference is single-process; this is the B200 build's
data-parallel layer.

Partitioning.  Fact rows are split into contiguous ranges of the FK of one
dimension, the *shard source* (normally the largest): rank r owns the
dimension rows [dim_lo, dim_hi) of that source and exactly the fact rows that
reference them, so the shard source is row-sharded (its FKs are rebased to
dim_lo) and every other source is replicated.  Rows without a match in the
shard source (left / outer joins) are split evenly in row order.

Exchange.  Every session (`GlmSession`, `KMeansSession`, `GnmfSession`)
produces per-rank partial sums in one fp64 reduce buffer (GLM: gradient +
loss; K-means: centroid sums, counts, loss; GNMF: W^T T, W^T W).  One
all-reduce of that buffer per iteration, then every rank applies the identical
update -- there is no other collective on the data path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ShardPlan:
    rank: int
    world: int
    rows: np.ndarray        # target rows owned by this rank (ascending)
    dim_lo: int             # shard-source rows [dim_lo, dim_hi)
    dim_hi: int

    @property
    def n_rows(self) -> int:
        return int(self.rows.size)


def plan_shards(fk: np.ndarray, r_dim: int, world: int) -> list[ShardPlan]:
    """Split target rows by contiguous FK ranges of the shard source so every
    rank gets ~r_T / world rows (boundaries fall between dimension rows)."""
    fk = np.asarray(fk, dtype=np.int64)
    if world < 1:
        raise ValueError("world must be >= 1")
    matched = fk >= 0
    counts = np.bincount(fk[matched], minlength=r_dim)
    cum = np.concatenate([[0], np.cumsum(counts)])
    total = int(cum[-1])
    bounds = [0]
    for r in range(1, world):
        bounds.append(int(np.searchsorted(cum, r * total / world, side="left")))
    bounds.append(r_dim)
    bounds = np.maximum.accumulate(np.minimum(bounds, r_dim))
    null_rows = np.nonzero(~matched)[0]
    null_split = np.array_split(null_rows, world)
    plans = []
    for r in range(world):
        lo, hi = int(bounds[r]), int(bounds[r + 1])
        mine = np.nonzero(matched & (fk >= lo) & (fk < hi))[0]
        rows = np.sort(np.concatenate([mine, null_split[r]]))
        plans.append(ShardPlan(r, world, rows, lo, hi))
    return plans


def shard_arrays(sources, ind_sels, plan: ShardPlan, shard_source: int):
    """Rank-local (sources, ind_sels) for `TargetHandle.from_arrays`.

    sources[k]: r_k x c_k arrays; ind_sels[k]: r_T int FK (None = identity,
    the fact table).  The fact rows and every FK are restricted to
    `plan.rows`; the shard source keeps rows [dim_lo, dim_hi) with rebased
    FKs; other dimensions are replicated."""
    out_s, out_i = [], []
    rows = plan.rows
    for k, (src, sel) in enumerate(zip(sources, ind_sels)):
        if sel is None:                     # identity indicator: the fact table
            out_s.append(np.asarray(src)[rows])
            out_i.append(None)
            continue
        sel = np.asarray(sel, dtype=np.int64)[rows]
        if k == shard_source:
            local = np.where(sel >= 0, sel - plan.dim_lo, -1)
            out_s.append(np.asarray(src)[plan.dim_lo:max(plan.dim_hi, plan.dim_lo + 1)])
            out_i.append(local.astype(np.int32))
        else:
            out_s.append(np.asarray(src))
            out_i.append(sel.astype(np.int32))
    return out_s, out_i


def kmeans_seed_rows(r_t: int, k: int, seed: int) -> np.ndarray:
    """Global seed rows of the reference K-means init (trainers.py:209-210)."""
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(r_t, size=k, replace=False)).astype(np.int64)


def local_seed_slots(plan: ShardPlan, pick: np.ndarray):
    """(slots, local_rows): which of the k seed rows this rank owns and their
    positions in the rank-local target.  The seed centroid matrix is the
    all-reduce (sum) of every rank's rows placed at their slots."""
    pos = np.searchsorted(plan.rows, pick)
    pos_c = np.minimum(pos, max(plan.n_rows - 1, 0))
    owned = (pos < plan.n_rows) & (plan.rows[pos_c] == pick) if plan.n_rows else np.zeros(
        pick.size, dtype=bool)
    slots = np.nonzero(owned)[0]
    return slots, pos[slots].astype(np.int64)


def sharded_kmeans_seed(handle, plan: ShardPlan, r_t: int, k: int, seed: int, dist,
                        group=None) -> np.ndarray:
    """The reference's K-means seed centroids (k global rows, trainers.py:
    209-218) on a sharded table: each rank fetches the seed rows it owns on
    the device (exact copies) and an all-reduce assembles the k x c_T matrix."""
    import torch

    from .trainers import target_rows
    pick = kmeans_seed_rows(r_t, k, seed)
    slots, local = local_seed_slots(plan, pick)
    cents = torch.zeros((k, handle.shape[1]), dtype=torch.float64)
    if slots.size:
        cents[torch.as_tensor(slots)] = torch.as_tensor(target_rows(handle, local)).double()
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    cents = cents.to(dev)
    dist.all_reduce(cents, op=dist.ReduceOp.SUM, group=group)
    return cents.cpu().numpy()


def all_reduce_(buf, dist, group=None):
    """Sum a reduce buffer (torch tensor) over ranks in place."""
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


class DeviceBuffer:
    """`__cuda_array_interface__` view of a library-owned fp64 device buffer
    (the session reduce buffer), so torch / NCCL can all-reduce it in place."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                         "data": (ptr, False), "version": 3}


class NcclComm:
    """The library's own NCCL communicator over the ranks of `group`
    (`fl_comm_*`, include/fl_b200.h): rank 0 draws the unique id, the host
    process group broadcasts it, every rank joins.  Attached to a session
    (`session.set_comm`), the per-iteration all-reduce runs inside the
    session's CUDA graphs."""

    def __init__(self, dist, device: int, group=None):
        import ctypes as C

        from . import _lib
        rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        buf = (C.c_uint8 * 128)()
        if rank == 0:
            _lib.call("fl_comm_unique_id", buf, 128)
        obj = [bytes(buf)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        idb = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        self.ptr = C.c_void_p()
        _lib.call("fl_comm_init", idb, 128, int(world), int(rank), int(device),
                  C.byref(self.ptr))
        self.rank, self.world, self.device = rank, world, device

    def all_reduce(self, ptr: int, n: int, stream=None):
        import ctypes as C

        from . import _lib
        _lib.call("fl_comm_allreduce", self.ptr, C.c_void_p(ptr), int(n),
                  stream if stream is not None else C.c_void_p(0))

    def close(self):
        from . import _lib
        if getattr(self, "ptr", None):
            try:
                _lib.load().fl_comm_destroy(self.ptr)
            except Exception:
                pass
            self.ptr = None

    def __del__(self):
        self.close()


def run_sharded(session, iterations: int, dist, device, group=None, comm=None):
    """`iterations` x (partial -> all-reduce -> update) on one rank.  The
    session must expose partial(), update() and reduce_buffer().

    comm: an `NcclComm` -- the session runs its iterations itself, the
    all-reduce captured in its CUDA graphs next to the kernels (no host
    round trip per iteration).  Without it the loop is host-driven and the
    all-reduce goes through torch.distributed (any backend, e.g. gloo)."""
    import torch

    from .trainers import KMeansSession
    if comm is not None:
        session.set_comm(comm)
        session.run(iterations)
        return
    ptr, n = session.reduce_buffer()
    red = torch.as_tensor(DeviceBuffer(ptr, n), device=device)
    if getattr(session, "needs_prime", False):    # GNMF: products of W_0 first
        session.partial()
        all_reduce_(red, dist, group)
    # K-means: the last iteration writes the assignments it made against the
    # centroids of that iteration (reference trainers.py:229-245 returns the
    # final iteration's argmin, not one against the updated centroids)
    assigns = isinstance(session, KMeansSession)
    for it in range(iterations):
        if assigns:
            session.partial(write_assign=(it == iterations - 1))
        else:
            session.partial()
        all_reduce_(red, dist, group)
        session.update()


__all__ = ["DeviceBuffer", "NcclComm", "ShardPlan", "all_reduce_", "kmeans_seed_rows",
           "local_seed_slots", "plan_shards", "run_sharded", "shard_arrays",
           "sharded_kmeans_seed"]
