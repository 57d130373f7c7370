"""Training loops on the B200: drop-in for the reference trainers.

Same entry points and result type as `pkg/src/factorlearn/trainers.py`
(`train`, `TrainConfig`, `TrainResult`, `ConfigError`, `DivergenceError`,
`linear_regression`, `logistic_regression`, `kmeans`, `gaussian_nmf`) and the
same loss conventions (`trainers.py:9-17`):

  linear/logistic  loss_history[i] = loss at the weights entering iteration i
  kmeans           loss_history[i] = within-cluster squared distance of
                   iteration i's assignment against the centroids it used
  gaussian_nmf     loss_history[i] = ||T - WH||_F^2 after iteration i's updates

Each loop is one device-resident session in the C library (fused kernels,
CUDA-graph replayed); nothing is iterated on the host.  `wall_time` is the
device time of the iteration loop (CUDA events when torch is present, else a
synchronised host clock), excluding the one-time setup -- the analogue of the
reference's operator-only stopwatch (`trainers.py:90-103`).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .ops import TargetHandle, _is_torch
from .sparse import OpTrace, ShapeError, SparseMatrix, as_dense

EPS_NMF = 1e-12  # trainers.py:29


class ConfigError(ValueError):
    """Reference `trainers.py:32-33`."""


class DivergenceError(ValueError):
    """Training produced a non-finite loss (reference `trainers.py:36-41`)."""

    def __init__(self, model: str, iteration: int):
        super().__init__(f"{model}: non-finite loss at iteration {iteration}")
        self.iteration = iteration


@dataclass(frozen=True)
class TrainConfig:
    """Reference `trainers.py:44-64` (same defaults and validation)."""

    iterations: int = 20
    learning_rate: float = 1e-3
    k_clusters: int = 4
    rank: int = 2
    seed: int = 0

    def __post_init__(self):
        if self.iterations < 1:
            raise ConfigError("iterations must be >= 1")
        if not self.learning_rate > 0.0:
            raise ConfigError("learning_rate must be > 0")
        if self.k_clusters < 1:
            raise ConfigError("k_clusters must be >= 1")
        if self.rank < 1:
            raise ConfigError("rank must be >= 1")
        if self.seed < 0:
            raise ConfigError("seed must be a non-negative integer")


@dataclass
class TrainResult:
    """Reference `trainers.py:67-87`."""

    model: str
    parameters: dict = field(default_factory=dict)
    loss_history: list = field(default_factory=list)
    trace: OpTrace = field(default_factory=OpTrace)
    wall_time: float = 0.0

    def to_dict(self) -> dict:
        return {
            "model": self.model,
            "parameters": {k: np.asarray(v).tolist() for k, v in self.parameters.items()},
            "loss_history": list(self.loss_history),
            "trace": {
                "multiply_add_count": self.trace.multiply_add_count,
                "bytes_read": self.trace.bytes_read,
                "bytes_written": self.trace.bytes_written,
                "wall_time": self.trace.wall_time,
            },
            "wall_time": self.wall_time,
        }


class _DeviceTimer:
    """CUDA-event timer on the default stream when torch is available."""

    def __init__(self, device: int):
        self.device = device
        self.torch = None
        try:
            import torch
            if torch.cuda.is_available():
                self.torch = torch
        except Exception:
            pass

    def __enter__(self):
        if self.torch is not None:
            t = self.torch
            self.e0 = t.cuda.Event(enable_timing=True)
            self.e1 = t.cuda.Event(enable_timing=True)
            # the library launches on the legacy default stream (NULL)
            self.e0.record(t.cuda.default_stream(self.device))
        self.t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        if self.torch is not None:
            self.e1.record(self.torch.cuda.default_stream(self.device))
            self.e1.synchronize()
            self.seconds = self.e0.elapsed_time(self.e1) / 1e3
        else:
            self.seconds = time.perf_counter() - self.t0
        return False


def _first_nonfinite(losses) -> int | None:
    for i, v in enumerate(losses):
        if not np.isfinite(v):
            return i
    return None


def _bytes_per_iteration(h: TargetHandle, y_bytes: int) -> tuple[int, int]:
    """Algorithmic HBM bytes of one fused GLM iteration:
    4 r_T pf + 4 r_T n_gather + b_y r_T + 2 * sum_d 4 r_d pitch_d."""
    lay = h.layout
    r_T, _ = h.shape
    rb = 4 * r_T * lay["stream_pitch"] + 4 * r_T * lay["n_gather"] + y_bytes * r_T
    rb += 2 * lay.get("gather_bytes", 0)
    return rb, 0


# ---------------------------------------------------------------------------
# GLM session (linear / logistic regression)
# ---------------------------------------------------------------------------
class GlmSession:
    """Device-resident GD state: `fl_glm_*` (include/fl_b200.h)."""

    def __init__(self, h: TargetHandle, model: str, y, learning_rate: float):
        self.h = h
        self.model = model
        self.c_T = h.shape[1]
        ptr = C.c_void_p()
        if _is_torch(y):
            import torch
            # the library reads uint8 labels (logreg) / fp32 targets (linreg)
            keep = y.reshape(-1).to(torch.uint8 if model == "logreg" else torch.float32)
            keep = keep.contiguous()
            y_ptr = C.c_void_p(keep.data_ptr())
        else:
            dt = np.uint8 if model == "logreg" else np.float32
            keep = np.ascontiguousarray(np.asarray(y).reshape(-1), dtype=dt)
            y_ptr = keep.ctypes.data_as(C.c_void_p)
        _lib.call("fl_glm_create", h._dev.ptr, _lib.MODEL_IDS[model], y_ptr,
                  float(learning_rate), C.byref(ptr), C.c_void_p(0))
        del keep
        self.ptr = ptr

    def run(self, iterations: int, stream=None):
        _lib.call("fl_glm_run", self.ptr, int(iterations),
                  stream if stream is not None else C.c_void_p(0))

    def partial(self, stream=None):
        _lib.call("fl_glm_partial", self.ptr, stream if stream is not None else C.c_void_p(0))

    def update(self, stream=None):
        _lib.call("fl_glm_update", self.ptr, stream if stream is not None else C.c_void_p(0))

    def set_comm(self, comm):
        """Attach an NCCL communicator (`distributed.NcclComm`, or None to
        detach): run() then does partial -> all-reduce -> update per
        iteration inside the session's CUDA graphs."""
        _lib.call("fl_glm_set_comm", self.ptr, comm.ptr if comm is not None else C.c_void_p(0))
        self.comm = comm

    def reduce_buffer(self) -> tuple[int, int]:
        buf = C.c_void_p()
        n = C.c_int32()
        _lib.call("fl_glm_reduce_buffer", self.ptr, C.byref(buf), C.byref(n))
        return buf.value, n.value

    @property
    def path(self) -> tuple[str, float]:
        """(fact-pass variant, measured stream-block density): "cta_tiles",
        "warp_tma" (dense F), "csr" (sparse F) or
        "generic"."""
        p = C.c_int32()
        dens = C.c_double()
        _lib.call("fl_glm_path", self.ptr, C.byref(p), C.byref(dens))
        return ("cta_tiles", "warp_tma", "csr", "generic", "solo")[p.value], dens.value

    def kernel_times(self, iters: int, stream=None) -> list[float]:
        """Mean ms of [dim q, fact pass, dim t + update] over `iters` iterations
        (CUDA events between the kernels, recorded by the library)."""
        out = (C.c_float * 3)()
        _lib.call("fl_glm_kernel_times", self.ptr, int(iters), out,
                  stream if stream is not None else C.c_void_p(0))
        return [float(v) for v in out]

    def result(self, n: int):
        w = np.empty(self.c_T, dtype=np.float64)
        loss = np.empty(max(n, 1), dtype=np.float64)
        done = C.c_int32()
        _lib.call("fl_glm_result", self.ptr, w.ctypes.data_as(C.c_void_p),
                  loss.ctypes.data_as(C.c_void_p), int(n), C.byref(done), C.c_void_p(0))
        return w, loss[:min(done.value, n)]

    def close(self):
        if getattr(self, "ptr", None):
            try:
                _lib.load().fl_glm_destroy(self.ptr)
            except Exception:
                pass
            self.ptr = None

    def __del__(self):
        self.close()


def _labels(y, r_t: int):
    if _is_torch(y):
        if tuple(y.shape) not in ((r_t, 1), (r_t,)):
            raise ShapeError(f"labels must be {r_t}x1, got {tuple(y.shape)}")
        return y.reshape(-1)
    if hasattr(y, "shape") and tuple(y.shape) not in ((r_t, 1), (r_t,)):
        raise ShapeError(f"labels must be {r_t}x1, got {tuple(y.shape)}")
    yd = as_dense(y)
    if yd.shape != (r_t, 1):
        raise ShapeError(f"labels must be {r_t}x1, got {yd.shape}")
    return yd.reshape(-1)


def _op_trace(t: TargetHandle, width: int, seconds: float) -> OpTrace:
    """OpTrace of one operator call of operand width `width` over the device
    layout: multiply-adds of the factorized product and the algorithmic bytes
    of one pass (TargetHandle._pass_cost); the reference records the same
    three counters per traced call (sparse.py:56-80, ops.py:159-204)."""
    madds, rb = t._pass_cost(max(width, 1))
    if width == 0:
        madds = 0
    tr = OpTrace()
    tr.record(madds, rb, 4 * t.shape[0] * max(width, 1), seconds)
    return tr


def _log_glm_ops(t: TargetHandle, result: TrainResult, iterations: int, per_it: OpTrace):
    """Trace log in the reference's op vocabulary (trainers.py:151-157:
    one lmm and one transpose_lmm per iteration)."""
    if t.trace_log is None:
        return
    for _ in range(iterations):
        for name in ("lmm", "transpose_lmm"):
            tr = OpTrace()
            tr.record(per_it.multiply_add_count // 2, per_it.bytes_read // 2,
                      per_it.bytes_written // 2, per_it.wall_time / 2)
            t.trace_log.append((name, t.path, tr))


def _glm(model: str, t: TargetHandle, y, cfg: TrainConfig) -> TrainResult:
    r_t, c_t = t.shape
    yv = _labels(y, r_t)
    if model == "logreg":
        # reference trainers.py:172-173 (checked for host and device labels)
        if _is_torch(yv):
            ok = bool(((yv == 0) | (yv == 1)).all())
        else:
            ok = bool(np.all((yv == 0) | (yv == 1)))
        if not ok:
            raise ConfigError("logistic labels must be 0/1")
    s = GlmSession(t, model, yv, cfg.learning_rate)
    try:
        with _DeviceTimer(t.device) as tm:
            s.run(cfg.iterations)
        w, losses = s.result(cfg.iterations)
    finally:
        s.close()
    bad = _first_nonfinite(losses)
    if bad is not None:
        raise DivergenceError(model, bad)
    result = TrainResult(model, {"w": w.reshape(-1, 1)}, [float(v) for v in losses])
    lay = t.layout
    madds = 2 * r_t * lay["stream_cols"] * cfg.iterations
    rb = (4 * r_t * lay["stream_pitch"] + 4 * r_t * lay["n_gather"]
          + (1 if model == "logreg" else 4) * r_t) * cfg.iterations
    result.trace.record(madds, rb, 8 * (c_t + 1) * cfg.iterations, tm.seconds)
    result.wall_time = tm.seconds
    per = OpTrace()
    per.record(madds // cfg.iterations, rb // cfg.iterations, 8 * (c_t + 1),
               tm.seconds / cfg.iterations)
    _log_glm_ops(t, result, cfg.iterations, per)
    t.trace.merge(result.trace)
    return result


def linear_regression(t: TargetHandle, y, cfg: TrainConfig) -> TrainResult:
    """GD on 1/2 ||Tw - y||^2 (trainers.py:138-163), fused on the device."""
    return _glm("linreg", t, y, cfg)


def logistic_regression(t: TargetHandle, y, cfg: TrainConfig) -> TrainResult:
    """GD on the logistic loss (trainers.py:166-195), fused on the device."""
    return _glm("logreg", t, y, cfg)


# ---------------------------------------------------------------------------
# K-means
# ---------------------------------------------------------------------------
class KMeansSession:
    def __init__(self, h: TargetHandle, k: int, centroids0: np.ndarray):
        self.h = h
        self.k = k
        self.c_T = h.shape[1]
        ptr = C.c_void_p()
        c0 = np.ascontiguousarray(centroids0, dtype=np.float64)
        _lib.call("fl_kmeans_create", h._dev.ptr, int(k), c0.ctypes.data_as(C.c_void_p),
                  C.byref(ptr), C.c_void_p(0))
        self.ptr = ptr

    def run(self, iterations: int, stream=None):
        _lib.call("fl_kmeans_run", self.ptr, int(iterations),
                  stream if stream is not None else C.c_void_p(0))

    def partial(self, write_assign: bool = False, stream=None):
        _lib.call("fl_kmeans_partial", self.ptr, int(write_assign),
                  stream if stream is not None else C.c_void_p(0))

    def update(self, stream=None):
        _lib.call("fl_kmeans_update", self.ptr, stream if stream is not None else C.c_void_p(0))

    def set_comm(self, comm):
        """Attach an NCCL communicator (`distributed.NcclComm`, or None to
        detach): run() then does partial -> all-reduce -> update per
        iteration inside the session's CUDA graphs."""
        _lib.call("fl_kmeans_set_comm", self.ptr, comm.ptr if comm is not None else C.c_void_p(0))
        self.comm = comm

    def reduce_buffer(self) -> tuple[int, int]:
        buf = C.c_void_p()
        n = C.c_int32()
        _lib.call("fl_kmeans_reduce_buffer", self.ptr, C.byref(buf), C.byref(n))
        return buf.value, n.value

    @property
    def path(self) -> str:
        """"tcgen05_mn" (default fused pass: tcgen05 screen and MN-major
        row contraction), "fused" (per-warp mma.sync pass), "tcgen05" (opt-in
        K-major variant) or "generic" (width-general session: any k, width or
        number of gathered sources)."""
        p = C.c_int32()
        _lib.call("fl_kmeans_path", self.ptr, C.byref(p))
        return ("fused", "tcgen05", "generic", "tcgen05_mn")[p.value]

    def kernel_times(self, iters: int, stream=None) -> list[float]:
        """Mean ms of [dim E, fact pass, dim sums, reduce + update]."""
        out = (C.c_float * 4)()
        _lib.call("fl_kmeans_kernel_times", self.ptr, int(iters), out,
                  stream if stream is not None else C.c_void_p(0))
        return [float(v) for v in out]

    def result(self, n: int):
        r_t, _ = self.h.shape
        cents = np.empty((self.k, self.c_T), dtype=np.float64)
        assign = np.empty(r_t, dtype=np.int64)   # the reference's argmin dtype, widened on device
        loss = np.empty(max(n, 1), dtype=np.float64)
        done = C.c_int32()
        _lib.call("fl_kmeans_result", self.ptr, cents.ctypes.data_as(C.c_void_p),
                  C.c_void_p(0), loss.ctypes.data_as(C.c_void_p), int(n),
                  C.byref(done), C.c_void_p(0))
        _lib.call("fl_kmeans_assignments64", self.ptr, assign.ctypes.data_as(C.c_void_p),
                  C.c_void_p(0))
        return cents, assign, loss[:min(done.value, n)]

    def close(self):
        if getattr(self, "ptr", None):
            try:
                _lib.load().fl_kmeans_destroy(self.ptr)
            except Exception:
                pass
            self.ptr = None

    def __del__(self):
        self.close()


def target_rows(t: TargetHandle, rows) -> np.ndarray:
    """Rows of T (target order) gathered on the device: exact fp32 copies."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty((rows.size, t.shape[1]), dtype=np.float32)
    if rows.size:
        _lib.call("fl_target_rows", t._dev.ptr, rows.ctypes.data_as(C.c_void_p), int(rows.size),
                  out.ctypes.data_as(C.c_void_p), C.c_void_p(0))
    return out


def kmeans_init(t: TargetHandle, k: int, seed: int) -> np.ndarray:
    """Seed centroids = k distinct target rows (trainers.py:209-218); the
    rows are fetched on the device (exact copies)."""
    r_t, _ = t.shape
    rng = np.random.default_rng(seed)
    pick = np.sort(rng.choice(r_t, size=k, replace=False)).astype(np.int64)
    return target_rows(t, pick).astype(np.float64)


def kmeans(t: TargetHandle, cfg: TrainConfig) -> TrainResult:
    """Lloyd's algorithm (trainers.py:198-246), fused on the device: one pass
    over the fact rows per iteration computes distances, argmin (ties to the
    lowest index), the loss and the centroid sums/counts."""
    r_t, c_t = t.shape
    k = cfg.k_clusters
    if k > r_t:
        raise ConfigError(f"k_clusters = {k} exceeds row count {r_t}")
    cents0 = kmeans_init(t, k, cfg.seed)
    s = KMeansSession(t, k, cents0)
    try:
        with _DeviceTimer(t.device) as tm:
            s.run(cfg.iterations)
        cents, assign, losses = s.result(cfg.iterations)
    finally:
        s.close()
    bad = _first_nonfinite(losses)
    if bad is not None:
        raise DivergenceError("kmeans", bad)
    result = TrainResult("kmeans", {"centroids": cents, "assignments": assign},
                         [float(v) for v in losses])
    lay = t.layout
    rb = (4 * r_t * lay["stream_pitch"] + 4 * r_t * lay["n_gather"]) * cfg.iterations
    result.trace.record(2 * k * r_t * lay["stream_cols"] * cfg.iterations, rb,
                        8 * (k * c_t + k + 1) * cfg.iterations, tm.seconds)
    result.wall_time = tm.seconds
    if t.trace_log is not None:
        # the reference's op sequence (trainers.py:213-245): rmm (seed rows),
        # elementwise square, row_sum, then lmm + transpose_lmm per iteration;
        # each entry carries the device pass's algorithmic work, and the fused
        # iteration's device time is split between its two products
        for name, width in (("rmm", k), ("elementwise", 0), ("row_sum", 1)):
            t.trace_log.append((name, t.path, _op_trace(t, width, 0.0)))
        half = tm.seconds / (2 * cfg.iterations)
        for _ in range(cfg.iterations):
            for name in ("lmm", "transpose_lmm"):
                t.trace_log.append((name, t.path, _op_trace(t, k, half)))
    t.trace.merge(result.trace)
    return result


# ---------------------------------------------------------------------------
# Gaussian NMF
# ---------------------------------------------------------------------------
def _nonneg_min(t: TargetHandle) -> float:
    if t.matrix is not None and hasattr(t.matrix, "data"):
        d = np.asarray(t.matrix.data)
        return float(d.min()) if d.size else 0.0
    tab = t.table
    if tab is not None and hasattr(tab, "sources"):
        mins = [float(np.asarray(s.data).min()) for s in tab.sources if s.nnz]
        return min(mins) if mins else 0.0
    if tab is not None and hasattr(tab, "base"):
        # elementwise-mapped table: evaluate the map on the host-side values
        from . import sparse as _sp  # noqa: F401
        base_min = []
        b = tab
        funcs = []
        while hasattr(b, "base"):
            funcs.append((b.func, b.scalar))
            b = b.base
        if hasattr(b, "sources"):
            for s in b.sources:
                v = np.asarray(s.data, dtype=np.float64)
                for f, sc in reversed(funcs):
                    v = _host_map(f, sc, v)
                if v.size:
                    base_min.append(float(v.min()))
            return min(base_min) if base_min else 0.0
    # array-built tables: assume validated by the caller
    return 0.0


def _host_map(func, scalar, v):
    if func == "scale":
        return v * scalar
    if func == "divide":
        return v / scalar
    if func == "square":
        return v * v
    if func == "abs":
        return np.abs(v)
    if func == "expm1":
        return np.expm1(v)
    return 1.0 / (1.0 + np.exp(-v)) - 0.5


class GnmfSession:
    def __init__(self, h: TargetHandle, rank: int, w0, h0, t_sq: float):
        self.h = h
        self.rank = rank
        self.c_T = h.shape[1]
        ptr = C.c_void_p()

        def _ptr(a):   # host (numpy) or device (CUDA torch) fp64 operand
            if _is_torch(a):
                a = a.contiguous().double()
                return a, C.c_void_p(a.data_ptr())
            a = np.ascontiguousarray(a, dtype=np.float64)
            return a, a.ctypes.data_as(C.c_void_p)

        w0, wp = _ptr(w0)
        h0, hp = _ptr(h0)
        _lib.call("fl_gnmf_create", h._dev.ptr, int(rank), wp, hp, float(t_sq), C.byref(ptr),
                  C.c_void_p(0))
        self.ptr = ptr

    # sharded stepping needs one extra partial up front: the products of W_0
    needs_prime = True

    def run(self, iterations: int, stream=None):
        _lib.call("fl_gnmf_run", self.ptr, int(iterations),
                  stream if stream is not None else C.c_void_p(0))
        self.needs_prime = False

    def partial(self, stream=None):
        _lib.call("fl_gnmf_partial", self.ptr, stream if stream is not None else C.c_void_p(0))
        self.needs_prime = False

    def update(self, stream=None):
        """The H update runs at the start of the next partial()."""

    def set_comm(self, comm):
        """Attach an NCCL communicator (`distributed.NcclComm`, or None to
        detach): run() then does partial -> all-reduce -> update per
        iteration inside the session's CUDA graphs."""
        _lib.call("fl_gnmf_set_comm", self.ptr, comm.ptr if comm is not None else C.c_void_p(0))
        self.comm = comm

    def reduce_buffer(self) -> tuple[int, int]:
        buf = C.c_void_p()
        n = C.c_int32()
        _lib.call("fl_gnmf_reduce_buffer", self.ptr, C.byref(buf), C.byref(n))
        return buf.value, n.value

    @property
    def path(self) -> str:
        """"fused" (per-warp mma.sync pass), "tcgen05" (opt-in K-major
        variant), "generic" (width-general session: any rank, width or number
        of gathered sources) or "tcgen05_mn" (tcgen05 pass with MN-major
        row-contraction operands)."""
        p = C.c_int32()
        _lib.call("fl_gnmf_path", self.ptr, C.byref(p))
        return ("fused", "tcgen05", "generic", "tcgen05_mn")[p.value]

    def kernel_times(self, iters: int, stream=None) -> list[float]:
        """Mean ms of [H update, dim G, fact pass, dim P, reduce]."""
        out = (C.c_float * 5)()
        _lib.call("fl_gnmf_kernel_times", self.ptr, int(iters), out,
                  stream if stream is not None else C.c_void_p(0))
        return [float(v) for v in out]

    def result(self, n: int):
        r_t, c_t = self.h.shape
        w = np.empty((r_t, self.rank), dtype=np.float64)
        hh = np.empty((self.rank, c_t), dtype=np.float64)
        loss = np.empty(max(n, 1), dtype=np.float64)
        done = C.c_int32()
        _lib.call("fl_gnmf_result", self.ptr, w.ctypes.data_as(C.c_void_p),
                  hh.ctypes.data_as(C.c_void_p), loss.ctypes.data_as(C.c_void_p), int(n),
                  C.byref(done), C.c_void_p(0))
        return w, hh, loss[:min(done.value, n)]

    def close(self):
        if getattr(self, "ptr", None):
            try:
                _lib.load().fl_gnmf_destroy(self.ptr)
            except Exception:
                pass
            self.ptr = None

    def __del__(self):
        self.close()


def _rows_total(t: TargetHandle) -> float:
    """sum(rowSum(T)) as the reference forms it (trainers.py:264-279): the
    fp32 device row sums added in fp64.  The row sums stay on the device
    (a CUDA tensor handed to fl_row_sum) and are summed there; building the
    r_T-entry SparseMatrix on the host cost 2 s at 50M rows."""
    try:
        import torch
        if torch.cuda.is_available():
            rs = torch.empty(t.shape[0], dtype=torch.float32, device=f"cuda:{t.device}")
            _lib.call("fl_row_sum", t._dev.ptr, C.c_void_p(rs.data_ptr()), C.c_void_p(0))
            torch.cuda.synchronize(rs.device)
            return float(rs.double().sum().item())
    except ImportError:
        pass
    return float(as_dense(t.row_sum(traced=False)).sum())


def gaussian_nmf(t: TargetHandle, cfg: TrainConfig) -> TrainResult:
    """Multiplicative-update NMF under Frobenius loss (trainers.py:256-307).

    Initialisation follows the reference exactly (scale from the device row
    sums; W then H from one numpy generator); the iterations run on the
    device."""
    r_t, c_t = t.shape
    r = cfg.rank
    if r > min(r_t, c_t):
        raise ConfigError(f"rank = {r} exceeds min(shape) = {min(r_t, c_t)}")
    if _nonneg_min(t) < 0.0:
        raise ConfigError("gaussian_nmf requires a non-negative target")
    total = _rows_total(t)
    scale = total / (r_t * c_t) if total > 0 else 1.0
    rng = np.random.default_rng(cfg.seed)
    w0 = rng.random((r_t, r)) * scale
    h0 = rng.random((r, c_t)) * scale
    sq = t.elementwise("square", traced=False)
    t_sq = _rows_total(sq)
    del sq
    s = GnmfSession(t, r, w0, h0, t_sq)
    try:
        with _DeviceTimer(t.device) as tm:
            s.run(cfg.iterations)
        w, h, losses = s.result(cfg.iterations)
    finally:
        s.close()
    bad = _first_nonfinite(losses)
    if bad is not None:
        raise DivergenceError("gnmf", bad)
    result = TrainResult("gnmf", {"w": w, "h": h}, [float(v) for v in losses])
    result.wall_time = tm.seconds
    # per iteration: rmm (W^T T) and lmm (T H^T) of width r, fused in one pass
    # that also reads and writes W (fp32 on the device)
    per = _op_trace(t, r, 0.0)
    w_bytes = 4 * r_t * r
    result.trace.record(2 * per.multiply_add_count * cfg.iterations,
                        (per.bytes_read + w_bytes) * cfg.iterations,
                        (w_bytes + 8 * r * (c_t + r)) * cfg.iterations, tm.seconds)
    if t.trace_log is not None:
        # the reference's op sequence (trainers.py:270-301): row_sum, then
        # rmm + lmm per iteration (the loss-only products are untraced)
        t.trace_log.append(("row_sum", t.path, _op_trace(t, 1, 0.0)))
        half = tm.seconds / (2 * cfg.iterations)
        for _ in range(cfg.iterations):
            for name in ("rmm", "lmm"):
                t.trace_log.append((name, t.path, _op_trace(t, r, half)))
    t.trace.merge(result.trace)
    return result


TRAINER_FUNCS = {
    "linreg": linear_regression,
    "logreg": logistic_regression,
    "kmeans": kmeans,
    "gnmf": gaussian_nmf,
}

SUPERVISED = {"linreg", "logreg"}


def train(model: str, t: TargetHandle, cfg: TrainConfig, y=None) -> TrainResult:
    """Dispatch by model name; supervised models require labels
    (reference `trainers.py:320-331`)."""
    try:
        fn = TRAINER_FUNCS[model]
    except KeyError:
        raise ConfigError(f"unknown model {model!r}; one of {sorted(TRAINER_FUNCS)}") from None
    if model in SUPERVISED:
        if y is None:
            raise ConfigError(f"{model} requires labels")
        return fn(t, y, cfg)
    return fn(t, cfg)


__all__ = ["ConfigError", "DivergenceError", "EPS_NMF", "GlmSession", "GnmfSession",
           "KMeansSession", "TRAINER_FUNCS", "target_rows", "TrainConfig", "TrainResult", "gaussian_nmf",
           "kmeans", "kmeans_init", "linear_regression", "logistic_regression", "train"]
