"""Drop-in operator surface: `TargetHandle` on the B200.

Mirrors the reference class `TargetHandle` (`pkg/src/factorlearn/ops.py:147-328`):
same constructors (`factorized`, `materialized`), same methods (`lmm`, `rmm`,
`transpose_lmm`, `elementwise`, `row_sum`, `col_sum`, `materialize_target`),
same attributes (`path`, `shape`, `trace`, `trace_log`, `table`, `matrix`,
`threads`, `selectors`) and the same error classes.  Every operator runs on the
GPU through the C ABI (`include/fl_b200.h`); the host only converts operands
between the CSR boundary type and dense fp32 buffers.

Operands may be a `SparseMatrix` (this package's or the reference's -- duck
typed), a numpy array, or a CUDA `torch.Tensor` (device-resident path: the
result is returned as a CUDA tensor and nothing crosses PCIe).
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import time

import numpy as np

from . import _lib
from .metadata import (FactorizedTable, IndicatorMatrix, MappingMatrix,
                       SourceSelectors, ind_sel_of, map_sel_t_of)
from .sparse import OpTrace, ShapeError, SparseMatrix, as_dense

DENSE_ACCUM_THRESHOLD = 0.25   # kept for API compatibility (ops.py:30)
ELEMENTWISE_FUNCS = tuple(_lib.EW_IDS)


class OpError(ValueError):
    """Reference `ops.py:33-34`."""


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch") and hasattr(x, "data_ptr")


def _stream_ptr(x=None):
    if x is not None and _is_torch(x):
        import torch
        return C.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
    return C.c_void_p(0)


class DeviceTable:
    """Owner of one `fl_table*` (library-owned device buffers)."""

    def __init__(self, ptr, r_T: int, c_T: int, n_sources: int, device: int):
        self.ptr = ptr
        self.r_T = r_T
        self.c_T = c_T
        self.n_sources = n_sources
        self.device = device

    def layout(self) -> dict:
        sc, sp, ng, ss = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        nb = C.c_int64()
        _lib.call("fl_table_layout", self.ptr, C.byref(sc), C.byref(sp), C.byref(ng),
                  C.byref(ss), C.byref(nb))
        lay = {"stream_cols": sc.value, "stream_pitch": sp.value, "n_gather": ng.value,
               "sort_source": ss.value, "device_bytes": nb.value}
        gathers = []
        for i in range(ng.value):
            si, rows, cols, pitch, matched = (C.c_int32(), C.c_int64(), C.c_int32(),
                                              C.c_int32(), C.c_int64())
            _lib.call("fl_table_gather_info", self.ptr, i, C.byref(si), C.byref(rows),
                      C.byref(cols), C.byref(pitch), C.byref(matched))
            gathers.append({"source": si.value, "rows": rows.value, "cols": cols.value,
                            "pitch": pitch.value, "matched": matched.value})
        lay["gathers"] = gathers
        # one read of every dimension table (bytes), as the fused passes read them
        lay["gather_bytes"] = sum(4 * g["rows"] * g["pitch"] for g in gathers)
        return lay

    def perm(self) -> np.ndarray:
        out = np.empty(self.r_T, dtype=np.int32)
        _lib.call("fl_table_perm", self.ptr, out.ctypes.data_as(C.c_void_p), C.c_void_p(0))
        return out

    def close(self):
        if self.ptr:
            try:
                _lib.load().fl_table_destroy(self.ptr)
            except Exception:
                pass
            self.ptr = None

    def __del__(self):
        self.close()


def upload_arrays(sources, ind_sels, col_maps, r_T: int, c_T: int, *,
                  device: int = 0, stream=None) -> DeviceTable:
    """Upload plain arrays: sources[k] (r_k x c_k, cast to fp32), ind_sels[k]
    (r_T int32, -1 = no match), col_maps[k] (c_k int32 target columns)."""
    trace = os.environ.get("FL_TRACE_UPLOAD") is not None
    t_0 = time.perf_counter()

    def mark(what):
        if trace:
            print(f"[upload_arrays] {what:<28s} {1e3 * (time.perf_counter() - t_0):8.3f} ms",
                  file=sys.stderr, flush=True)

    lib = _lib.load()
    ptr = C.c_void_p()
    _lib.check(lib.fl_table_create(device, int(r_T), int(c_T), C.byref(ptr)), "fl_table_create")
    mark("created")
    tab = DeviceTable(ptr, int(r_T), int(c_T), len(sources), device)
    alive = []   # host buffers must outlive the asynchronous uploads (until finalize)
    for vals, sel, cmap in zip(sources, ind_sels, col_maps):
        if _is_torch(vals):
            import torch
            if vals.dim() != 2:
                raise ShapeError(f"source values must be 2-D, got {tuple(vals.shape)}")
            keep = vals.to(torch.float32).contiguous()   # same cast as the numpy path
            v_ptr, r_k, c_k = keep.data_ptr(), keep.shape[0], keep.shape[1]
        else:
            keep = np.ascontiguousarray(vals, dtype=np.float32)
            v_ptr, (r_k, c_k) = keep.ctypes.data, keep.shape
        if sel is None:           # identity indicator (r_k == r_T)
            s_keep, s_ptr = None, 0
        elif _is_torch(sel):
            import torch
            s_keep = sel.to(torch.int32).reshape(-1).contiguous()
            if s_keep.numel() != int(r_T):
                raise ShapeError(f"ind_sel must have r_T = {r_T} entries, got {s_keep.numel()}")
            s_ptr = s_keep.data_ptr()
        else:
            s_keep = np.ascontiguousarray(sel, dtype=np.int32).reshape(-1)
            if s_keep.size != int(r_T):
                raise ShapeError(f"ind_sel must have r_T = {r_T} entries, got {s_keep.size}")
            s_ptr = s_keep.ctypes.data
        m_keep = np.ascontiguousarray(cmap, dtype=np.int32)
        _lib.check(lib.fl_table_add_source(ptr, int(r_k), int(c_k), C.c_void_p(v_ptr),
                                           C.c_void_p(s_ptr), m_keep.ctypes.data_as(C.c_void_p)),
                   "fl_table_add_source")
        alive.append((keep, s_keep, m_keep))
        mark("source added")
    _lib.check(lib.fl_table_finalize(ptr, stream if stream is not None else C.c_void_p(0)),
               "fl_table_finalize")
    mark("finalized")
    del alive
    return tab


def upload_table(ft, *, device: int = 0) -> DeviceTable:
    """FactorizedTable (product or reference type) -> device layout.

    Indicator / mapping matrices become ind_sel / map_sel_t exactly as the
    reference's `_build_selectors` derives them (`ops.py:58-72`)."""
    srcs, sels, maps = [], [], []
    for k, s in enumerate(ft.sources):
        srcs.append(np.asarray(s.to_dense(), dtype=np.float32))
        sels.append(ind_sel_of(ft, k).astype(np.int32))
        mst = map_sel_t_of(ft, k)
        if np.any(mst < 0):
            from .metadata import MetadataError, ValidationReport
            rep = ValidationReport()
            rep.add(k, "column unmapped", "source column maps to no target column")
            raise MetadataError(rep)
        maps.append(mst.astype(np.int32))
    return upload_arrays(srcs, sels, maps, ft.r_T, ft.c_T, device=device)


def _identity_table(matrix) -> FactorizedTable:
    r, c = matrix.n_rows, matrix.n_cols
    ident_r = SparseMatrix.identity(r)
    ident_c = SparseMatrix.identity(c)
    return FactorizedTable([matrix], [MappingMatrix(ident_c)], [IndicatorMatrix(ident_r)],
                           "inner", r, c)


class TargetHandle:
    """Uniform view of the target table for either execution path, on the B200."""

    def __init__(self, *, table=None, matrix=None, threads: int = 1,
                 accum_threshold: float = DENSE_ACCUM_THRESHOLD, device: int = 0,
                 _dev: DeviceTable | None = None):
        if (table is None) == (matrix is None):
            raise OpError("exactly one of table or matrix must be given")
        self.table = table
        self.matrix = matrix
        self.threads = threads          # accepted for API parity; the GPU ignores it
        self.accum_threshold = accum_threshold
        self.device = device
        self.trace = OpTrace()
        self.trace_log = None
        self._selectors = None
        if _dev is None:
            src = table if table is not None else _identity_table(matrix)
            _dev = upload_table(src, device=device)
        self._dev = _dev

    # -- constructors (ops.py:164-173)
    @classmethod
    def factorized(cls, ft, *, threads: int = 1, check: bool = True,
                   device: int = 0) -> "TargetHandle":
        if check:
            if hasattr(ft, "require_valid"):
                ft.require_valid()
            else:
                FactorizedTable.validate(ft)
        return cls(table=ft, threads=threads, device=device)

    @classmethod
    def materialized(cls, matrix, *, threads: int = 1, device: int = 0) -> "TargetHandle":
        return cls(matrix=matrix, threads=threads, device=device)

    @classmethod
    def from_arrays(cls, sources, ind_sels, col_maps, r_T, c_T, *, device: int = 0,
                    join_type: str = "inner") -> "TargetHandle":
        """Factorized handle straight from plain arrays (bench / large inputs:
        no CSR round trip).  `table` is a lightweight descriptor."""
        dev = upload_arrays(sources, ind_sels, col_maps, r_T, c_T, device=device)
        desc = _ArrayTable(sources, ind_sels, col_maps, r_T, c_T, join_type)
        return cls(table=desc, device=device, _dev=dev)

    @property
    def path(self) -> str:
        return "factorized" if self.table is not None else "materialized"

    @property
    def shape(self) -> tuple[int, int]:
        return (self._dev.r_T, self._dev.c_T)

    @property
    def layout(self) -> dict:
        return self._dev.layout()

    @property
    def selectors(self) -> list[SourceSelectors]:
        """Index-array metadata (reference `ops.py:183-187`).  Gathered sources
        report what the DEVICE derived (perm / stable sort / scan); streamed
        (injective) sources are derived on the host."""
        if self._selectors is None:
            self._selectors = device_selectors(self)
        return self._selectors

    def enable_trace_log(self) -> None:
        self.trace_log = []

    def _record(self, name, traced, t0, madds, rbytes, wbytes):
        if not traced:
            return
        call = OpTrace()
        call.record(madds, rbytes, wbytes, time.perf_counter() - t0)
        self.trace.merge(call)
        if self.trace_log is not None:
            self.trace_log.append((name, self.path, call))

    # -- algorithmic work of one pass over the device layout
    def _pass_cost(self, width: int) -> tuple[int, int]:
        """(multiply-adds, algorithmic bytes read) of one factorized pass of
        operand width `width`: the stream block and the FKs once per target
        row, every dimension table once (its product is formed per dimension
        row, then gathered per target row)."""
        lay = self._dev.layout()
        r_T = self._dev.r_T
        madds = width * r_T * lay["stream_cols"]
        for g in lay["gathers"]:
            madds += width * (g["rows"] * g["cols"] + g["matched"])
        rbytes = 4 * r_T * lay["stream_pitch"] + 4 * r_T * lay["n_gather"]
        rbytes += lay["gather_bytes"]
        return madds, rbytes

    # -- operators
    def lmm(self, x, *, traced: bool = True):
        """T @ x (ops.py:219-235)."""
        r, c = self.shape
        t0 = time.perf_counter()
        if _is_torch(x):
            import torch
            if x.shape[0] != c:
                raise ShapeError(f"lmm: target is {r}x{c} but operand is {tuple(x.shape)}")
            xf = x.to(torch.float32).contiguous()
            out = torch.empty((r, x.shape[1]), dtype=torch.float32, device=x.device)
            _lib.call("fl_lmm", self._dev.ptr, C.c_void_p(xf.data_ptr()), x.shape[1],
                      C.c_void_p(out.data_ptr()), _stream_ptr(x))
            result = out
        else:
            xd = as_dense(x)
            if xd.shape[0] != c:
                raise ShapeError(f"lmm: target is {r}x{c} but operand is {xd.shape}")
            xf = np.ascontiguousarray(xd, dtype=np.float32)
            out = np.empty((r, xd.shape[1]), dtype=np.float32)
            _lib.call("fl_lmm", self._dev.ptr, xf.ctypes.data_as(C.c_void_p), xd.shape[1],
                      out.ctypes.data_as(C.c_void_p), C.c_void_p(0))
            result = _wrap(out.astype(np.float64), x)
        madds, rb = self._pass_cost(int(x.shape[1]) if hasattr(x, "shape") else 1)
        self._record("lmm", traced, t0, madds, rb, 4 * r * int(x.shape[1]))
        return result

    def transpose_lmm(self, x, *, traced: bool = True):
        """T^T @ x (ops.py:255-271)."""
        r, c = self.shape
        t0 = time.perf_counter()
        if _is_torch(x):
            import torch
            if x.shape[0] != r:
                raise ShapeError(f"transpose_lmm: target is {r}x{c} but operand is {tuple(x.shape)}")
            yf = x.to(torch.float32).contiguous()
            out = torch.empty((c, x.shape[1]), dtype=torch.float64, device=x.device)
            _lib.call("fl_tlmm", self._dev.ptr, C.c_void_p(yf.data_ptr()), x.shape[1],
                      C.c_void_p(out.data_ptr()), _stream_ptr(x))
            result = out
        else:
            yd = as_dense(x)
            if yd.shape[0] != r:
                raise ShapeError(f"transpose_lmm: target is {r}x{c} but operand is {yd.shape}")
            yf = np.ascontiguousarray(yd, dtype=np.float32)
            out = np.empty((c, yd.shape[1]), dtype=np.float64)
            _lib.call("fl_tlmm", self._dev.ptr, yf.ctypes.data_as(C.c_void_p), yd.shape[1],
                      out.ctypes.data_as(C.c_void_p), C.c_void_p(0))
            result = _wrap(out, x)
        madds, rb = self._pass_cost(int(x.shape[1]))
        self._record("transpose_lmm", traced, t0, madds, rb + 4 * r * int(x.shape[1]),
                     8 * c * int(x.shape[1]))
        return result

    def rmm(self, x, *, traced: bool = True):
        """x @ T (ops.py:237-253)."""
        r, c = self.shape
        t0 = time.perf_counter()
        if _is_torch(x):
            import torch
            if x.shape[1] != r:
                raise ShapeError(f"rmm: target is {r}x{c} but operand is {tuple(x.shape)}")
            xf = x.to(torch.float32).contiguous()
            out = torch.empty((x.shape[0], c), dtype=torch.float64, device=x.device)
            _lib.call("fl_rmm", self._dev.ptr, C.c_void_p(xf.data_ptr()), x.shape[0],
                      C.c_void_p(out.data_ptr()), _stream_ptr(x))
            result = out
        else:
            xd = as_dense(x)
            if xd.shape[1] != r:
                raise ShapeError(f"rmm: target is {r}x{c} but operand is {xd.shape}")
            xf = np.ascontiguousarray(xd, dtype=np.float32)
            out = np.empty((xd.shape[0], c), dtype=np.float64)
            _lib.call("fl_rmm", self._dev.ptr, xf.ctypes.data_as(C.c_void_p), xd.shape[0],
                      out.ctypes.data_as(C.c_void_p), C.c_void_p(0))
            result = _wrap(out, x)
        madds, rb = self._pass_cost(int(x.shape[0]))
        self._record("rmm", traced, t0, madds, rb + 4 * r * int(x.shape[0]),
                     8 * c * int(x.shape[0]))
        return result

    def row_sum(self, *, traced: bool = True) -> SparseMatrix:
        """Column vector of row sums (ops.py:297-311)."""
        r, _ = self.shape
        t0 = time.perf_counter()
        out = np.empty(r, dtype=np.float32)
        _lib.call("fl_row_sum", self._dev.ptr, out.ctypes.data_as(C.c_void_p), C.c_void_p(0))
        madds, rb = self._pass_cost(1)
        self._record("row_sum", traced, t0, madds, rb, 4 * r)
        return SparseMatrix.from_dense(out.astype(np.float64).reshape(-1, 1))

    def col_sum(self, *, traced: bool = True) -> SparseMatrix:
        """Row vector of column sums (ops.py:313-328)."""
        _, c = self.shape
        t0 = time.perf_counter()
        out = np.empty(c, dtype=np.float64)
        _lib.call("fl_col_sum", self._dev.ptr, out.ctypes.data_as(C.c_void_p), C.c_void_p(0))
        madds, rb = self._pass_cost(1)
        self._record("col_sum", traced, t0, madds, rb, 8 * c)
        return SparseMatrix.from_dense(out.reshape(1, -1))

    def crossprod(self, *, traced: bool = True) -> np.ndarray:
        """T^T T (c_T x c_T) -- the north star's crossprod; the reference has
        no such operator (its composition is transpose_lmm(lmm(I)))."""
        _, c = self.shape
        t0 = time.perf_counter()
        out = np.empty((c, c), dtype=np.float64)
        _lib.call("fl_crossprod", self._dev.ptr, out.ctypes.data_as(C.c_void_p), C.c_void_p(0))
        madds, rb = self._pass_cost(c)
        self._record("crossprod", traced, t0, madds, rb, 8 * c * c)
        return out

    def materialize_target(self, *, traced: bool = False) -> SparseMatrix:
        """The full target matrix (ops.py:206-217); values are exact copies."""
        return SparseMatrix.from_dense(self.materialize_dense(traced=traced).astype(np.float64))

    def materialize_dense(self, *, traced: bool = False, out=None):
        """Dense fp32 target (numpy, or into a CUDA tensor `out`)."""
        r, c = self.shape
        t0 = time.perf_counter()
        if out is not None and _is_torch(out):
            _lib.call("fl_materialize", self._dev.ptr, C.c_void_p(out.data_ptr()),
                      _stream_ptr(out))
            res = out
        else:
            res = np.empty((r, c), dtype=np.float32)
            _lib.call("fl_materialize", self._dev.ptr, res.ctypes.data_as(C.c_void_p),
                      C.c_void_p(0))
        _, rb = self._pass_cost(0)
        self._record("materialize", traced, t0, 0, rb, 4 * r * c)
        return res

    def elementwise(self, func: str, scalar: float | None = None, *,
                    traced: bool = True) -> "TargetHandle":
        """Registered zero-preserving map on the stored values (ops.py:273-295)."""
        if func not in _lib.EW_IDS:
            raise OpError(f"elementwise map {func!r} is not registered "
                          "(or does not preserve zero): requires materialization fallback")
        needs_scalar = func in ("scale", "divide")
        if needs_scalar and scalar is None:
            raise OpError(f"{func!r} requires a scalar argument")
        if func == "divide" and scalar == 0.0:
            raise OpError("division by zero scalar")
        t0 = time.perf_counter()
        ptr = C.c_void_p()
        _lib.call("fl_elementwise", self._dev.ptr, _lib.EW_IDS[func],
                  float(scalar) if scalar is not None else 0.0, C.byref(ptr), C.c_void_p(0))
        dev = DeviceTable(ptr, self._dev.r_T, self._dev.c_T, self._dev.n_sources, self.device)
        new_table = None
        if self.table is not None:
            new_table = _MappedTable(self.table, func, scalar)
        out = TargetHandle(table=new_table, matrix=None if self.table is not None else
                           _MappedMatrix(self.matrix, func, scalar),
                           threads=self.threads, accum_threshold=self.accum_threshold,
                           device=self.device, _dev=dev)
        out._selectors = self._selectors
        madds, rb = self._pass_cost(0)
        self._record("elementwise", traced, t0, madds // max(1, 1), rb, rb)
        return out


def _wrap(arr: np.ndarray, like):
    """Return the boundary type matching the operand: SparseMatrix in ->
    SparseMatrix out (reference contract), array in -> array out."""
    if hasattr(like, "indptr"):
        return SparseMatrix.from_dense(arr)
    return arr


class _ArrayTable:
    """Minimal table descriptor for handles built from arrays."""

    def __init__(self, sources, ind_sels, col_maps, r_T, c_T, join_type):
        self.n_sources = len(sources)
        self.r_T = int(r_T)
        self.c_T = int(c_T)
        self.join_type = join_type
        self.shapes = [tuple(s.shape) for s in sources]

    @property
    def shape(self):
        return (self.r_T, self.c_T)


class _MappedTable:
    """Descriptor of `elementwise(f)` applied to a table: shares mappings and
    indicators (reference `ops.py:285-293`); values live on the device."""

    def __init__(self, base, func, scalar):
        self.base = base
        self.func = func
        self.scalar = scalar
        self.mappings = getattr(base, "mappings", None)
        self.indicators = getattr(base, "indicators", None)
        self.join_type = getattr(base, "join_type", "inner")
        self.r_T = base.r_T
        self.c_T = base.c_T

    @property
    def shape(self):
        return (self.r_T, self.c_T)


class _MappedMatrix:
    def __init__(self, base, func, scalar):
        self.base = base
        self.func = func
        self.scalar = scalar
        self.n_rows = base.n_rows
        self.n_cols = base.n_cols

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)


def device_selectors(h: TargetHandle) -> list[SourceSelectors]:
    """Selectors as derived by the device (gathered sources) plus host-side
    derivation for streamed sources (their rows live expanded on the device)."""
    out = []
    dev = h._dev
    ft = h.table if h.table is not None and hasattr(h.table, "indicators") else None
    for k in range(dev.n_sources):
        ind_sel = np.empty(dev.r_T, dtype=np.int32)
        lib = _lib.load()
        st = lib.fl_table_selectors(dev.ptr, k, ind_sel.ctypes.data_as(C.c_void_p), None, None,
                                    C.c_void_p(0))
        if st == _lib.FL_OK:
            n_rows = int(ind_sel.max()) + 1 if ind_sel.size else 0
            if ft is not None:
                n_rows = ft.sources[k].n_rows
            gptr = np.empty(n_rows + 1, dtype=np.int64)
            matched = int((ind_sel >= 0).sum())
            grows = np.empty(max(matched, 1), dtype=np.int32)
            _lib.call("fl_table_selectors", dev.ptr, k, None, gptr.ctypes.data_as(C.c_void_p),
                      grows.ctypes.data_as(C.c_void_p), C.c_void_p(0))
            ind = ind_sel.astype(np.int64)
            grows = grows[:matched].astype(np.int64)
        else:
            if ft is None:
                raise OpError("selectors of a streamed source need the host table")
            ind = ind_sel_of(ft, k)
            n_rows = ft.sources[k].n_rows
            order = np.argsort(ind, kind="stable")
            grows = order[ind[order] >= 0]
            gptr = np.zeros(n_rows + 1, dtype=np.int64)
            np.cumsum(np.bincount(ind[ind >= 0], minlength=n_rows), out=gptr[1:])
        if ft is not None:
            mst = map_sel_t_of(ft, k)
            map_sel = np.full(dev.c_T, -1, dtype=np.int64)
            map_sel[mst[mst >= 0]] = np.nonzero(mst >= 0)[0]
        else:
            mst = np.empty(0, dtype=np.int64)
            map_sel = np.full(dev.c_T, -1, dtype=np.int64)
        out.append(SourceSelectors(ind, gptr, grows, map_sel, mst))
    return out


def export_trace_csv(path, rows) -> None:
    """Write logged per-op traces as CSV (reference `ops.py:331-341`)."""
    import csv
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["op", "side", "multiply_adds", "bytes_read", "bytes_written", "wall_time"])
        for name, side, tr in rows:
            w.writerow([name, side, tr.multiply_add_count, tr.bytes_read,
                        tr.bytes_written, f"{tr.wall_time:.9f}"])
