"""Host-side CSR container and operator trace record.

This is the *boundary data type* of the reference's operator API
(`pkg/src/factorlearn/sparse.py:83-189`): every TargetHandle operand and
result is a CSR float64 matrix.  Here it is only a container plus the
dense<->CSR format conversions needed at the API edge; no arithmetic kernel
lives on the host.  All products run on the B200 through the C ABI
(`include/fl_b200.h`).

Invariants (same as the reference, `sparse.py:83-89`): column indices strictly
increasing within a row and below n_cols, no explicit zeros, indptr monotone
with indptr[0] == 0 and indptr[-1] == nnz.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class ShapeError(ValueError):
    """Operand shapes do not conform (reference `sparse.py:39-40`)."""


class SparseStructureError(ValueError):
    """A CSR triple violates the storage invariants (reference `sparse.py:43-44`)."""


_STRUCTURE_ERRORS = {
    1: "row extents are not monotone or do not span the stored values",
    2: "column index out of range",
    3: "column indices not strictly increasing within a row",
    4: "explicit zero stored",
    5: "non-finite value stored",
}


@dataclass
class OpTrace:
    """Work record of one or more operator calls (reference `sparse.py:56-80`).

    On the GPU path `multiply_add_count` is the dense multiply-add count of the
    kernels launched and `bytes_read` / `bytes_written` are the *algorithmic*
    HBM bytes of those kernels (the roofline numerator), not the reference's
    16-bytes-per-stored-element CPU charge.  `wall_time` is device time
    measured with CUDA events.
    """

    multiply_add_count: int = 0
    bytes_read: int = 0
    bytes_written: int = 0
    wall_time: float = 0.0

    def record(self, madds: int, bytes_read: int, bytes_written: int,
               seconds: float) -> None:
        self.multiply_add_count += int(madds)
        self.bytes_read += int(bytes_read)
        self.bytes_written += int(bytes_written)
        self.wall_time += float(seconds)

    def merge(self, other: "OpTrace") -> None:
        self.record(other.multiply_add_count, other.bytes_read,
                    other.bytes_written, other.wall_time)


def _structure_code(n_rows, n_cols, indptr, indices, data) -> int:
    """Vectorised restatement of the reference's `structure_ok`
    (`_kernels.py:347-372`); returns the same error codes."""
    if indptr[0] != 0 or indptr[n_rows] != indices.shape[0]:
        return 1
    if np.any(np.diff(indptr) < 0):
        return 1
    if indices.size:
        if indices.min() < 0 or indices.max() >= n_cols:
            return 2
        rows = np.repeat(np.arange(n_rows), np.diff(indptr))
        same_row = rows[1:] == rows[:-1]
        if np.any(same_row & (indices[1:] <= indices[:-1])):
            return 3
        if np.any(data == 0.0):
            return 4
        if not np.all(np.isfinite(data)):
            return 5
    return 0


class SparseMatrix:
    """2-D CSR matrix with float64 values (API mirror of reference
    `sparse.py:83-189`)."""

    __slots__ = ("n_rows", "n_cols", "indptr", "indices", "data")

    def __init__(self, n_rows: int, n_cols: int, indptr, indices, data, *,
                 check: bool = True):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int64)
        self.data = np.ascontiguousarray(data, dtype=np.float64)
        if check:
            if self.indptr.shape[0] != self.n_rows + 1:
                raise SparseStructureError(
                    f"indptr has length {self.indptr.shape[0]}, expected {self.n_rows + 1}")
            if self.indices.shape[0] != self.data.shape[0]:
                raise SparseStructureError("indices and data lengths differ")
            code = _structure_code(self.n_rows, self.n_cols, self.indptr,
                                   self.indices, self.data)
            if code:
                raise SparseStructureError(_STRUCTURE_ERRORS[code])

    @property
    def nnz(self) -> int:
        return int(self.indices.shape[0])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    @property
    def density(self) -> float:
        cells = self.n_rows * self.n_cols
        return self.nnz / cells if cells else 0.0

    @classmethod
    def from_dense(cls, arr) -> "SparseMatrix":
        arr = np.asarray(arr, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError("from_dense expects a 2-D array")
        rows, cols = np.nonzero(arr)
        indptr = np.zeros(arr.shape[0] + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, minlength=arr.shape[0]), out=indptr[1:])
        return cls(arr.shape[0], arr.shape[1], indptr, cols, arr[rows, cols],
                   check=False)

    @classmethod
    def from_coo(cls, n_rows: int, n_cols: int, rows, cols, vals) -> "SparseMatrix":
        """Coordinate triples; duplicates summed (reference `sparse.py:133-154`)."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        if rows.size:
            if rows.min() < 0 or rows.max() >= n_rows:
                raise SparseStructureError("row index out of range")
            if cols.min() < 0 or cols.max() >= n_cols:
                raise SparseStructureError("column index out of range")
        order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        if rows.size:
            keys = rows * n_cols + cols
            uniq, start = np.unique(keys, return_index=True)
            vals = np.add.reduceat(vals, start)
            rows = uniq // n_cols
            cols = uniq % n_cols
        keep = vals != 0.0
        rows, cols, vals = rows[keep], cols[keep], vals[keep]
        indptr = np.zeros(n_rows + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, minlength=n_rows), out=indptr[1:])
        return cls(n_rows, n_cols, indptr, cols, vals, check=False)

    @classmethod
    def identity(cls, n: int) -> "SparseMatrix":
        return cls(n, n, np.arange(n + 1), np.arange(n), np.ones(n), check=False)

    @classmethod
    def zeros(cls, n_rows: int, n_cols: int) -> "SparseMatrix":
        return cls(n_rows, n_cols, np.zeros(n_rows + 1, dtype=np.int64),
                   np.empty(0, dtype=np.int64), np.empty(0), check=False)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols))
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.indptr))
        out[rows, self.indices] = self.data
        return out

    def row_nnz(self) -> np.ndarray:
        return np.diff(self.indptr)

    def __repr__(self) -> str:
        return f"SparseMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz})"


def as_dense(x) -> np.ndarray:
    """Dense float64 2-D view of a SparseMatrix / array-like operand
    (duck-typed so a reference `factorlearn.SparseMatrix` works too)."""
    if hasattr(x, "indptr") and hasattr(x, "to_dense"):
        return np.asarray(x.to_dense(), dtype=np.float64)
    arr = np.asarray(x, dtype=np.float64)
    if arr.ndim == 1:
        arr = arr.reshape(-1, 1)
    return arr


def equal_exact(a: SparseMatrix, b: SparseMatrix) -> bool:
    """Bitwise structural and value equality (reference `sparse.py:192-197`)."""
    return (a.shape == b.shape
            and np.array_equal(a.indptr, b.indptr)
            and np.array_equal(a.indices, b.indices)
            and np.array_equal(a.data, b.data))


__all__ = ["OpTrace", "ShapeError", "SparseMatrix", "SparseStructureError",
           "as_dense", "equal_exact"]
