"""Float64 numpy restatement of the reference operators (TEST ORACLE ONLY).

Follows `pkg/src/factorlearn/ops.py` (factorized branch of each
`TargetHandle` method) with dense numpy arrays in place of CSR:

  lmm            ops.py:219-235   T x   = sum_k I_k (S_k (M_k^T x))
  transpose_lmm  ops.py:255-271   T^T y = sum_k M_k (S_k^T (I_k^T y))
  rmm            ops.py:237-253   x T   = sum_k ((x I_k) S_k) M_k^T
  row_sum        ops.py:297-311   sum_k I_k rowSum(S_k)
  col_sum        ops.py:313-328   sum_k (fanout_k^T S_k) M_k^T
  materialize    metadata.py:215-225 / ops.py:206-217
  selectors      ops.py:55-74

Per-source partials are accumulated in source order (`ops.py:122-144`);
I_k^T is the grouped sum in ascending member order (`_kernels.py:252-288`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class OracleTable:
    """Plain-array form of a FactorizedTable: dense float64 sources plus
    ind_sel (r_T, int64, -1 = padding) and map_sel_t (c_k, int64) per source."""

    sources: list          # list[np.ndarray (r_k, c_k) float64]
    ind_sel: list          # list[np.ndarray (r_T,) int64]
    map_sel_t: list        # list[np.ndarray (c_k,) int64]
    r_T: int
    c_T: int

    @classmethod
    def from_ft(cls, ft) -> "OracleTable":
        """From any FactorizedTable-like object (reference or product type);
        ind_sel / map_sel_t restate `ops.py:58-61`, `ops.py:67-72`."""
        srcs, sels, maps = [], [], []
        for s, mp, ind in zip(ft.sources, ft.mappings, ft.indicators):
            srcs.append(np.asarray(s.to_dense(), dtype=np.float64))
            im = ind.matrix
            ip = np.asarray(im.indptr)
            sel = np.full(ft.r_T, -1, dtype=np.int64)
            matched = np.nonzero(np.diff(ip) == 1)[0]
            sel[matched] = np.asarray(im.indices)[ip[matched]]
            sels.append(sel)
            mm = mp.matrix
            mp_ip = np.asarray(mm.indptr)
            map_sel = np.full(ft.c_T, -1, dtype=np.int64)
            mapped = np.nonzero(np.diff(mp_ip) == 1)[0]
            map_sel[mapped] = np.asarray(mm.indices)[mp_ip[mapped]]
            mst = np.full(s.n_cols, -1, dtype=np.int64)
            mst[map_sel[mapped]] = mapped
            maps.append(mst)
        return cls(srcs, sels, maps, int(ft.r_T), int(ft.c_T))

    @property
    def shape(self):
        return (self.r_T, self.c_T)


def build_selectors(tab: OracleTable):
    """Per-source (ind_sel, group_indptr, group_rows, map_sel, map_sel_t),
    restating `ops.py:55-74` (stable argsort, negatives dropped)."""
    out = []
    for s, ind_sel, mst in zip(tab.sources, tab.ind_sel, tab.map_sel_t):
        order = np.argsort(ind_sel, kind="stable")
        order = order[ind_sel[order] >= 0]
        counts = np.bincount(ind_sel[ind_sel >= 0], minlength=s.shape[0])
        group_indptr = np.zeros(s.shape[0] + 1, dtype=np.int64)
        np.cumsum(counts, out=group_indptr[1:])
        map_sel = np.full(tab.c_T, -1, dtype=np.int64)
        ok = mst >= 0
        map_sel[mst[ok]] = np.nonzero(ok)[0]
        out.append((ind_sel, group_indptr, order, map_sel, mst))
    return out


def _gather_rows(sel, a):
    """Row gather with -1 -> zero row (`_kernels.py:224-249`)."""
    out = np.zeros((sel.shape[0], a.shape[1]))
    ok = sel >= 0
    out[ok] = a[sel[ok]]
    return out


def _group_sum(ind_sel, n_groups, x):
    """I_k^T x: ascending-member grouped sum (`_kernels.py:252-288`)."""
    out = np.zeros((n_groups, x.shape[1]))
    ok = ind_sel >= 0
    idx = ind_sel[ok]
    xs = x[ok]
    for c in range(x.shape[1]):
        out[:, c] = np.bincount(idx, weights=xs[:, c], minlength=n_groups)
    return out


def lmm(tab: OracleTable, x: np.ndarray) -> np.ndarray:
    """T @ x (`ops.py:219-235`, factorized branch)."""
    x = np.asarray(x, dtype=np.float64)
    assert x.shape[0] == tab.c_T
    acc = np.zeros((tab.r_T, x.shape[1]))
    for s, sel, mst in zip(tab.sources, tab.ind_sel, tab.map_sel_t):
        u = _gather_rows(mst, x)          # M_k^T x   (ops.py:230)
        v = s @ u                         # S_k u     (ops.py:231)
        acc += _gather_rows(sel, v)       # I_k v     (ops.py:232)
    return acc


def transpose_lmm(tab: OracleTable, y: np.ndarray) -> np.ndarray:
    """T^T @ y (`ops.py:255-271`, factorized branch)."""
    y = np.asarray(y, dtype=np.float64)
    assert y.shape[0] == tab.r_T
    acc = np.zeros((tab.c_T, y.shape[1]))
    for s, sel, mst in zip(tab.sources, tab.ind_sel, tab.map_sel_t):
        u = _group_sum(sel, s.shape[0], y)  # I_k^T y  (ops.py:266)
        v = s.T @ u                         # S_k^T u  (ops.py:267)
        ok = mst >= 0
        acc[mst[ok]] += v[ok]               # M_k v    (ops.py:268)
    return acc


def rmm(tab: OracleTable, x: np.ndarray) -> np.ndarray:
    """x @ T (`ops.py:237-253`, factorized branch)."""
    x = np.asarray(x, dtype=np.float64)
    assert x.shape[1] == tab.r_T
    acc = np.zeros((x.shape[0], tab.c_T))
    for s, sel, mst in zip(tab.sources, tab.ind_sel, tab.map_sel_t):
        w = _group_sum(sel, s.shape[0], x.T).T   # x I_k   (ops.py:248)
        z = w @ s                                # (x I_k) S_k (ops.py:249)
        ok = mst >= 0
        acc[:, mst[ok]] += z[:, ok]              # . M_k^T (ops.py:250)
    return acc


def row_sum(tab: OracleTable) -> np.ndarray:
    """(`ops.py:297-311`) sum_k I_k rowSum(S_k); padding rows are zero."""
    acc = np.zeros((tab.r_T, 1))
    for s, sel in zip(tab.sources, tab.ind_sel):
        acc += _gather_rows(sel, s.sum(axis=1, keepdims=True))
    return acc


def col_sum(tab: OracleTable) -> np.ndarray:
    """(`ops.py:313-328`) fanout-weighted source column sums, remapped."""
    acc = np.zeros((1, tab.c_T))
    for s, sel, mst in zip(tab.sources, tab.ind_sel, tab.map_sel_t):
        fan = np.bincount(sel[sel >= 0], minlength=s.shape[0]).astype(np.float64)
        z = fan.reshape(1, -1) @ s
        ok = mst >= 0
        acc[:, mst[ok]] += z[:, ok]
    return acc


ELEMENTWISE = {
    # registered zero-preserving maps (`sparse.py:300-307`)
    "scale": (True, lambda v, x: v * x),
    "divide": (True, lambda v, x: v / x),
    "square": (False, lambda v, _: v * v),
    "abs": (False, lambda v, _: np.abs(v)),
    "expm1": (False, lambda v, _: np.expm1(v)),
    "logistic_centered": (False, lambda v, _: 1.0 / (1.0 + np.exp(-v)) - 0.5),
}


def elementwise(tab: OracleTable, func: str, scalar=None) -> OracleTable:
    """(`ops.py:273-295`, `sparse.py:312-339`) map applied to source values."""
    _, fn = ELEMENTWISE[func]
    return OracleTable([fn(s, scalar) for s in tab.sources], tab.ind_sel,
                       tab.map_sel_t, tab.r_T, tab.c_T)


def materialize(tab: OracleTable) -> np.ndarray:
    """(`metadata.py:215-225`) sum_k I_k (S_k M_k^T), dense."""
    out = np.zeros((tab.r_T, tab.c_T))
    for s, sel, mst in zip(tab.sources, tab.ind_sel, tab.map_sel_t):
        scattered = np.zeros((s.shape[0], tab.c_T))
        ok = mst >= 0
        scattered[:, mst[ok]] = s[:, ok]
        out += _gather_rows(sel, scattered)
    return out
