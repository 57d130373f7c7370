"""Float64 restatement of the reference trainers (TEST ORACLE ONLY).

Follows `pkg/src/factorlearn/trainers.py` line by line, written against the
oracle operators in `reference_ops.py` so the call sequence is the reference's:

  linear_regression    trainers.py:138-163
  logistic_regression  trainers.py:166-195
  kmeans               trainers.py:198-246
  gaussian_nmf         trainers.py:256-307
  train                trainers.py:320-331
  safe_learning_rate   bench.py:112-123 (computed from the dense target)

Returns plain dicts: {"model", "parameters", "loss_history"}.
"""

from __future__ import annotations

import numpy as np

from . import reference_ops as ops

EPS_NMF = 1e-12  # trainers.py:29


class OracleDivergence(ValueError):
    def __init__(self, model, iteration):
        super().__init__(f"{model}: non-finite loss at iteration {iteration}")
        self.iteration = iteration


def _finite(loss, model, it):
    if not np.isfinite(loss):
        raise OracleDivergence(model, it)
    return float(loss)


def linear_regression(tab, y, iterations, lr):
    """trainers.py:138-163: w <- w - lr T^T(Tw - y); loss at entering w."""
    yd = np.asarray(y, dtype=np.float64).reshape(-1, 1)
    w = np.zeros((tab.c_T, 1))
    losses = []
    for it in range(iterations):
        z = ops.lmm(tab, w)
        resid = z - yd
        losses.append(_finite(0.5 * (resid.T @ resid).item(), "linreg", it))
        grad = ops.transpose_lmm(tab, resid)
        w = w - lr * grad
    return {"model": "linreg", "parameters": {"w": w}, "loss_history": losses}


def logistic_regression(tab, y, iterations, lr):
    """trainers.py:166-195: sigma on the dense z, clipped log-loss."""
    yd = np.asarray(y, dtype=np.float64).reshape(-1, 1)
    w = np.zeros((tab.c_T, 1))
    losses = []
    for it in range(iterations):
        z = ops.lmm(tab, w)
        p = 1.0 / (1.0 + np.exp(-z))
        pc = np.clip(p, 1e-12, 1.0 - 1e-12)
        loss = -(yd.T @ np.log(pc) + (1.0 - yd).T @ np.log1p(-pc)).item()
        losses.append(_finite(loss, "logreg", it))
        grad = ops.transpose_lmm(tab, p - yd)
        w = w - lr * grad
    return {"model": "logreg", "parameters": {"w": w}, "loss_history": losses}


def kmeans(tab, iterations, k, seed):
    """trainers.py:198-246 (Lloyd in LA form; ties -> lowest index; empty
    clusters keep their centroid)."""
    r_t, _ = tab.shape
    if k > r_t:
        raise ValueError(f"k_clusters = {k} exceeds row count {r_t}")
    rng = np.random.default_rng(seed)
    pick = np.sort(rng.choice(r_t, size=k, replace=False))      # :209-210
    sel = np.zeros((k, r_t))
    sel[np.arange(k), pick] = 1.0
    centroids = ops.rmm(tab, sel)                                 # :217-218
    sq_rows = ops.row_sum(ops.elementwise(tab, "square"))        # :219-223
    ones_k = np.ones((1, k))
    losses = []
    assign = None
    for it in range(iterations):
        tc = ops.lmm(tab, centroids.T)                            # :227
        dist = sq_rows @ ones_k - 2.0 * tc + (centroids ** 2).sum(axis=1)
        assign = np.argmin(dist, axis=1)                          # :229
        losses.append(_finite(float(dist[np.arange(r_t), assign].sum()),
                              "kmeans", it))
        onehot = np.zeros((r_t, k))
        onehot[np.arange(r_t), assign] = 1.0
        sums = ops.transpose_lmm(tab, onehot).T                   # :236
        counts = onehot.sum(axis=0)
        live = counts > 0
        centroids = centroids.copy()
        centroids[live] = sums[live] / counts[live, None]
    return {"model": "kmeans",
            "parameters": {"centroids": centroids, "assignments": assign},
            "loss_history": losses}


def gaussian_nmf(tab, iterations, rank, seed):
    """trainers.py:256-307 (multiplicative updates; H first, then W; loss via
    the Gram identity after each iteration's updates)."""
    r_t, c_t = tab.shape
    r = rank
    if r > min(r_t, c_t):
        raise ValueError(f"rank = {r} exceeds min(shape) = {min(r_t, c_t)}")
    total = ops.row_sum(tab).sum()                                # :272
    scale = total / (r_t * c_t) if total > 0 else 1.0
    rng = np.random.default_rng(seed)
    w = rng.random((r_t, r)) * scale                              # :275
    h = rng.random((r, c_t)) * scale                              # :276
    t_sq = float(ops.row_sum(ops.elementwise(tab, "square")).sum())

    def frob_loss(p):
        wtw = w.T @ w
        return t_sq - 2.0 * float((p * h).sum()) + float((wtw * (h @ h.T)).sum())

    losses = []
    for it in range(iterations):
        p = ops.rmm(tab, w.T)                                     # :288
        if it > 0:
            losses.append(_finite(frob_loss(p), "gnmf", it - 1))
        h = h * p / (w.T @ w @ h + EPS_NMF)                       # :296
        q = ops.lmm(tab, h.T)                                     # :297
        w = w * q / (w @ (h @ h.T) + EPS_NMF)                     # :298
    p_final = ops.rmm(tab, w.T)
    losses.append(_finite(frob_loss(p_final), "gnmf", iterations - 1))
    return {"model": "gnmf", "parameters": {"w": w, "h": h}, "loss_history": losses}


def train(model, tab, *, iterations, learning_rate=1e-3, k_clusters=4,
          rank=2, seed=0, y=None):
    """Dispatcher mirroring trainers.py:320-331."""
    if model == "linreg":
        return linear_regression(tab, y, iterations, learning_rate)
    if model == "logreg":
        return logistic_regression(tab, y, iterations, learning_rate)
    if model == "kmeans":
        return kmeans(tab, iterations, k_clusters, seed)
    if model == "gnmf":
        return gaussian_nmf(tab, iterations, rank, seed)
    raise ValueError(f"unknown model {model!r}")


def safe_learning_rate(tab) -> float:
    """bench.py:112-123: 1 / (max row L1 * max col L1) of |T|, computed
    factorized: row L1 = sum_k I_k rowsum|S_k|, col L1 = fanout-weighted."""
    a = ops.elementwise(tab, "abs")
    row = ops.row_sum(a).max()
    col = ops.col_sum(a).max()
    bound = row * col
    return 1.0 / bound if bound > 0 else 1.0
