"""Small dense helpers with decision rules shared (by specification, not by code)
with the CUDA path (oracle; test infrastructure only).

R7 tie-window argmax: the pivot is the LOWEST index whose magnitude
is >= (1 - 1e-10) * max.  Exact ties of the paper's symmetric grid workloads are
then broken identically on CPU and GPU, although the two round differently.

R8 pivoted-QR truncation (the paper's RRQR, "relative residual ...
O(eps_A)"): column-pivoted Gram-Schmidt with re-orthogonalisation; after t
steps the residual is W_t = (I - Q_t Q_t^T) W; stop when ||W_t||_F <= tau.
A pivot column whose re-orthogonalised norm keeps collapsing (it lies in the span
of the basis to working precision) is discarded rather than normalised.
"""
from __future__ import annotations

import numpy as np

TIE = 1e-10


def pick(values: np.ndarray, used: np.ndarray | None = None):
    """R7: lowest index with |v| >= (1 - TIE) * max|v| over unused entries; None if max is 0."""
    a = np.abs(values).astype(np.float64)
    if used is not None:
        a = np.where(used, -1.0, a)
    if a.size == 0:
        return None
    mx = a.max()
    if not mx > 0.0:
        return None
    thr = mx * (1.0 - TIE)
    return int(np.flatnonzero(a >= thr)[0])


def pivoted_qr_extend(W: np.ndarray, basis: np.ndarray, tau: float, tmin: int, tmax: int):
    """Pivoted Gram-Schmidt on the columns of W (already projected against `basis`).

    Takes pivots while (t < tmin) or (||W_t||_F > tau), never more than tmax, and
    stops when no column has a non-zero residual.  Returns (Q_new, t_truncation)
    where t_truncation is the count taken before the tau test first stopped
    (== len(Q_new) when tmin does not bind).
    """
    W = np.array(W, dtype=np.float64, copy=True)
    m = W.shape[0]
    B = basis.copy() if basis is not None else np.zeros((m, 0))
    qs = []
    t_trunc = None
    while len(qs) < tmax:
        norms2 = np.sum(W * W, axis=0) if W.shape[1] else np.zeros(0)
        res = np.sqrt(np.sum(norms2))
        if t_trunc is None and not res > tau:
            t_trunc = len(qs)
        if len(qs) >= tmin and not res > tau:
            break
        j = pick(np.sqrt(norms2))
        if j is None:
            break
        w = W[:, j].copy()
        # R8 re-orthogonalisation against everything taken so far: two passes, a third
        # if the second cancelled more than half; a column still collapsing after the
        # third pass lies in span(B) numerically and is discarded
        w = w - B @ (B.T @ w)
        n1 = np.linalg.norm(w)
        w = w - B @ (B.T @ w)
        nw = np.linalg.norm(w)
        if not nw > 0.5 * n1:
            n2 = nw
            w = w - B @ (B.T @ w)
            nw = np.linalg.norm(w)
            if not nw > 0.5 * n2:
                nw = 0.0
        if not nw > 0.0:
            W[:, j] = 0.0
            continue
        q = w / nw
        qs.append(q)
        B = np.concatenate([B, q[:, None]], axis=1)
        W = W - np.outer(q, q @ W)
        W[:, j] = 0.0
    if t_trunc is None:
        t_trunc = len(qs)
    Q = np.stack(qs, axis=1) if qs else np.zeros((m, 0))
    return Q, t_trunc
