"""Matrix entries A_ij = K(x_i, x_j) (oracle; test infrastructure only).

P:105-111: A_ij is the interaction between target u_i and source v_j; here u = v
(P:1248).  Kernel ids follow BASELINE.json `configs`:
  0  log r          (configs 1-2; diagonal A_ii = diag)
  1  exp(-r / ell)  (config 3, Matern-1/2; A_ii = 1 + nugget = diag)
  2  1 / r          (configs 4-5, and the paper's Exp. 3 kernel P:1370-1378 with diag sqrt(1000 N))
Off-diagonal entries use r = sqrt(sum_a (x_a - y_a)^2); a zero distance off the
diagonal for a singular kernel is an error (coincident points).
"""
from __future__ import annotations

import numpy as np


def entries(kernel_id: int, kparams, X: np.ndarray, Y: np.ndarray, ix=None, iy=None):
    """Block A(X, Y) for point sets X (p x d), Y (q x d).

    ix, iy: global indices of the rows / columns; where ix[a] == iy[b] the entry
    is the diagonal value (self interaction)."""
    diag, ell = kparams
    diff = X[:, None, :] - Y[None, :, :]
    r = np.sqrt(np.sum(diff * diff, axis=2))
    self_mask = None
    if ix is not None and iy is not None:
        self_mask = np.asarray(ix)[:, None] == np.asarray(iy)[None, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        if kernel_id == 0:
            k = np.log(r)
        elif kernel_id == 1:
            k = np.exp(-r / ell)
        elif kernel_id == 2:
            k = 1.0 / r
        else:
            raise ValueError("unknown kernel id")
    if self_mask is not None:
        k = np.where(self_mask, diag, k)
    if not np.all(np.isfinite(k)):
        raise FloatingPointError("coincident points with a singular kernel")
    return k


def block(kernel_id, kparams, pts: np.ndarray, rows, cols):
    """A(rows, cols) for global (tree-order) index arrays."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    return entries(kernel_id, kparams, pts[rows], pts[cols], rows, cols)
