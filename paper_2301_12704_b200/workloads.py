"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no tree, no kernel entries, no
factorization): it only draws points, right-hand sides and residual-sample rows
from documented seeded generators, so that the oracle (`oracle/`) and the CUDA
path read identical bytes.

Configs follow BASELINE.json `configs` (0-based index here = config number - 1):

  0  2D, N=4096,  linspace(-1,1,64)^2 grid, log r,  A_ii=10,   leaf 64,  tol 1e-8,  1 RHS  (seed 0)
  1  2D, N=65536, U[-1,1]^2 (seed 1),      log r,  A_ii=10,   leaf 64,  tol 1e-10, 16 RHS
  2  2D, N=2^20,  U[-1,1]^2 (seed 2),      exp(-r/0.1), A_ii=1+1e-2, leaf 128, tol 1e-8, 1 RHS
  3  3D, N=2^18,  linspace(-1,1,64)^3 grid, 1/r, A_ii=128,   leaf 64,  tol 1e-7,  8 RHS (seed 3)
  4  3D, N=2^21,  U[0,1)^3 (seed 4),        1/r, A_ii=100,   leaf 128, tol 1e-3 (preconditioner)

Kernel ids (the C-ABI's `kernel_id`): 0 = log r, 1 = exp(-r/ell), 2 = 1/r.
`kparams` = (diag, ell) — diag is A_ii, ell is the exp length scale.
"""
from __future__ import annotations

import dataclasses
import numpy as np

KERNEL_LOG, KERNEL_EXP, KERNEL_INVR = 0, 1, 2


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    d: int
    n: int
    points: str          # "grid" | "uniform_pm1" | "uniform_01"
    kernel_id: int
    diag: float
    ell: float
    leaf_size: int
    tol: float
    nrhs: int
    seed: int

    @property
    def kparams(self):
        return (float(self.diag), float(self.ell))


CONFIGS = [
    Workload("cfg1_grid2d_log_4096", 2, 4096, "grid", KERNEL_LOG, 10.0, 0.0, 64, 1e-8, 1, 0),
    Workload("cfg2_rand2d_log_65536", 2, 65536, "uniform_pm1", KERNEL_LOG, 10.0, 0.0, 64, 1e-10, 16, 1),
    Workload("cfg3_rand2d_matern_1M", 2, 1 << 20, "uniform_pm1", KERNEL_EXP, 1.0 + 1e-2, 0.1, 128, 1e-8, 1, 2),
    Workload("cfg4_grid3d_invr_262144", 3, 1 << 18, "grid", KERNEL_INVR, 128.0, 0.0, 64, 1e-7, 8, 3),
    Workload("cfg5_rand3d_invr_2M", 3, 1 << 21, "uniform_01", KERNEL_INVR, 100.0, 0.0, 128, 1e-3, 1, 4),
]


def make_points(kind: str, n: int, d: int, seed: int) -> np.ndarray:
    """N x d float64, C-contiguous (row-major), user order."""
    if kind == "grid":
        side = int(round(n ** (1.0 / d)))
        if side ** d != n:
            raise ValueError("grid workload needs a perfect power")
        ax = np.linspace(-1.0, 1.0, side)
        mesh = np.meshgrid(*([ax] * d), indexing="ij")
        # axis 0 varies slowest in user order; order is irrelevant to the method
        return np.ascontiguousarray(np.stack([m.reshape(-1) for m in mesh], axis=1))
    rng = np.random.default_rng(seed)
    if kind == "uniform_pm1":
        return rng.uniform(-1.0, 1.0, size=(n, d))
    if kind == "uniform_01":
        return rng.random(size=(n, d))
    raise ValueError(kind)


def make_rhs(n: int, nrhs: int, seed: int) -> np.ndarray:
    """N x nrhs float64, column-major (Fortran order), b ~ N(0,1).

    Drawn from its own generator (seed + 10_000) so the points do not depend on nrhs.
    """
    rng = np.random.default_rng(seed + 10_000)
    return np.asfortranarray(rng.standard_normal(size=(n, nrhs)))


def residual_rows(n: int, seed: int, count: int = 4096) -> np.ndarray:
    """Rows used for the sampled direct-sum residual (all rows when n <= count)."""
    if n <= count:
        return np.arange(n, dtype=np.int64)
    rng = np.random.default_rng(seed + 20_000)
    return np.sort(rng.choice(n, size=count, replace=False)).astype(np.int64)


def make(cfg: Workload, n: int | None = None, nrhs: int | None = None):
    """(points, B) for a config, optionally at a reduced N (uniform kinds only)."""
    n = cfg.n if n is None else n
    nrhs = cfg.nrhs if nrhs is None else nrhs
    pts = make_points(cfg.points, n, cfg.d, cfg.seed)
    return pts, make_rhs(n, nrhs, cfg.seed)


def small_problem(d=2, n=2048, kind="uniform_pm1", seed=7, nrhs=1):
    """Small seeded problems used by tests (ragged leaves, several tiles)."""
    return make_points(kind, n, d, seed), make_rhs(n, nrhs, seed)
