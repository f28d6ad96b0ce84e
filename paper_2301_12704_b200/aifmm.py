"""Thin Python binding of libaifmm.so (include/aifmm.h): argument marshalling only.

Every step of build / factor / solve runs in the library's sm_100a kernels; torch is used
for device memory only.  There is no CPU fallback: importing this module without the
built library, or calling it without a CUDA device, raises.
"""
from __future__ import annotations

import contextlib
import ctypes
import os
import shutil
import tempfile
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libaifmm.so")

ERRORS = {
    -1: "EINVALID_ARG", -2: "ENONFINITE", -3: "ECOINCIDENT", -4: "ESINGULAR_SKELETON",
    -5: "ESINGULAR_PIVOT", -6: "ESTATE", -7: "ECUDA", -8: "ENCCL", -9: "EOOM",
}
SYMBOLS = ["aifmm_build", "aifmm_set_compression_tol", "aifmm_factor", "aifmm_solve",
           "aifmm_solve_host", "aifmm_free", "aifmm_last_error", "aifmm_set_stream",
           "aifmm_get_tree", "aifmm_get_level_offsets", "aifmm_get_lists", "aifmm_get_colours",
           "aifmm_get_ranks", "aifmm_get_skeletons", "aifmm_stats", "aifmm_reset_counters", "aifmm_set_timing",
           "aifmm_debug_inverse", "aifmm_debug_inverse_batch", "aifmm_debug_tri_root", "aifmm_matvec_build", "aifmm_matvec", "aifmm_gmres",
           "aifmm_residual", "aifmm_set_algorithm", "aifmm_dist_unique_id", "aifmm_dist_init",
           "aifmm_dist_init_local", "aifmm_dist_finalize", "aifmm_get_owners"]
STAT_NAMES = ["build_ms", "factor_ms", "solve_ms", "levels", "top_size", "factor_flops",
              "schur_flops", "schur_ms", "launches", "compressions", "max_rank", "device_bytes",
              "schur_bytes", "schur_launches", "solve_bytes", "host_syncs",
              "pivot_ms", "pivot_flops", "pivot_bytes", "tri_ms", "tri_flops", "tri_bytes",
              "pqr_ms", "pqr_flops", "pqr_bytes", "redir_ms", "redir_flops", "redir_bytes",
              "mult_ms", "mult_flops", "mult_bytes", "proj_ms", "proj_flops", "proj_bytes",
              "fresh_ms", "fresh_flops", "fresh_bytes", "orth_ms", "orth_flops", "orth_bytes",
              "dist_bytes", "dist_exchanges"]


class AIFMMError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


_lib = None
_tls = threading.local()   # per-thread library instance (in-process multi-rank validation)


def load(path: str = LIB_PATH):
    """Load libaifmm.so (raises if it has not been built).  Inside `use(lib)` the calling
    thread's instance is returned instead."""
    global _lib
    inst = getattr(_tls, "lib", None)
    if inst is not None:
        return inst
    if _lib is not None:
        return _lib
    _lib = _open(path)
    return _lib


def load_copy(rank: int):
    """A separate instance of the library (its own context, pools and stream): a private copy
    of libaifmm.so loaded RTLD_LOCAL.  Used to run `world` ranks of the distributed
    factorization in one process on one GPU (aifmm_dist_init_local), one host thread each."""
    load()
    d = tempfile.mkdtemp(prefix="aifmm_rank")
    path = os.path.join(d, f"libaifmm_rank{rank}.so")
    shutil.copyfile(LIB_PATH, path)
    return _open(path)


@contextlib.contextmanager
def use(lib):
    """Route this thread's calls of this module to `lib` (from load_copy)."""
    old = getattr(_tls, "lib", None)
    _tls.lib = lib
    try:
        yield lib
    finally:
        _tls.lib = old


def _open(path: str):
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path, mode=os.RTLD_LOCAL | os.RTLD_NOW)
    P, I, D, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64
    lib.aifmm_build.argtypes = [P, I64, I, I, P, I, D]
    lib.aifmm_set_compression_tol.argtypes = [D]
    lib.aifmm_factor.argtypes = []
    lib.aifmm_solve.argtypes = [P, I]
    lib.aifmm_solve_host.argtypes = [P, I]
    lib.aifmm_free.restype = None
    lib.aifmm_last_error.restype = ctypes.c_char_p
    lib.aifmm_set_stream.argtypes = [P]
    lib.aifmm_get_tree.argtypes = [P, P]
    lib.aifmm_get_level_offsets.argtypes = [I, P]
    lib.aifmm_get_lists.argtypes = [I, P, P, P, P]
    lib.aifmm_get_colours.argtypes = [I, P]
    lib.aifmm_get_ranks.argtypes = [I, I, P]
    lib.aifmm_get_skeletons.argtypes = [I, P, P, P]
    lib.aifmm_stats.argtypes = [P]
    lib.aifmm_set_timing.argtypes = [I]
    lib.aifmm_debug_inverse.argtypes = [P, I, I]
    lib.aifmm_debug_tri_root.argtypes = [P, I, I, I, P]
    lib.aifmm_debug_inverse_batch.argtypes = [P, I, I, I]
    lib.aifmm_matvec_build.argtypes = [D]
    lib.aifmm_matvec.argtypes = [P, P, I]
    lib.aifmm_gmres.argtypes = [P, P, I, D, I, I, P, P]
    lib.aifmm_residual.argtypes = [P, P, I, P, I64, P]
    lib.aifmm_set_algorithm.argtypes = [I]
    lib.aifmm_dist_unique_id.argtypes = [P]
    lib.aifmm_dist_init.argtypes = [I, I, P, I]
    lib.aifmm_dist_init_local.argtypes = [I, I, P, I]
    lib.aifmm_dist_finalize.argtypes = []
    lib.aifmm_get_owners.argtypes = [I, P]
    lib.bound_stream = None
    return lib


def _check(rc):
    if rc != 0:
        raise AIFMMError(rc, load().aifmm_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _bind_stream():
    """Run the library on torch's current CUDA stream, so that the tensors this module prepares
    (.to / .contiguous / .clone on that stream) are complete before the library reads them and
    the library's results are ordered before torch's later work (no cross-stream race)."""
    import torch
    lib = load()
    s = torch.cuda.current_stream().cuda_stream
    if s != lib.bound_stream:
        _check(lib.aifmm_set_stream(ctypes.c_void_p(s)))
        lib.bound_stream = s


def build(points, kernel_id: int, kparams, leaf_size: int, tol: float):
    """points: torch.cuda float64 tensor (n, d), any layout (made contiguous)."""
    import torch
    lib = load()
    if not (isinstance(points, torch.Tensor) and points.is_cuda):
        raise TypeError("points must be a CUDA tensor (device memory)")
    _bind_stream()
    pts = points.to(torch.float64).contiguous()
    kp = np.asarray(kparams, dtype=np.float64)
    _check(lib.aifmm_build(ctypes.c_void_p(pts.data_ptr()), pts.shape[0], pts.shape[1], int(kernel_id),
                           _ptr(kp), int(leaf_size), float(tol)))


def set_compression_tol(tol_c: float):
    _check(load().aifmm_set_compression_tol(float(tol_c)))


def set_algorithm(alg: int):
    """3 = Algorithm 3 (deferred compression, default), 2 = Algorithm 2 (compress on creation)."""
    _check(load().aifmm_set_algorithm(int(alg)))


def factor():
    _bind_stream()
    _check(load().aifmm_factor())


def solve(B):
    """B: torch.cuda float64 (n,) or (n, nrhs). Returns X with the same shape (new tensor)."""
    import torch
    lib = load()
    one = B.dim() == 1
    Bm = B[:, None] if one else B
    _bind_stream()
    # (nrhs, n) row-major == (n, nrhs) column-major; always a fresh buffer (the library solves in
    # place, and for one column .t().contiguous() would alias the caller's tensor)
    Bc = Bm.to(torch.float64).t().contiguous().clone()
    _check(lib.aifmm_solve(ctypes.c_void_p(Bc.data_ptr()), Bc.shape[0]))
    X = Bc.t()
    return X[:, 0] if one else X


def solve_device_ptr(ptr: int, nrhs: int):
    """In-place solve of a column-major n x nrhs device buffer given by its address."""
    _bind_stream()
    _check(load().aifmm_solve(ctypes.c_void_p(ptr), int(nrhs)))


def solve_host(B: np.ndarray) -> np.ndarray:
    """End-to-end path: host B (n,) or (n, nrhs) -> host X (copies inside the library)."""
    lib = load()
    one = B.ndim == 1
    Bf = np.asfortranarray(np.array(B[:, None] if one else B, dtype=np.float64))
    _check(lib.aifmm_solve_host(_ptr(Bf), Bf.shape[1]))
    return Bf[:, 0] if one else Bf


def free():
    load().aifmm_free()


def get_tree(n: int):
    lib = load()
    perm = np.zeros(n, dtype=np.int64)
    L = ctypes.c_int(0)
    _check(lib.aifmm_get_tree(_ptr(perm), ctypes.byref(L)))
    return perm, L.value


def get_level_offsets(level: int, d: int):
    off = np.zeros((1 << (d * level)) + 1, dtype=np.int64)
    _check(load().aifmm_get_level_offsets(level, _ptr(off)))
    return off


def get_lists(level: int, d: int):
    lib = load()
    nb = 1 << (d * level)
    nptr = np.zeros(nb + 1, dtype=np.int32)
    iptr = np.zeros(nb + 1, dtype=np.int32)
    _check(lib.aifmm_get_lists(level, _ptr(nptr), None, _ptr(iptr), None))
    nidx = np.zeros(max(int(nptr[-1]), 1), dtype=np.int32)
    iidx = np.zeros(max(int(iptr[-1]), 1), dtype=np.int32)
    _check(lib.aifmm_get_lists(level, _ptr(nptr), _ptr(nidx), _ptr(iptr), _ptr(iidx)))
    return nptr, nidx[:nptr[-1]], iptr, iidx[:iptr[-1]]


def get_colours(level: int, d: int):
    col = np.zeros(1 << (d * level), dtype=np.int32)
    _check(load().aifmm_get_colours(level, _ptr(col)))
    return col


def get_ranks(level: int, d: int, which: int = 0):
    r = np.zeros(1 << (d * level), dtype=np.int32)
    _check(load().aifmm_get_ranks(level, which, _ptr(r)))
    return r


def get_skeletons(level: int, d: int):
    """(sk_ptr, sk_idx, fp_idx): NNCA skeleton rows and far pivots per box (tree-order indices)."""
    lib = load()
    ptr = np.zeros((1 << (d * level)) + 1, dtype=np.int32)
    _check(lib.aifmm_get_skeletons(level, _ptr(ptr), None, None))
    sk = np.zeros(max(int(ptr[-1]), 1), dtype=np.int32)
    fp = np.zeros(max(int(ptr[-1]), 1), dtype=np.int32)
    _check(lib.aifmm_get_skeletons(level, _ptr(ptr), _ptr(sk), _ptr(fp)))
    return ptr, sk[:ptr[-1]], fp[:ptr[-1]]


def stats() -> dict:
    out = np.zeros(len(STAT_NAMES), dtype=np.float64)
    _check(load().aifmm_stats(_ptr(out)))
    return dict(zip(STAT_NAMES, out.tolist()))


def reset_counters():
    _check(load().aifmm_reset_counters())


def set_timing(on: bool):
    _check(load().aifmm_set_timing(1 if on else 0))


def set_stream(stream_ptr: int):
    lib = load()
    _check(lib.aifmm_set_stream(ctypes.c_void_p(stream_ptr)))
    lib.bound_stream = stream_ptr


def debug_inverse(M):
    """In-place GPU inverse of a square CUDA float64 tensor (test hook); returns the inverse."""
    import torch
    _bind_stream()
    Mc = M.to(torch.float64).t().contiguous()   # column-major storage of M
    _check(load().aifmm_debug_inverse(ctypes.c_void_p(Mc.data_ptr()), Mc.shape[0], Mc.shape[0]))
    return Mc.t()


def debug_inverse_batch(M, path: int = 0):
    """In-place GPU inverses of a (batch, n, n) CUDA float64 tensor (test hook; path 0 automatic,
    1 panel + GEMM launches, 2 fused one-CTA-per-matrix kernel).  Returns the inverses."""
    import torch
    b, n, _ = M.shape
    _bind_stream()
    Mc = M.to(torch.float64).transpose(1, 2).contiguous()   # column-major storage per matrix
    _check(load().aifmm_debug_inverse_batch(ctypes.c_void_p(Mc.data_ptr()), n, b, int(path)))
    return Mc.transpose(1, 2)


def debug_tri_root(A):
    """R^T of the Householder / TSQR factorisation of each matrix of a (batch, n, m) CUDA float64
    tensor (test hook; R unique up to row signs).  Returns (batch, m, min(n, m))."""
    import torch
    b, n, m = A.shape
    _bind_stream()
    Ac = A.to(torch.float64).transpose(1, 2).contiguous()   # column-major storage per matrix
    r = min(n, m)
    M = torch.empty((b, r, m), dtype=torch.float64, device=A.device)
    _check(load().aifmm_debug_tri_root(ctypes.c_void_p(Ac.data_ptr()), n, m, b, ctypes.c_void_p(M.data_ptr())))
    return M.transpose(1, 2)


def residual(X, B, rows=None) -> float:
    """||A X - B||_F / ||B||_F over `rows` (user indices; all rows if None) by exact direct sum on
    the GPU (row a9, verification).  X, B: torch.cuda float64 (N,) or (N, nrhs), user order."""
    import torch
    _bind_stream()
    Xm = X[:, None] if X.dim() == 1 else X
    Bm = B[:, None] if B.dim() == 1 else B
    if Xm.shape != Bm.shape:
        raise ValueError("X and B shapes differ")
    Xf = Xm.to(torch.float64).t().contiguous()
    Bf = Bm.to(torch.float64).t().contiguous()
    r = None if rows is None else np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    out = ctypes.c_double(0.0)
    _check(load().aifmm_residual(ctypes.c_void_p(Xf.data_ptr()), ctypes.c_void_p(Bf.data_ptr()), int(Xf.shape[0]),
                                 None if r is None else _ptr(r), 0 if r is None else int(r.size), ctypes.byref(out)))
    return out.value


def matvec_build(tol: float):
    """Second NNCA at the matvec tolerance (row a8); requires build()."""
    _bind_stream()
    _check(load().aifmm_matvec_build(float(tol)))


def matvec(X):
    """Y = A_H2 X for a torch.cuda float64 tensor X (N,) or (N, nrhs); returns a new tensor."""
    import torch
    one = X.dim() == 1
    Xm = X[:, None] if one else X
    _bind_stream()
    Xf = Xm.to(torch.float64).t().contiguous()      # (nrhs, N) row-major == N x nrhs column-major
    Yf = torch.empty_like(Xf)
    _check(load().aifmm_matvec(ctypes.c_void_p(Xf.data_ptr()), ctypes.c_void_p(Yf.data_ptr()), int(Xf.shape[0])))
    Y = Yf.t()
    return Y[:, 0].contiguous() if one else Y.contiguous()


PRECOND = {False: 0, True: 1, None: 0, 0: 0, 1: 1, 2: 2, "none": 0, "aifmm": 1, "block_diagonal": 2}


def gmres(b, restart: int = 30, rtol: float = 1e-10, maxit: int = 1000, precond=True):
    """GMRES(restart) with the H2 matvec; right preconditioner: True / 1 / "aifmm" the AIFMM
    factor, 2 / "block_diagonal" the leaf block-diagonal inverse, False / 0 / "none" none.
    b: torch.cuda float64 (N,).  Returns (x, iterations, relative residual)."""
    import torch
    if not (isinstance(b, torch.Tensor) and b.is_cuda and b.dim() == 1):
        raise TypeError("b must be a 1-D CUDA tensor")
    _bind_stream()
    bc = b.to(torch.float64).contiguous()
    x = torch.empty_like(bc)
    it = ctypes.c_int(0)
    rr = ctypes.c_double(0.0)
    _check(load().aifmm_gmres(ctypes.c_void_p(bc.data_ptr()), ctypes.c_void_p(x.data_ptr()), int(restart), float(rtol),
                              int(maxit), PRECOND[precond], ctypes.byref(it), ctypes.byref(rr)))
    return x, it.value, rr.value


# ---------------------------------------------------------------- SURVEY §8(e), multi-GPU
def dist_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for dist_init; create it on one rank and send it to
    the others (torch.distributed.broadcast_object_list)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().aifmm_dist_unique_id(buf))
    return buf.raw


def dist_init(rank: int, world: int, unique_id: bytes, level_p: int = -1):
    """Join the NCCL communicator: the next factorizations split their work by subtree
    (include/aifmm.h).  Every rank must then call build/factor with the same arguments."""
    _bind_stream()
    uid = ctypes.create_string_buffer(bytes(unique_id), 128)
    _check(load().aifmm_dist_init(int(rank), int(world), uid, int(level_p)))


def local_shared():
    """Zeroed host rendezvous block for dist_init_local (keep a reference while in use)."""
    return ctypes.create_string_buffer(4096)


def dist_init_local(rank: int, world: int, shared, level_p: int = -1):
    """In-process transport (validation on one GPU): `world` library instances (load_copy),
    one host thread each, all passing the same `shared` block."""
    _bind_stream()
    _check(load().aifmm_dist_init_local(int(rank), int(world), ctypes.cast(shared, ctypes.c_void_p), int(level_p)))


def dist_finalize():
    _check(load().aifmm_dist_finalize())


def get_owners(level: int, d: int):
    o = np.zeros(1 << (d * level), dtype=np.int32)
    _check(load().aifmm_get_owners(level, _ptr(o)))
    return o
