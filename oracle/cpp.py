"""ctypes shim over the serial C++ oracle (oracle/cpp/aifmm_oracle.cpp; test infrastructure only).

The C++ oracle is the north_star's "plain serial CPU C++ implementation of tree, NNCA, AIFMM
factorization and solve": plain dense loops (no BLAS / LAPACK), the same algorithm and
readings as the numpy oracle (oracle/factor.py etc.), no code shared with the CUDA path.
`threads > 1` parallelises independent boxes with OpenMP; results are bit-identical to
`threads = 1` (tested).  Only tests/, bench.py's cpu_baseline leg and tools/ may use it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "cpp", "aifmm_oracle.cpp")
LIB = os.path.join(_HERE, "cpp", "liboracle.so")
# /usr/bin/g++ ships libgomp (an image-level CXX may point at a gcc without OpenMP)
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else os.environ.get("CXX", "g++")
# x86-64-v3 (AVX2) so the library built here also runs on the GPU box's host; no FMA
# contraction and no fast-math: IEEE evaluation order as written
FLAGS = ["-O3", "-march=x86-64-v3", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC", "-std=c++17"]

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run([CXX, *FLAGS, SRC, "-o", LIB + ".tmp"], check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P, I, D, LL = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_longlong
        lib.oc_build.restype = P
        lib.oc_build.argtypes = [P, LL, I, I, P, I, D, D, I, P]
        lib.oc_factor.argtypes = [P]
        lib.oc_solve.argtypes = [P, P, I, P]
        lib.oc_free.argtypes = [P]
        lib.oc_free.restype = None
        lib.oc_depth.argtypes = [P]
        lib.oc_perm.argtypes = [P, P]
        lib.oc_offsets.argtypes = [P, I, P]
        lib.oc_lists.argtypes = [P, I, P, P, P, P]
        lib.oc_colours.argtypes = [P, I, P]
        lib.oc_ranks.argtypes = [P, I, I, P]
        lib.oc_skeleton.argtypes = [P, I, I, P]
        lib.oc_stats.argtypes = [P, P]
        lib.oc_set_algorithm.argtypes = [P, I]
        lib.oc_last_error.restype = ctypes.c_char_p
        _lib = lib
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{code}: {msg}")
        self.code = code


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class CppAIFMM:
    """build (tree, lists, colours, NNCA) in the constructor, then factor() and solve(B)."""

    def __init__(self, points, kernel_id, kparams, leaf_size, tol, tol_c=None, threads=1, algorithm=3):
        lib = load()
        self.points = np.ascontiguousarray(points, dtype=np.float64)
        self.n, self.d = self.points.shape
        kp = np.asarray(kparams, dtype=np.float64)
        err = ctypes.c_int(0)
        self._h = lib.oc_build(_p(self.points), self.n, self.d, int(kernel_id), _p(kp), int(leaf_size), float(tol),
                               -1.0 if tol_c is None else float(tol_c), int(threads), ctypes.byref(err))
        if not self._h:
            raise OracleError(err.value, lib.oc_last_error().decode())
        self.L = lib.oc_depth(self._h)
        if lib.oc_set_algorithm(self._h, int(algorithm)):
            raise ValueError("algorithm must be 2 or 3")

    def __del__(self):
        if getattr(self, "_h", None):
            load().oc_free(self._h)
            self._h = None

    def factor(self):
        rc = load().oc_factor(self._h)
        if rc:
            raise OracleError(rc, load().oc_last_error().decode())
        return self

    def solve(self, B):
        B = np.asarray(B, dtype=np.float64)
        one = B.ndim == 1
        Bf = np.asfortranarray(B[:, None] if one else B)
        X = np.zeros_like(Bf, order="F")
        rc = load().oc_solve(self._h, _p(Bf), Bf.shape[1], _p(X))
        if rc:
            raise OracleError(rc, load().oc_last_error().decode())
        return X[:, 0] if one else X

    # integer outputs (same layout as the C-ABI's introspection)
    def perm(self):
        out = np.zeros(self.n, dtype=np.int64)
        load().oc_perm(self._h, _p(out))
        return out

    def offsets(self, l):
        out = np.zeros((1 << (self.d * l)) + 1, dtype=np.int64)
        load().oc_offsets(self._h, l, _p(out))
        return out

    def lists(self, l):
        nb = 1 << (self.d * l)
        nptr = np.zeros(nb + 1, dtype=np.int32)
        iptr = np.zeros(nb + 1, dtype=np.int32)
        load().oc_lists(self._h, l, _p(nptr), None, _p(iptr), None)
        nidx = np.zeros(max(int(nptr[-1]), 1), dtype=np.int32)
        iidx = np.zeros(max(int(iptr[-1]), 1), dtype=np.int32)
        load().oc_lists(self._h, l, _p(nptr), _p(nidx), _p(iptr), _p(iidx))
        return nptr, nidx[:nptr[-1]], iptr, iidx[:iptr[-1]]

    def colours(self, l):
        out = np.zeros(1 << (self.d * l), dtype=np.int32)
        load().oc_colours(self._h, l, _p(out))
        return out

    def ranks(self, l, which=0):
        out = np.zeros(1 << (self.d * l), dtype=np.int32)
        load().oc_ranks(self._h, l, which, _p(out))
        return out

    def skeleton(self, l, b):
        k = load().oc_skeleton(self._h, l, b, None)
        out = np.zeros(k, dtype=np.int64)
        if k:
            load().oc_skeleton(self._h, l, b, _p(out))
        return out

    def stats(self):
        out = np.zeros(5)
        load().oc_stats(self._h, _p(out))
        return dict(zip(["build_s", "factor_s", "solve_s", "compressions", "top_size"], out.tolist()))
