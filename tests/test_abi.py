"""CPU checks of the C-ABI boundary: the library builds, loads and exports every symbol that
include/aifmm.h declares; the Python binding marshals the same names; the product package
never imports the oracle (no CPU fallback)."""
import os
import re
import subprocess

import pytest

from paper_2301_12704_b200 import aifmm as binding


def _declared(root):
    src = open(os.path.join(root, "include", "aifmm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(aifmm_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(root):
    from paper_2301_12704_b200.build import build_library
    lib = build_library()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (aifmm_[a-z_]+)", out))
    declared = _declared(root)
    assert len(declared) >= 16
    missing = [s for s in declared if s not in exported]
    assert not missing, missing


def test_binding_names_match_header(root):
    assert sorted(binding.SYMBOLS) == _declared(root)
    lib = binding.load()
    for s in binding.SYMBOLS:
        assert hasattr(lib, s)


def test_sm100a_dmma_in_sass():
    from paper_2301_12704_b200.build import build_library
    lib = build_library()
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "DMMA" in sass              # FP64 tensor-core GEMM (mma.sync f64 -> DMMA.8x8x4)
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", lib], capture_output=True, text=True).stdout or \
        "sm_100" in sass


def test_product_path_never_imports_oracle(root):
    pkg = os.path.join(root, "paper_2301_12704_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, flags=re.M), f


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(ImportError):
        binding.load.__wrapped__(str(tmp_path / "nope.so")) if hasattr(binding.load, "__wrapped__") else \
            _load_elsewhere(str(tmp_path / "nope.so"))


def _load_elsewhere(path):
    saved = binding._lib
    binding._lib = None
    try:
        binding.load(path)
    finally:
        binding._lib = saved


def test_private_copies_share_no_state():
    """The in-process multi-rank validation (tests/test_gpu_dist.py) loads private copies of the
    library: no STB_GNU_UNIQUE symbol (function-local statics such as the device chunk cache)
    may be merged across copies, and NCCL is resolved at run time (no link dependency)."""
    from paper_2301_12704_b200.build import build_library
    lib = build_library()
    out = subprocess.run(["nm", "-D", lib], capture_output=True, text=True, check=True).stdout
    assert not re.search(r" u ", out), "GNU_UNIQUE symbols present (build without -fno-gnu-unique?)"
    ldd = subprocess.run(["ldd", lib], capture_output=True, text=True).stdout
    assert "nccl" not in ldd
    a, b = binding.load(), binding.load_copy(0)
    assert a is not b and hasattr(b, "aifmm_dist_init_local")
