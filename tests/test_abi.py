"""C-ABI boundary: the library builds, loads, and exports every declared symbol."""

import ctypes
import os
import re

import pytest

from paper_1007_3753_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ell1_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ell1_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_bound_symbols():
    assert set(declared_symbols()) == set(_lib.EXPORTS)


def test_library_loads_and_exports_everything():
    assert os.path.exists(_lib.LIB_PATH), "run python -m paper_1007_3753_b200.build"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_version_string():
    assert b"sm_100a" in _lib.lib().ell1_version()


def test_struct_sizes_match_header():
    assert ctypes.sizeof(_lib.State) == 256
    assert ctypes.sizeof(_lib.Dict) == 48
    assert ctypes.sizeof(_lib.FistaOpts) == 56


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1007_3753_b200.exceptions import DeviceError
    from paper_1007_3753_b200.model import ProblemInstance, SolverConfig
    from paper_1007_3753_b200.shrinkage import fista_solve
    import numpy as np
    P = ProblemInstance(np.eye(3), np.ones(3))
    with pytest.raises(DeviceError):
        fista_solve(P, SolverConfig(lam=0.1))


def test_library_has_no_blas_dependency():
    """Every dictionary product is the library's own kernel (tcgen05 3xTF32 for
    fp32, DMMA for fp64): libell1b200.so links no cuBLAS / cuSOLVER and
    references none of their symbols."""
    import subprocess
    from paper_1007_3753_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    dyn = subprocess.run(["readelf", "-d", _lib.LIB_PATH], capture_output=True, text=True).stdout
    needed = [ln for ln in dyn.splitlines() if "NEEDED" in ln]
    assert needed and not any("cublas" in ln or "cusolver" in ln for ln in needed), needed
    syms = subprocess.run(["nm", "-D", "--undefined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "cublas" not in syms and "cusolver" not in syms
