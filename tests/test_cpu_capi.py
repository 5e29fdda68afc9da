"""CPU: the C-ABI library builds for sm_100a, loads, and exports every
symbol include/tslb_cuda.h declares (no compute calls without a GPU)."""
import ctypes
import os
import subprocess

from paper_2304_06437_b200 import _lib, build


def test_library_exports_every_declared_symbol():
    path = build.build()
    lib = ctypes.CDLL(path)
    names = _lib.header_symbols()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert _lib.load().tslb_cuda_abi_version() == 3


def test_library_is_sm100a_native():
    path = build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "k_streamcoll" in sass and "k_moments" in sass and "k_mstep" in sass and "STG" in sass


def test_no_cpu_fallback_without_device():
    """With no visible GPU every compute entry point reports an error."""
    import numpy as np
    import pytest
    from paper_2304_06437_b200 import tslb as T
    n = ctypes.c_int()
    if _lib.load().tslb_cuda_device_count(ctypes.byref(n)) == 0 and n.value > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(_lib.TslbCudaError):
        T.SingleFluidSim(T.D2Q9, T.GridDims(8, 8, 1), T.CollisionParams(1.0), T.BoundarySpec())
