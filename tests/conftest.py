"""pytest configuration: the `gpu` marker and shared fixtures.

`-m "not gpu"` (CPU, here): oracle vs reference/golden, host logic, the
C-ABI library loads and exports every declared symbol, gloo multi-rank tests.
`-m gpu` (a B200): parity of the CUDA path against the oracle via the C-ABI.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtslb_cuda.so")


@pytest.fixture(scope="session")
def oracle_port():
    from oracle import oracle as O
    if not os.path.exists(O.PORT_SO):
        O.build(ref=False)
    return O.Oracle("port")


@pytest.fixture(scope="session")
def oracle_ref():
    from oracle import oracle as O
    if not os.path.exists(O.REF_SO):
        if os.path.exists(os.path.join(O.REF_INC, "tslb", "kernels.hpp")):
            O.build(ref=True)
        else:
            pytest.skip("reference build oracle/_ref/libtslb_ref.so not present")
    return O.Oracle("ref")


@pytest.fixture(scope="session")
def gpu():
    """The product library on a real device; fails loudly if either is missing."""
    from paper_2304_06437_b200 import _lib, build
    if not os.path.exists(_lib.LIB_PATH):
        build.build()
    lib = _lib.load()
    import ctypes
    n = ctypes.c_int()
    _lib.check(lib.tslb_cuda_device_count(ctypes.byref(n)))
    assert n.value >= 1, "no CUDA device visible"
    return lib
