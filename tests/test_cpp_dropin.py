"""The C++ drop-in (include/tslb -> include/tslb_b200/tslb.hpp over the C-ABI).

CPU: a reference-style driver (tests/cpp/dropin_demo.cpp) compiles against the
drop-in; where /root/reference exists, the reference's OWN unit suites
(proj/tests/unit_*.cpp) compile unchanged against it (oracle/Makefile,
target dropin-tests; binaries land in oracle/_ref/ and travel to the GPU box).
GPU: both run on the device and must pass.
"""
import glob
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2304_06437_b200")
REF_TESTS = "/root/reference/proj/tests"


def _compile_demo(out):
    from paper_2304_06437_b200 import build
    build.build()
    cmd = ["g++", "-std=gnu++20", "-O2", f"-I{ROOT}/include", f"-I{ROOT}/oracle/shim",
           os.path.join(ROOT, "tests", "cpp", "dropin_demo.cpp"), "-o", out, f"-L{LIBDIR}", "-ltslb_cuda",
           f"-Wl,-rpath,{LIBDIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def test_dropin_demo_compiles(tmp_path):
    _compile_demo(str(tmp_path / "dropin_demo"))


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tests not present")
def test_reference_suites_compile_against_dropin():
    from paper_2304_06437_b200 import build
    build.build()
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "dropin-tests", "ref-tests",
                        "dropin-acceptance"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tests not present")
def test_reference_suites_pass_on_reference_headers():
    """Sanity of the doctest / Eigen shims: the suites pass on the reference."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref-tests"], check=True)
    for exe in sorted(glob.glob(os.path.join(ROOT, "oracle", "_ref", "ref_unit_*"))):
        r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, (exe, r.stdout[-2000:], r.stderr[-2000:])


@pytest.mark.gpu
def test_dropin_demo_runs_on_gpu(tmp_path, gpu):
    out = str(tmp_path / "dropin_demo")
    _compile_demo(out)
    r = subprocess.run([out], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["unit_lattice_fields", "unit_collision_stream", "unit_boundary",
                                   "unit_multicomponent", "unit_analysis_bench", "unit_config_io"])
def test_reference_unit_suite_passes_against_dropin(gpu, suite):
    """The reference's own unit suite, compiled unchanged against the B200
    drop-in, passes on the device."""
    exe = os.path.join(ROOT, "oracle", "_ref", f"dropin_{suite}")
    if not os.path.exists(exe):
        pytest.skip("drop-in suite binaries are built where /root/reference exists (make -C oracle dropin-tests)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:])
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])


@pytest.mark.gpu
def test_reference_acceptance_gate_passes_against_dropin(gpu):
    """The reference's acceptance gate (proj/tests/acceptance.cpp, every check
    prints PASS/FAIL, exit status = failures), compiled unchanged against the
    B200 drop-in, passes on the device."""
    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_acceptance")
    if not os.path.exists(exe):
        pytest.skip("built where /root/reference exists (make -C oracle dropin-acceptance)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1500)
    print(r.stdout[-5000:])
    assert r.returncode == 0, (r.stdout[-5000:], r.stderr[-3000:])
