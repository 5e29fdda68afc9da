"""The peer-memory slab transport (tslb_cuda_ipc_handle /
tslb_cuda_attach_ipc): M slabs whose boundary planes are copied straight
into the neighbours' ghost buffers (CUDA IPC mappings, parity double
buffering, flag words published with system-scope release stores). Checked
bit for bit against the oracle's undivided domain -- with one process whose
faces wrap onto itself, and with 2 and 3 separate processes (one rank each,
all on this device: the same cross-process mapping and flags as one process
per GPU)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from paper_2304_06437_b200 import _lib
from paper_2304_06437_b200 import tslb as T

from helpers import assert_bitwise, spec_of, zwalls_3d

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("lzb", ["", "2"])
def test_ipc_self_exchange_equals_periodic_box(gpu, dtype, lzb, monkeypatch):
    """One slab [0, nzl) of a 2*nzl box whose up and down neighbour is itself
    (its own handle on both faces): every step copies its boundary planes into
    its own ghost buffers of the next parity and waits on its own flags --
    exactly a periodic box of height nzl. f is materialised from the ghost
    moments mid-run and the run continues from it."""
    monkeypatch.setenv("TSLB_LZ", "2")
    if lzb:
        monkeypatch.setenv("TSLB_LZB", lzb)
    lat, nx, ny, nzl = "d3q19", 32, 16, 8
    f0 = O.random_state(lat, (nx, ny, nzl), 5, dtype)
    spec = spec_of(O.periodic())
    ref = T.DeviceSolver(lat, T.GridDims(nx, ny, nzl), 1.2, spec, dtype)
    slab = T.DeviceSolver(lat, T.GridDims(nx, ny, 2 * nzl), 1.2, spec, dtype, 1, None, slab=(0, nzl))
    try:
        assert slab.schedule == "m"
        own = slab.ipc_handle()
        assert len(own) == T.DeviceSolver.IPC_HANDLE_BYTES
        slab.attach_ipc(own, own)
        with pytest.raises(_lib.TslbCudaError):
            slab.attach_ipc(own, own)  # (one transport per slab)
        for d in (ref, slab):
            d.upload_f(f0)
            d.step(3)
        assert_bitwise(slab.download_f(), ref.download_f(), "IPC self-exchange f(3)")
        for d in (ref, slab):
            d.step(4)
        assert_bitwise(slab.download_f(), ref.download_f(), "IPC self-exchange f(7)")
        for fld in ("rho", "mom", "pineq"):
            assert_bitwise(slab.download_field(fld), ref.download_field(fld), f"IPC self-exchange {fld}")
    finally:
        slab.close()
        ref.close()


def test_ipc_rejects_two_fluid_and_f1_steps(gpu):
    spec = spec_of(O.periodic())
    slab = T.DeviceSolver("d3q19", T.GridDims(32, 16, 16), 1.2, spec, np.float32, 1, None, slab=(0, 8))
    try:
        own = slab.ipc_handle()
        slab.attach_ipc(own, own)
        slab.set_schedule("f1")
        slab.init_analytic("taylor_green", 0.02)
        with pytest.raises(_lib.TslbCudaError):
            slab.step(1)
    finally:
        slab.close()


def run_ranks(tmp_path, parts, lat, dims, dtype, steps, mid, faces):
    env = dict(os.environ)
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "ipc_worker.py"), str(r), str(parts),
                               str(tmp_path), lat, *map(str, dims), "f32" if dtype == np.float32 else "f64",
                               str(steps), str(mid), faces], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(parts)]
    logs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(out.decode(errors="replace")[-3000:])
    for r, (p, log) in enumerate(zip(procs, logs)):
        assert p.returncode == 0, f"rank {r} failed:\n{log}"
    res = [np.load(os.path.join(tmp_path, f"out{r}.npz")) for r in range(parts)]
    cat = {k: np.concatenate([x[k] for x in res], axis=1) for k in ("f", "f_mid", "m")}
    return cat


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("lat,parts,faces", [("d3q19", 2, "periodic"), ("d3q19", 3, "periodic"),
                                             ("d3q19", 2, "zwalls"), ("d3q27", 2, "periodic")])
def test_ipc_processes_equal_oracle(gpu, oracle_port, tmp_path, lat, parts, faces, dtype):
    """`parts` processes, one z slab each, stepping over the peer-memory
    transport == fused_step on the undivided domain, bit for bit (f at the
    mid-run materialisation, f and the moment arrays at the end)."""
    dims, steps, mid = (32, 16, 12), 6, 2
    got = run_ranks(tmp_path, parts, lat, dims, dtype, steps, mid, faces)
    fc = O.periodic() if faces == "periodic" else zwalls_3d()
    f0 = O.random_state(lat, dims, 91, dtype)
    ref_mid = f0.copy()
    oracle_port.single_run(lat, dims, 1.25, fc, ref_mid, None, mid, 0)
    ref = ref_mid.copy()
    rmo = np.zeros((10, ref.shape[1]), dtype)
    oracle_port.single_run(lat, dims, 1.25, fc, ref, rmo, steps - mid, 0)
    assert_bitwise(got["f_mid"], ref_mid, f"IPC x{parts} f({mid})")
    assert_bitwise(got["f"], ref, f"IPC x{parts} f({steps})")
    assert_bitwise(got["m"], rmo, f"IPC x{parts} moments")


def test_bench_two_ranks_on_one_device_over_ipc(gpu, tmp_path):
    """`bench.py --gpus 2 --transport ipc` end to end on a one-GPU box
    (TSLB_BENCH_ONE_GPU=1: both ranks on device 0; the timing is meaningless,
    the launch, handle exchange, peer-memory halos and max-over-ranks report
    are the real N-rank path)."""
    import json
    root = os.path.dirname(HERE)
    env = dict(os.environ, TSLB_BENCH_ONE_GPU="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--transport", "ipc",
                        "--n", "64", "--steps", "4", "--warmup", "3"], env=env, capture_output=True, text=True,
                       timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert "peer-memory" in line["config"]["parallelism"]
    assert line["roofline"]["launches_per_step"].get("exchange", 0) > 0


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_ipc_self_exchange_masked(gpu, dtype, monkeypatch):
    """A masked M slab on the peer-memory transport (its own neighbour; masked
    slabs copy their boundary planes after the chunks instead of storing them
    from the kernel) equals the periodic masked box of the slab's height."""
    from helpers import random_solid
    monkeypatch.setenv("TSLB_LZ", "2")
    lat, nx, ny, nzl = "d3q19", 32, 16, 8
    mask = random_solid((nx, ny, nzl), 0.15, 9)
    f0 = O.random_state(lat, (nx, ny, nzl), 6, dtype, mask)
    spec = spec_of(O.periodic())
    ref = T.DeviceSolver(lat, T.GridDims(nx, ny, nzl), 1.2, spec, dtype, 1, mask)
    slab = T.DeviceSolver(lat, T.GridDims(nx, ny, 2 * nzl), 1.2, spec, dtype, 1, np.concatenate([mask, mask]),
                          slab=(0, nzl))
    try:
        assert slab.schedule == "m" and ref.schedule == "m"
        own = slab.ipc_handle()
        slab.attach_ipc(own, own)
        for d in (ref, slab):
            d.upload_f(f0)
            d.step(7)
        assert_bitwise(slab.download_f(), ref.download_f(), "masked IPC self-exchange f")
        for fld in ("rho", "mom", "pineq"):
            assert_bitwise(slab.download_field(fld), ref.download_field(fld), f"masked IPC self-exchange {fld}")
    finally:
        slab.close()
        ref.close()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_init_equilibrium_on_an_ipc_slab(gpu, oracle_port, dtype, monkeypatch):
    """tslb_cuda_init_equilibrium on a slab (rho, u of the local planes; the
    first step's moments come from the initialiser and go out by copy, every
    later exchange from the kernel epilogue) over the peer-memory transport
    == the oracle's initialize_regularized (Pi = 0) + fused_step."""
    monkeypatch.setenv("TSLB_LZB", "2")
    lat, nx, ny, nzl = "d3q19", 32, 8, 8
    n = nx * ny * nzl
    rng = np.random.default_rng(5)
    st = np.zeros((10, n))
    st[:4] = rng.uniform(-0.02, 0.02, (4, n))
    st[0] += 1.0
    st = st.astype(dtype)
    spec = spec_of(O.periodic())
    slab = T.DeviceSolver(lat, T.GridDims(nx, ny, 2 * nzl), 1.2, spec, dtype, 1, None, slab=(0, nzl))
    try:
        own = slab.ipc_handle()
        slab.attach_ipc(own, own)
        slab.init_equilibrium(np.ascontiguousarray(st[:4]))
        slab.step(6)
        fs = slab.download_f()
    finally:
        slab.close()
    fo = oracle_port.init_regularized(lat, (nx, ny, nzl), st)
    oracle_port.single_run(lat, (nx, ny, nzl), 1.2, O.periodic(), fo, None, 6, 0)
    assert_bitwise(fs, fo, "init_equilibrium IPC slab vs oracle f")
