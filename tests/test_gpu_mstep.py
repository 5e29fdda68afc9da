"""GPU parity of the moment-resident single-pass schedule (M, tslb_mstep.cu)
against the CPU oracle: f(N) (materialised from m(N-1)) and the moment
arrays m(N-1) must be bit-identical to fused_step run N times (kernels.hpp:
209-215), for double and float storage, every face combination of a box,
multiple z chunks per column (TSLB_LZ), graph replay, and every host-mirror
transition (download, upload, refresh, phase calls, math-mode switch)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2304_06437_b200 import _lib
from paper_2304_06437_b200 import tslb as T

from helpers import assert_bitwise, block_solid, corner_box_3d, random_solid, spec_of, zwalls_3d

pytestmark = pytest.mark.gpu

DT = [np.float64, np.float32]


def xwalls_3d():
    f = O.periodic()
    f[0] = ("moving", (0.0, 0.02, -0.01))
    f[1] = ("wall", (0, 0, 0))
    return f


def ylid_3d():
    f = O.periodic()
    f[2] = ("wall", (0, 0, 0))
    f[3] = ("moving", (0.05, 0.0, 0.01))
    return f


CASES = [
    ("periodic", (32, 8, 5), O.periodic()),
    ("periodic-nz1", (32, 8, 1), O.periodic()),
    ("periodic-wide", (64, 16, 11), O.periodic()),
    ("zwalls", (32, 16, 9), zwalls_3d()),
    ("zwalls-nz2", (32, 8, 2), zwalls_3d()),
    ("xwalls", (64, 8, 4), xwalls_3d()),
    ("ylid", (32, 16, 5), ylid_3d()),
    ("closed-box", (64, 8, 4), O.closed_box()),
    ("box-corners", (32, 16, 7), corner_box_3d()),
]


def _moments(dev, lat):
    L = T.lattice_of(lat)
    return np.concatenate([dev.download_field("rho")[None], dev.download_field("mom").reshape(L.dim, -1),
                           dev.download_field("pineq").reshape(L.npineq, -1)])


def _oracle(oracle_port, lat, dims, omega, faces, f0, steps):
    f = f0.copy()
    mo = np.zeros((O.moments_layout(lat), f.shape[1]), f.dtype)
    oracle_port.single_run(lat, dims, omega, faces, f, mo, steps, 0)
    return f, mo


@pytest.mark.parametrize("lz", ["", "3"])
@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("lat", ["d3q19", "d3q27"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_mstep_bitwise(gpu, oracle_port, case, lat, dtype, lz, monkeypatch):
    name, dims, faces = case
    if lz:
        monkeypatch.setenv("TSLB_LZ", lz)
    f0 = O.random_state(lat, dims, 11, dtype)
    steps = 5
    dev = T.DeviceSolver(lat, T.GridDims(*dims), 0.87, spec_of(faces), dtype)
    try:
        assert dev.schedule == "m", "M schedule should be the default for this box"
        dev.upload_f(f0)
        dev.step(steps)
        mg = _moments(dev, lat)
        fg = dev.download_f()
    finally:
        dev.close()
    fo, mo = _oracle(oracle_port, lat, dims, 0.87, faces, f0, steps)
    assert_bitwise(mg, mo, f"M {lat}/{name} moments m(N-1)")
    assert_bitwise(fg, fo, f"M {lat}/{name} f(N)")


@pytest.mark.parametrize("lat", ["d3q19", "d3q27"])
@pytest.mark.parametrize("case", [CASES[2], CASES[8]], ids=lambda c: c[0])
def test_mstep_f32_math_equals_f1(gpu, case, lat):
    """fp32 node arithmetic (opt-in): no oracle bits, but the two schedules
    perform the same float operations, so they must agree bit for bit."""
    name, dims, faces = case
    f0 = O.random_state(lat, dims, 5, np.float32)
    out = {}
    for sched in ("f1", "m"):
        dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.3, spec_of(faces), np.float32)
        try:
            dev.set_schedule(sched)
            dev.set_math(_lib.MATH_F32)
            dev.upload_f(f0)
            dev.step(6)
            out[sched] = (dev.download_f(), _moments(dev, lat))
        finally:
            dev.close()
    assert_bitwise(out["m"][0], out["f1"][0], f"f32 math {lat}/{name} f")
    assert_bitwise(out["m"][1], out["f1"][1], f"f32 math {lat}/{name} moments")


@pytest.mark.parametrize("dtype", DT)
def test_mstep_graph_replay_parity(gpu, oracle_port, dtype):
    """Small domains replay a captured graph of 32 M passes; odd step counts
    leave the ping-pong buffers swapped, which the next call must honour."""
    lat, dims, faces = "d3q19", (32, 16, 12), zwalls_3d()
    f0 = O.random_state(lat, dims, 3, dtype)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.15, spec_of(faces), dtype)
    try:
        dev.upload_f(f0)
        for n in (40, 33, 35, 64):
            dev.step(n)
        mg = _moments(dev, lat)
        fg = dev.download_f()
    finally:
        dev.close()
    fo, mo = _oracle(oracle_port, lat, dims, 1.15, faces, f0, 172)
    assert_bitwise(mg, mo, "graph M moments")
    assert_bitwise(fg, fo, "graph M f")


def test_mstep_host_mirror_transitions(gpu, oracle_port):
    """Every API that reads or replaces state while f is implicit."""
    lat, dims, faces, om = "d3q19", (32, 8, 6), corner_box_3d(), 1.4
    dt = np.float64
    f0 = O.random_state(lat, dims, 21, dt)
    ref = f0.copy()
    rmo = np.zeros((O.moments_layout(lat), ref.shape[1]), dt)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), om, spec_of(faces), dt)
    try:
        dev.upload_f(f0)
        # step, read f mid-run (materialise), keep stepping
        dev.step(3)
        oracle_port.single_run(lat, dims, om, faces, ref, rmo, 3, 0)
        assert_bitwise(dev.download_f(), ref, "f after 3")
        dev.step(4)
        oracle_port.single_run(lat, dims, om, faces, ref, rmo, 4, 0)
        assert_bitwise(_moments(dev, lat), rmo, "lagged moments after 7")
        # refresh_moments: moments of the current f
        dev.phase("refresh_moments")
        oracle_port.single_run(lat, dims, om, faces, ref, rmo, 1, 2)
        assert_bitwise(_moments(dev, lat), rmo, "refreshed moments")
        assert_bitwise(dev.download_f(), ref, "f after refresh")
        # step again from the stored-f state
        dev.step(2)
        oracle_port.single_run(lat, dims, om, faces, ref, rmo, 2, 0)
        # overwrite moments while f is implicit: the step that follows
        # recomputes them from f, as fused_step does
        junk = np.full_like(rmo[0], 7.0)
        dev.upload_field("rho", junk)
        dev.step(2)
        oracle_port.single_run(lat, dims, om, faces, ref, rmo, 2, 0)
        assert_bitwise(dev.download_f(), ref, "f after moment upload + steps")
        # phase calls on an implicit f
        dev.step(1)
        oracle_port.single_run(lat, dims, om, faces, ref, rmo, 1, 0)
        dev.phase("compute_moments")
        dev.phase("stream_collide")
        oracle_port.single_run(lat, dims, om, faces, ref, rmo, 1, 0)
        assert_bitwise(dev.download_f(), ref, "f after phase calls")
        # digest of an implicit f equals the digest of the stored one
        dev.step(2)
        oracle_port.single_run(lat, dims, om, faces, ref, rmo, 2, 0)
        d_implicit = dev.plane_digests()
        assert_bitwise(dev.download_f(), ref, "f after digest")
        assert np.array_equal(d_implicit, dev.plane_digests())
        # upload f while implicit: the next step starts from the upload
        f1 = O.random_state(lat, dims, 22, dt)
        dev.step(1)
        dev.upload_f(f1)
        dev.step(3)
        ref = f1.copy()
        oracle_port.single_run(lat, dims, om, faces, ref, rmo, 3, 0)
        assert_bitwise(dev.download_f(), ref, "f after re-upload")
        # switching schedules mid-run
        dev.step(2)
        dev.set_schedule("f1")
        dev.step(2)
        dev.set_schedule("m")
        dev.step(3)
        oracle_port.single_run(lat, dims, om, faces, ref, rmo, 7, 0)
        assert_bitwise(dev.download_f(), ref, "f across schedule switches")
        assert_bitwise(_moments(dev, lat), rmo, "moments across schedule switches")
    finally:
        dev.close()


def test_mstep_diagnostics_use_lagged_moments(gpu, oracle_port):
    lat, dims, faces = "d3q19", (32, 8, 4), O.periodic()
    f0 = O.random_state(lat, dims, 9, np.float64)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.2, spec_of(faces), np.float64)
    try:
        dev.upload_f(f0)
        dev.step(4)
        mass, mom = dev.totals()
        mg = _moments(dev, lat)
    finally:
        dev.close()
    fo, mo = _oracle(oracle_port, lat, dims, 1.2, faces, f0, 4)
    assert_bitwise(mg, mo, "moments")
    assert abs(mass - mo[0].sum()) <= 1e-12 * mo[0].size
    assert np.allclose(mom, mo[1:4].sum(1), rtol=0, atol=1e-12 * mo[0].size)


def test_schedule_rules(gpu):
    spec = spec_of(O.periodic())
    dev = T.DeviceSolver("d3q19", T.GridDims(30, 8, 4), 1.0, spec, np.float32)
    try:
        assert dev.schedule == "f1"
        with pytest.raises(RuntimeError):
            dev.set_schedule("m")
    finally:
        dev.close()
    dev = T.DeviceSolver("d2q9", T.GridDims(64, 64, 1), 1.0, spec, np.float32)
    try:
        assert dev.schedule == "m"  # the 2-D M kernel (tslb_mstep2d.cu)
    finally:
        dev.close()
    # 3-D rows of a multiple of 16 bytes tile partially: M
    for nx, dt in ((36, np.float32), (30, np.float64), (1000, np.float32)):
        dev = T.DeviceSolver("d3q19", T.GridDims(nx, 9, 3), 1.0, spec, dt)
        try:
            assert dev.schedule == "m", (nx, dt)
        finally:
            dev.close()


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("init", ["taylor_green", "shear", "rest"])
def test_mstep_device_init_without_f(gpu, init, dtype):
    """Under M the analytic initialiser stores m(0) instead of f(0) (the f
    buffer is allocated only when read): every observable equals the F1
    solver's, bit for bit -- f(0) on download before any step, the lagged
    moments, f(N) and m(N-1) after steps."""
    lat, dims, faces = "d3q19", (32, 16, 8), zwalls_3d()
    out = {}
    for sched in ("m", "f1"):
        dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.1, spec_of(faces), dtype)
        try:
            if sched == "f1":
                dev.set_schedule("f1")
            dev.init_analytic(init, 0.04)
            if sched == "m":  # two moment sets (20 arrays), no population buffer (19)
                assert dev.memory_bytes() < 30 * dims[0] * dims[1] * dims[2] * np.dtype(dtype).itemsize
            out[sched] = [dev.download_f(), _moments(dev, lat)]
            dev.step(4)
            out[sched] += [_moments(dev, lat), dev.download_f()]
            dev.init_analytic(init, 0.02)   # re-init after stepping
            dev.step(3)
            out[sched] += [dev.download_f()]
        finally:
            dev.close()
    for a, b, what in zip(out["m"], out["f1"], ["f(0)", "moments after init", "m(3)", "f(4)", "f(3) after re-init"]):
        assert_bitwise(a, b, f"M vs F1 {init}: {what}")


def test_mstep_lazy_f_memory(gpu):
    """A device-initialised M solver holds moments only until f is read."""
    dims = (64, 32, 16)
    dev = T.DeviceSolver("d3q19", T.GridDims(*dims), 1.2, spec_of(O.periodic()), np.float32)
    try:
        dev.init_analytic("taylor_green", 0.03)
        dev.step(5)
        before = dev.memory_bytes()
        f = dev.download_f()
        after = dev.memory_bytes()
        assert after - before >= 19 * dims[0] * dims[1] * dims[2] * 4
        assert np.isfinite(f).all()
    finally:
        dev.close()


# --- body-force extension (not in the reference; parity with the C port) ---
def _ywalls():
    f = O.periodic()
    f[2] = ("wall", (0, 0, 0))
    f[3] = ("moving", (0.01, 0.0, 0.0))
    return f


@pytest.mark.parametrize("sched", ["m", "f1"])
@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("lat,dims,faces", [("d3q19", (32, 16, 6), _ywalls()), ("d3q27", (32, 8, 5), O.periodic()),
                                            ("d2q9", (24, 20, 1), _ywalls())], ids=["d3q19", "d3q27", "d2q9"])
def test_body_force_bitwise(gpu, oracle_port, lat, dims, faces, dtype, sched):
    F = (3e-5, -1e-5, 2e-5 if dims[2] > 1 else 0.0)
    f0 = O.random_state(lat, dims, 31, dtype)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.05, spec_of(faces), dtype)
    try:
        if sched == "f1":
            dev.set_schedule("f1")
        dev.set_body_force(*F)
        dev.upload_f(f0)
        dev.step(6)
        mg = _moments(dev, lat)
        fg = dev.download_f()
    finally:
        dev.close()
    try:
        oracle_port.set_body_force(*F)
        fo, mo = _oracle(oracle_port, lat, dims, 1.05, faces, f0, 6)
    finally:
        oracle_port.set_body_force(0.0, 0.0, 0.0)
    assert_bitwise(mg, mo, f"forced {lat} {sched} moments")
    assert_bitwise(fg, fo, f"forced {lat} {sched} f")


@pytest.mark.parametrize("lat", ["d3q19", "d3q27"])
def test_poiseuille_profile(gpu, lat):
    """Body-force driven channel between no-slip walls (BASELINE config 3's
    flow): the steady profile is the analytic parabola u = F y'(H - y')/(2 nu)
    with the walls half a node outside the fluid (halfway bounce-back)."""
    H = 24
    dims = (32, H, 8)
    nu, om = 1.0 / 6.0, 1.0
    F = 8 * nu * 0.02 / H ** 2
    faces = O.periodic()
    faces[2] = ("wall", (0, 0, 0))
    faces[3] = ("wall", (0, 0, 0))
    dev = T.DeviceSolver(lat, T.GridDims(*dims), om, spec_of(faces), np.float64)
    try:
        assert dev.schedule == "m"
        dev.set_body_force(F, 0.0, 0.0)
        dev.init_analytic("rest")
        dev.step(12000)
        dev.phase("refresh_moments")
        u = dev.download_field("mom").reshape(3, dims[2], dims[1], dims[0])[0]
    finally:
        dev.close()
    tau = 1.0 / om
    prof = (u - tau * F + F / 2).mean(axis=(0, 2))   # stored u_eq = j + tau F; fluid velocity j + F/2
    y = np.arange(H) + 0.5
    ua = F / (2 * nu) * y * (H - y)
    assert np.abs(prof - ua).max() <= 5e-3 * ua.max()


# --- full-size, size-independent checks (BASELINE.json shapes) ------------
@pytest.mark.parametrize("lat,n", [("d3q19", 1024), ("d3q27", 512)])
def test_full_size_m_equals_f1_digests(gpu, lat, n):
    """At the benchmark sizes the oracle is too slow, so the two device
    schedules check each other: M and F1 from the same device-initialised
    Taylor-Green state agree on the FNV digest of every population plane
    after 6 steps (a checksum of checksums; each schedule is bit-exact
    against the oracle at small sizes), and mass is conserved."""
    dims = (n, n, n)
    dig, mass = {}, {}
    for sched in ("m", "f1"):
        dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.6, T.BoundarySpec.all_periodic(), np.float32)
        try:
            if sched == "f1":
                dev.set_schedule("f1")
            dev.init_analytic("taylor_green", 0.03)
            dev.step(1)
            m0, _ = dev.totals()
            dev.step(5)
            m1, _ = dev.totals()
            dig[sched] = dev.plane_digests()
            mass[sched] = (m0, m1)
        finally:
            dev.close()
    assert np.array_equal(dig["m"], dig["f1"])
    for m0, m1 in mass.values():
        assert abs(m1 - m0) <= 1e-6 * m0


# --- the 2-D M kernel (warp strips, shuffles, register rings) --------------
def _mixed2d():
    f = O.periodic()
    f[2] = ("wall", (0, 0, 0))
    f[3] = ("moving", (0.04, 0.0, 0.0))
    return f


def _xwalls2d():
    f = O.periodic()
    f[0] = ("moving", (0.0, 0.03, 0.0))
    f[1] = ("wall", (0, 0, 0))
    return f


CASES_2D = [
    ("periodic", (64, 20, 1), O.periodic()),
    ("periodic-narrow", (12, 9, 1), O.periodic()),
    ("periodic-odd", (97, 31, 1), O.periodic()),
    ("lid", (61, 33, 1), O.lid_cavity(0.05)),
    ("box", (30, 30, 1), O.closed_box()),
    ("mixed", (45, 17, 1), _mixed2d()),
    ("xwalls", (31, 40, 1), _xwalls2d()),
    ("rows-1", (40, 1, 1), O.periodic()),
]


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("case", CASES_2D, ids=lambda c: c[0])
def test_mstep2d_bitwise(gpu, oracle_port, case, dtype):
    name, dims, faces = case
    f0 = O.random_state("d2q9", dims, 13, dtype)
    dev = T.DeviceSolver("d2q9", T.GridDims(*dims), 1.37, spec_of(faces), dtype)
    try:
        assert dev.schedule == "m"
        dev.upload_f(f0)
        dev.step(7)
        mg = _moments(dev, "d2q9")
        fg = dev.download_f()
        dev.step(40)  # graph replay on small domains
        mg2 = _moments(dev, "d2q9")
        fg2 = dev.download_f()
    finally:
        dev.close()
    fo, mo = _oracle(oracle_port, "d2q9", dims, 1.37, faces, f0, 7)
    assert_bitwise(mg, mo, f"M2D {name} moments")
    assert_bitwise(fg, fo, f"M2D {name} f")
    mo2 = mo.copy()
    oracle_port.single_run("d2q9", dims, 1.37, faces, fo, mo2, 40, 0)
    assert_bitwise(mg2, mo2, f"M2D {name} moments after 47")
    assert_bitwise(fg2, fo, f"M2D {name} f after 47")


def test_mstep2d_f32_math_equals_f1(gpu):
    dims, faces = (97, 31, 1), O.lid_cavity(0.05)
    f0 = O.random_state("d2q9", dims, 5, np.float32)
    out = {}
    for sched in ("f1", "m"):
        dev = T.DeviceSolver("d2q9", T.GridDims(*dims), 1.3, spec_of(faces), np.float32)
        try:
            dev.set_schedule(sched)
            dev.set_math(_lib.MATH_F32)
            dev.upload_f(f0)
            dev.step(6)
            out[sched] = (dev.download_f(), _moments(dev, "d2q9"))
        finally:
            dev.close()
    assert_bitwise(out["m"][0], out["f1"][0], "2-D f32 math f")
    assert_bitwise(out["m"][1], out["f1"][1], "2-D f32 math moments")


# -- masked geometries (solid bits, tslb_mstep.cu k_solid_bits) --------------
SOLID_CASES = [
    ("periodic+random", (32, 8, 6), O.periodic(), lambda d: random_solid(d, 0.12, 3)),
    ("box+random", (32, 16, 7), O.closed_box(), lambda d: random_solid(d, 0.08, 9)),
    ("corners+block", (64, 8, 5), corner_box_3d(), lambda d: block_solid(d, (5, 2, 1), (40, 6, 4))),
    ("zwalls+dense", (32, 8, 9), zwalls_3d(), lambda d: random_solid(d, 0.45, 21)),
]


@pytest.mark.parametrize("lz", ["", "2"])
@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("lat", ["d3q19", "d3q27"])
@pytest.mark.parametrize("case", SOLID_CASES, ids=lambda c: c[0])
def test_mstep_solid_bitwise(gpu, oracle_port, case, lat, dtype, lz, monkeypatch):
    """M on a solid mask: fluid nodes bit-identical to the oracle; every node
    (solid ones included: moments carried through, f untouched) identical to
    the F1 schedule."""
    name, dims, faces, mk = case
    if lz:
        monkeypatch.setenv("TSLB_LZ", lz)
    solid = mk(dims)
    f0 = O.random_state(lat, dims, 17, dtype, solid)
    steps = 5
    out = {}
    for sched in ("m", "f1"):
        dev = T.DeviceSolver(lat, T.GridDims(*dims), 0.93, spec_of(faces), dtype, 1, solid)
        try:
            if sched == "m":
                assert dev.schedule == "m", "M should be the default on a masked whole domain"
            dev.set_schedule(sched)
            dev.upload_f(f0)
            dev.step(steps)
            out[sched] = (dev.download_f(), _moments(dev, lat))
        finally:
            dev.close()
    fo, mo = f0.copy(), np.zeros((O.moments_layout(lat), f0.shape[1]), dtype)
    oracle_port.single_run(lat, dims, 0.93, faces, fo, mo, steps, 0, solid)
    fluid = solid == 0
    assert_bitwise(out["m"][0], fo, f"M {lat}/{name} f", fluid)
    assert_bitwise(out["m"][1], mo, f"M {lat}/{name} moments", fluid)
    assert_bitwise(out["m"][0], out["f1"][0], f"M vs F1 {lat}/{name} f (all nodes)")
    assert_bitwise(out["m"][1], out["f1"][1], f"M vs F1 {lat}/{name} moments (all nodes)")


@pytest.mark.parametrize("dtype", DT)
def test_mstep_solid_graph_and_switch(gpu, oracle_port, dtype):
    """Graph replay (odd step counts) and F1 <-> M switches on a masked
    domain, with the solid bits built on the switch."""
    lat, dims, faces = "d3q19", (32, 16, 10), O.closed_box()
    solid = random_solid(dims, 0.15, 77)
    f0 = O.random_state(lat, dims, 8, dtype, solid)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.2, spec_of(faces), dtype, 1, solid)
    try:
        dev.set_schedule("f1")
        dev.upload_f(f0)
        dev.step(3)
        dev.set_schedule("m")
        dev.step(37)
        dev.set_schedule("f1")
        dev.step(2)
        dev.set_schedule("m")
        dev.step(33)
        mg = _moments(dev, lat)
        fg = dev.download_f()
    finally:
        dev.close()
    fo, mo = f0.copy(), np.zeros((O.moments_layout(lat), f0.shape[1]), dtype)
    oracle_port.single_run(lat, dims, 1.2, faces, fo, mo, 75, 0, solid)
    fluid = solid == 0
    assert_bitwise(fg, fo, "switch/graph M f", fluid)
    assert_bitwise(mg, mo, "switch/graph M moments", fluid)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("nsteps", [2, 33, 100])
def test_mstep2d_persistent_equals_per_pass_launches(gpu, dtype, nsteps, monkeypatch):
    # small 2-D domains run under one cooperative launch per step() call
    # (grid barrier between passes); TSLB_PERSIST=0 takes the per-pass
    # launches / graph replay. Same bits, including odd pass counts (the
    # ping-pong parity) and the first step after an upload (moments pass)
    dims, faces = (256, 256, 1), O.lid_cavity(0.1)
    f0 = O.random_state("d2q9", dims, 21, dtype)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("TSLB_PERSIST", mode)
        dev = T.DeviceSolver("d2q9", T.GridDims(*dims), 1.4450867, spec_of(faces), dtype)
        try:
            dev.upload_f(f0)
            l0 = dev.launch_count()
            dev.step(nsteps)
            launches = dev.launch_count() - l0
            dev.step(nsteps + 1)
            out[mode] = (_moments(dev, "d2q9"), dev.download_f(), launches)
        finally:
            dev.close()
    assert_bitwise(out["1"][0], out["0"][0], "persistent vs per-pass moments")
    assert_bitwise(out["1"][1], out["0"][1], "persistent vs per-pass f")
    if nsteps >= 3:  # the moments pass after the upload, then one cooperative launch
        assert out["1"][2] <= 3 < out["0"][2]


def _msums_fallback_fraction(f, q):
    """Share of nodes whose gathered populations fail the pair-form range
    check of tslb_msums.cuh (max|f| < 2^24 min|f|)."""
    a = np.abs(f.astype(np.float64))
    return float(np.mean(~(a.max(0) < a.min(0) * 2.0 ** 24)))


@pytest.mark.parametrize("lat", ["d3q19", "d3q27"])
def test_mstep_msums_both_forms_bitwise(gpu, oracle_port, lat):
    """The moment sums of the M kernel take the exact pair form where the
    node's populations span < 2^24 and the reference accumulation order
    elsewhere (tslb_msums.cuh). Node states scaled by 2^U(-12, 8) put both
    kinds of node side by side; f(N) and m(N-1) must stay bit-identical to
    fused_step. 2 % of the nodes start with all-zero populations (zero
    operands fail the check). The second step is the first M pass: it
    reduces f(1), whose populations come from differently scaled sources."""
    dims, faces, steps = (32, 16, 6), corner_box_3d(), 2
    f0 = O.random_state(lat, dims, 31, np.float64)
    rng = np.random.default_rng(7)
    scale = np.exp2(rng.uniform(-12, 8, f0.shape[1]))
    scale[rng.random(f0.shape[1]) < 0.3] = 1.0
    f0 = np.ascontiguousarray((f0 * scale[None, :]).astype(np.float32))
    f0[:, rng.random(f0.shape[1]) < 0.02] = 0.0
    dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.25, spec_of(faces), np.float32)
    try:
        assert dev.schedule == "m"
        dev.upload_f(f0)
        dev.step(steps)
        mg = _moments(dev, lat)
        fg = dev.download_f()
    finally:
        dev.close()
    fo, mo = _oracle(oracle_port, lat, dims, 1.25, faces, f0, steps)
    # f(N-1) is what the last finalize reduced: both forms must have run
    fprev, _ = _oracle(oracle_port, lat, dims, 1.25, faces, f0, steps - 1)
    frac = _msums_fallback_fraction(fprev, T.lattice_of(lat).q)
    assert 0.05 < frac < 0.95, f"fallback share {frac}: the state does not exercise both forms"
    assert_bitwise(mg, mo, f"M {lat} msums moments m(N-1)")
    assert_bitwise(fg, fo, f"M {lat} msums f(N)")


def test_persist_toggle_on_one_handle(gpu, oracle_port, monkeypatch):
    """TSLB_PERSIST is read per step() call: a graph captured under per-pass
    launches, then persistent calls with odd counts that swap the ping-pong
    buffers, must still take exactly the requested number of steps."""
    lat, dims, faces, om = "d2q9", (256, 256, 1), O.lid_cavity(0.08), 1.3
    f0 = O.random_state(lat, dims, 4, np.float64)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), om, spec_of(faces), np.float64)
    total = 0
    try:
        dev.upload_f(f0)
        for mode, n in (("0", 40), ("1", 33), ("0", 35), ("1", 35), ("0", 32)):
            monkeypatch.setenv("TSLB_PERSIST", mode)
            dev.step(n)
            total += n
            assert dev.steps_done() == total, f"after TSLB_PERSIST={mode} step({n})"
        fg = dev.download_f()
    finally:
        dev.close()
    fo, _ = _oracle(oracle_port, lat, dims, om, faces, f0, total)
    assert_bitwise(fg, fo, "persist toggles")


PARTIAL = [
    ("periodic-36x13", (36, 13, 7), O.periodic()),
    ("corners-44x10", (44, 10, 5), corner_box_3d()),
    ("xwalls-20x9", (20, 9, 6), xwalls_3d()),
    ("ylid-100x11", (100, 11, 4), ylid_3d()),
]


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("lat", ["d3q19", "d3q27"])
@pytest.mark.parametrize("case", PARTIAL, ids=lambda c: c[0])
def test_mstep_partial_tiles_bitwise(gpu, oracle_port, case, lat, dtype):
    """Grids that do not tile 32 x 8 run the M kernel with partial tiles at
    the high x / y edges (halo column / row right after the last node,
    inactive lanes push nothing) -- bit-identical to fused_step."""
    name, dims, faces = case
    f0 = O.random_state(lat, dims, 23, dtype)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), 0.93, spec_of(faces), dtype)
    try:
        assert dev.schedule == "m", "partial tiles should run the M schedule"
        dev.upload_f(f0)
        dev.step(5)
        mg = _moments(dev, lat)
        fg = dev.download_f()
    finally:
        dev.close()
    fo, mo = _oracle(oracle_port, lat, dims, 0.93, faces, f0, 5)
    assert_bitwise(mg, mo, f"M partial {lat}/{name} moments")
    assert_bitwise(fg, fo, f"M partial {lat}/{name} f")


@pytest.mark.parametrize("dtype", DT)
def test_mstep_partial_tiles_solid(gpu, oracle_port, dtype):
    lat, dims, faces = "d3q19", (44, 13, 6), zwalls_3d()
    solid = random_solid(dims, 0.2, 9)
    f0 = O.random_state(lat, dims, 29, dtype, solid)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.1, spec_of(faces), dtype, 1, solid)
    try:
        assert dev.schedule == "m"
        dev.upload_f(f0)
        dev.step(4)
        fg = dev.download_f()
    finally:
        dev.close()
    fo = f0.copy()
    oracle_port.single_run(lat, dims, 1.1, faces, fo, None, 4, 0, solid)
    assert_bitwise(fg, fo, "M partial tiles, solid mask", solid == 0)


# --- mixed precision: fp16 moment storage, fp32 node arithmetic -------------
def _tgv_f0(dims, dtype, amp=0.04):
    """Taylor-Green f(0) through the oracle's initialize_regularized."""
    nx, ny, nz = dims
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    X, Y, Z = (2 * np.pi * (a.ravel() + 0.5) / n for a, n in ((i, nx), (j, ny), (k, nz)))
    st = np.zeros((10, X.size))
    st[0] = 1 + 3 * (amp * amp / 16) * (np.cos(2 * X) + np.cos(2 * Y)) * (np.cos(2 * Z) + 2)
    st[1] = amp * np.sin(X) * np.cos(Y) * np.cos(Z)
    st[2] = -amp * np.cos(X) * np.sin(Y) * np.cos(Z)
    return O.Oracle("port").init_regularized("d3q19", dims, st.astype(dtype))


@pytest.mark.parametrize("lat", ["d3q19", "d3q27"])
def test_f16_moment_storage_within_tolerance(gpu, oracle_port, lat):
    """Mixed precision (fp16 moments, fp32 arithmetic; tslb_store16.cuh)
    against the fp64 reference arithmetic after 300 steps (D3Q19: a
    decaying Taylor-Green vortex; D3Q27: a random near-equilibrium state):
    stated tolerance max|drho| <= 2e-5, max|du| <= 2e-3 * max|u| (measured
    r02: fp16 storage 5.7e-6 / 8.1e-4, fp32 storage + fp32 math 4.6e-6 /
    9.9e-5). The fp32-storage run must sit inside it as well."""
    dims, steps, om = (32, 32, 16), 300, 1.6
    faces = O.periodic()
    f0 = _tgv_f0(dims, np.float64) if lat == "d3q19" else O.random_state(lat, dims, 3, np.float64)
    fo, mo = f0.copy(), np.zeros((O.moments_layout(lat), f0.shape[1]))
    oracle_port.single_run(lat, dims, om, faces, fo, mo, steps, 0)
    oracle_port.single_run(lat, dims, om, faces, fo, mo, 1, 2)  # refresh: moments of f(N)
    D = T.lattice_of(lat).dim
    umax = np.max(np.abs(mo[1:1 + D]))
    errs = {}
    for storage in ("f16", "native"):
        dev = T.DeviceSolver(lat, T.GridDims(*dims), om, spec_of(faces), np.float32)
        try:
            if storage == "f16":
                dev.set_moment_storage("f16")
            else:
                dev.set_math(_lib.MATH_F32)
            dev.upload_f(f0.astype(np.float32))
            dev.step(steps)
            dev.phase("refresh_moments")
            rho, mom = dev.download_field("rho").astype(np.float64), dev.download_field("mom").astype(np.float64)
        finally:
            dev.close()
        errs[storage] = (np.max(np.abs(rho - mo[0])), np.max(np.abs(mom - mo[1:1 + D])) / umax)
    print("f16 / fp32 errors:", errs)
    for storage, (drho, du) in errs.items():
        assert drho <= 2e-5, (storage, drho)
        assert du <= 2e-3, (storage, du)


def test_f16_moment_storage_reads_are_consistent(gpu):
    """In fp16 storage the host sees fp32 moments decoded from the fp16 state
    and f(t+1) = stream_collide(decoded m(t)) -- the F1 fp32-math phase on
    the same moments gives the same populations bit for bit; switching back
    to native storage continues from the decoded state."""
    lat, dims, om = "d3q19", (32, 16, 8), 1.3
    f0 = O.random_state(lat, dims, 13, np.float32)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), om, spec_of(zwalls_3d()), np.float32)
    f1 = T.DeviceSolver(lat, T.GridDims(*dims), om, spec_of(zwalls_3d()), np.float32)
    try:
        dev.set_moment_storage("f16")
        dev.upload_f(f0)
        dev.step(7)
        m = _moments(dev, lat)
        fg = dev.download_f()
        f1.set_schedule("f1")
        f1.set_math(_lib.MATH_F32)
        f1.upload_field("rho", m[0])
        f1.upload_field("mom", m[1:4])
        f1.upload_field("pineq", m[4:])
        f1.phase("stream_collide")
        assert_bitwise(fg, f1.download_f(), "f16 storage: f = stream_collide(decoded moments)")
        assert np.all(np.isfinite(m))
        dev.set_moment_storage("native")
        dev.step(3)
        assert np.all(np.isfinite(dev.download_f()))
    finally:
        dev.close()
        f1.close()


def test_f16_moment_storage_rules(gpu):
    spec = spec_of(O.periodic())
    for args, ok in ((("d3q19", (32, 8, 4), np.float32), True), (("d3q19", (36, 8, 4), np.float32), False),
                     (("d3q19", (32, 8, 4), np.float64), False), (("d2q9", (32, 8, 1), np.float32), False)):
        lat, dims, dt = args
        dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.0, spec, dt)
        try:
            if ok:
                dev.set_moment_storage("f16")
            else:
                with pytest.raises(_lib.InvalidArgument):
                    dev.set_moment_storage("f16")
        finally:
            dev.close()


@pytest.mark.parametrize("lat,dims", [("d3q19", (32, 8, 6)), ("d2q9", (45, 17, 1))])
def test_refresh_under_m_is_one_moment_pass(gpu, oracle_port, lat, dims):
    """refresh_moments under M runs one more moment-resident pass (no stored
    f): the host sees moments(f(t+1)); the next step takes them over without
    a kernel; any other call first leaves that state. Every transition
    against fused_step + compute_moments."""
    faces, om, dt = (corner_box_3d() if lat == "d3q19" else O.lid_cavity(0.05)), 1.3, np.float64
    f0 = O.random_state(lat, dims, 41, dt)
    ref = f0.copy()
    rmo = np.zeros((O.moments_layout(lat), ref.shape[1]), dt)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), om, spec_of(faces), dt)

    def oracle(n, mode=0):
        oracle_port.single_run(lat, dims, om, faces, ref, rmo, n, mode)

    try:
        assert dev.schedule == "m"
        dev.upload_f(f0)
        dev.step(5)
        oracle(5)
        launches = dev.launch_count()
        dev.phase("refresh_moments")
        dev.phase("refresh_moments")  # idempotent
        assert dev.launch_count() - launches == 1, "one moment pass, no f materialised"
        oracle(1, 2)
        assert_bitwise(_moments(dev, lat), rmo, "refreshed moments")
        mass, _ = dev.totals()
        assert abs(mass - rmo[0].sum()) <= 1e-12 * abs(mass)
        # the next step takes the refreshed moments over
        l0 = dev.launch_count()
        dev.step(1)
        assert dev.launch_count() == l0, "the step after a refresh is a swap"
        oracle(1)
        assert dev.steps_done() == 6
        dev.step(2)
        oracle(2)
        assert_bitwise(dev.download_f(), ref, "f after refresh + steps")
        assert_bitwise(_moments(dev, lat), rmo, "lagged moments after refresh + steps")
        # refresh, then read f (materialised from m(t)), then step
        dev.phase("refresh_moments")
        oracle(1, 2)
        assert_bitwise(dev.download_f(), ref, "f read after refresh")
        assert_bitwise(_moments(dev, lat), rmo, "moments after refresh + f read")
        dev.step(2)
        oracle(2)
        assert_bitwise(dev.download_f(), ref, "f after refresh, f read, steps")
        # refresh, then overwrite a moment array and step: the step
        # recomputes the moments from f, as fused_step does
        dev.phase("refresh_moments")
        dev.upload_field("rho", np.full(ref.shape[1], 3.0))
        dev.step(2)
        oracle(2)
        assert_bitwise(dev.download_f(), ref, "f after refresh, moment upload, steps")
    finally:
        dev.close()


TB_CASES = [
    ("lid-256", (256, 256, 1), O.lid_cavity(0.1), None),
    ("periodic-odd", (100, 70, 1), O.periodic(), None),
    ("lid-odd", (61, 45, 1), O.lid_cavity(0.05), None),
    ("ywalls-forced", (96, 40, 1), [("periodic", (0, 0, 0))] * 2 + [("wall", (0, 0, 0))] * 2
     + [("periodic", (0, 0, 0))] * 2, (2e-5, 0.0, 0.0)),
]


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("nsteps", [2, 5, 9, 33])
@pytest.mark.parametrize("name,dims,faces,force", TB_CASES, ids=[c[0] for c in TB_CASES])
def test_mstep2d_temporal_blocking_bitwise(gpu, oracle_port, name, dims, faces, force, nsteps, dtype, monkeypatch):
    """The persistent 2-D path's temporal blocking (tiles advanced up to K
    passes in shared memory between grid barriers; group count of the
    parity of the pass count) == fused_step, bit for bit: walls and the
    moving lid (bounces gathered from the node's own opposite push),
    periodic wrap, partial tiles, the body force."""
    f0 = O.random_state("d2q9", dims, 13, dtype)
    monkeypatch.setenv("TSLB_PERSIST", "1")
    monkeypatch.setenv("TSLB_TB2D", "1")
    dev = T.DeviceSolver("d2q9", T.GridDims(*dims), 1.37, spec_of(faces), dtype)
    try:
        if force:
            dev.set_body_force(*force)
        dev.upload_f(f0)
        l0 = dev.launch_count()
        dev.step(nsteps + 1)  # (the moments pass after the upload, then one launch)
        assert dev.launch_count() - l0 <= 3
        mg = _moments(dev, "d2q9")
        fg = dev.download_f()
    finally:
        dev.close()
    fo = f0.copy()
    mo = np.zeros((6, fo.shape[1]), dtype)
    if force:
        oracle_port.set_body_force(*force)
    try:
        oracle_port.single_run("d2q9", dims, 1.37, faces, fo, mo, nsteps + 1, 0)
    finally:
        oracle_port.set_body_force(0.0, 0.0, 0.0)
    assert_bitwise(mg, mo, f"TB {name} moments")
    assert_bitwise(fg, fo, f"TB {name} f")


@pytest.mark.parametrize("dtype", DT)
def test_mstep2d_temporal_blocking_f32_math_equals_per_pass(gpu, dtype, monkeypatch):
    """fp32 node math (the fused forms every single-fluid kernel shares):
    the temporally blocked persistent path == one grid barrier per pass,
    bit for bit."""
    dims, faces = (200, 120, 1), O.lid_cavity(0.08)
    f0 = O.random_state("d2q9", dims, 3, dtype)
    out = {}
    monkeypatch.setenv("TSLB_PERSIST", "1")
    for tb in ("1", "0"):
        monkeypatch.setenv("TSLB_TB2D", tb)
        dev = T.DeviceSolver("d2q9", T.GridDims(*dims), 1.51, spec_of(faces), dtype)
        try:
            dev.set_math(_lib.MATH_F32)
            dev.upload_f(f0)
            dev.step(23)
            out[tb] = (_moments(dev, "d2q9"), dev.download_f())
        finally:
            dev.close()
    assert_bitwise(out["1"][0], out["0"][0], "TB f32 math moments")
    assert_bitwise(out["1"][1], out["0"][1], "TB f32 math f")
