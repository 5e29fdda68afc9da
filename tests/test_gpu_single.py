"""GPU parity of the single-fluid hot path (fused_step and its phases)
against the CPU oracle, through the C-ABI. Bar: bit-exact (node-local
arithmetic in double, --fmad=false), for double AND float storage, as the
reference's own fused-vs-two-buffer check (unit_collision_stream.cpp:269-330,
acceptance.cpp:101-135)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2304_06437_b200 import _lib
from paper_2304_06437_b200 import tslb as T

from helpers import assert_bitwise, block_solid, corner_box_3d, mixed_2d, random_solid, spec_of, zwalls_3d

pytestmark = pytest.mark.gpu

DT = [np.float64, np.float32]

CASES_2D = [
    ("periodic", (16, 16, 1), O.periodic(), None),
    ("box", (16, 12, 1), O.closed_box(), None),
    ("lid", (20, 16, 1), O.lid_cavity(0.05), None),
    ("mixed+block", (16, 16, 1), mixed_2d(), block_solid((16, 16, 1), (6, 5, 0), (10, 8, 1))),
    ("periodic+random", (24, 20, 1), O.periodic(), random_solid((24, 20, 1), 0.1, 4)),
    ("odd-x", (131, 9, 1), O.lid_cavity(0.03), None),
]
CASES_3D = [
    ("periodic", (8, 7, 6), O.periodic(), None),
    ("zwalls", (8, 7, 6), zwalls_3d(), None),
    ("box-corners", (9, 8, 7), corner_box_3d(), None),
    ("box+random", (10, 9, 8), O.closed_box(), random_solid((10, 9, 8), 0.08, 7)),
    ("periodic+block", (12, 10, 9), O.periodic(), block_solid((12, 10, 9), (3, 2, 2), (7, 6, 5))),
    ("wide-x", (200, 4, 3), zwalls_3d(), None),
    ("multi-block-x-box", (1040, 3, 3), corner_box_3d(), None),
    ("multi-block-x-zwalls", (1032, 2, 3), zwalls_3d(), None),
]


def _gpu_single(lat, dims, omega, faces, f, steps, solid, phase="step", moments=None):
    dev = T.DeviceSolver(lat, T.GridDims(*dims), omega, spec_of(faces), f.dtype, 1, solid)
    try:
        dev.upload_f(f)
        if moments is not None:
            L = T.lattice_of(lat)
            dev.upload_field("rho", moments[0])
            dev.upload_field("mom", moments[1:1 + L.dim])
            dev.upload_field("pineq", moments[1 + L.dim:])
        if phase == "step":
            dev.step(steps)
        elif phase == "reference":
            dev.phase("reference_step", steps)
        else:
            for _ in range(steps):
                dev.phase(phase)
        L = T.lattice_of(lat)
        mo = np.concatenate([dev.download_field("rho")[None], dev.download_field("mom").reshape(L.dim, -1),
                             dev.download_field("pineq").reshape(L.npineq, -1)])
        return dev.download_f(0), mo
    finally:
        dev.close()


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("lat,case", [("d2q9", c) for c in CASES_2D] + [("d3q19", c) for c in CASES_3D]
                         + [("d3q27", c) for c in CASES_3D[:4]])
def test_fused_step_bitwise(gpu, oracle_port, lat, case, dtype):
    name, dims, faces, solid = case
    f0 = O.random_state(lat, dims, 2024, dtype, solid)
    omega = 1.31 if lat == "d2q9" else 0.77
    fo, mo = f0.copy(), np.zeros((O.moments_layout(lat), f0.shape[1]), dtype)
    oracle_port.single_run(lat, dims, omega, faces, fo, mo, 5, 0, solid)
    fg, mg = _gpu_single(lat, dims, omega, faces, f0, 5, solid)
    fluid = np.ones(f0.shape[1], bool) if solid is None else solid == 0
    assert_bitwise(fg, fo, f"{lat}/{name} f", fluid)
    # lagged moment semantics: arrays hold m(t) of the last step (solver.hpp:68-69)
    assert_bitwise(mg, mo, f"{lat}/{name} moments", fluid)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("lat,case", [("d2q9", CASES_2D[3]), ("d3q19", CASES_3D[2]), ("d3q19", CASES_3D[3])])
def test_matches_reference_build(gpu, oracle_ref, lat, case, dtype):
    """Directly against the UNMODIFIED reference headers (oracle/_ref)."""
    name, dims, faces, solid = case
    f0 = O.random_state(lat, dims, 55, dtype, solid)
    fr = f0.copy()
    oracle_ref.single_run(lat, dims, 1.1, faces, fr, None, 4, 0, solid)
    fg, _ = _gpu_single(lat, dims, 1.1, faces, f0, 4, solid)
    fluid = np.ones(f0.shape[1], bool) if solid is None else solid == 0
    assert_bitwise(fg, fr, f"{lat}/{name} vs reference build", fluid)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("mode,phase", [(1, "reference"), (2, "compute_moments"), (3, "stream_collide"),
                                        (4, "stream_only")])
@pytest.mark.parametrize("lat,case", [("d2q9", CASES_2D[3]), ("d3q19", CASES_3D[3])])
def test_phases_bitwise(gpu, oracle_port, lat, case, dtype, mode, phase):
    name, dims, faces, solid = case
    f0 = O.random_state(lat, dims, 91, dtype, solid)
    nm = O.moments_layout(lat)
    m0 = np.random.default_rng(5).uniform(-0.01, 0.01, (nm, f0.shape[1])).astype(dtype)
    m0[0] += 1
    fo, mo = f0.copy(), m0.copy()
    steps = 3 if mode in (1, 4) else 1
    oracle_port.single_run(lat, dims, 1.2, faces, fo, mo, steps, mode, solid)
    fg, mg = _gpu_single(lat, dims, 1.2, faces, f0, steps, solid, phase, m0)
    fluid = np.ones(f0.shape[1], bool) if solid is None else solid == 0
    assert_bitwise(fg, fo, f"{phase} f", fluid)
    if mode in (1, 2):
        assert_bitwise(mg, mo, f"{phase} moments", fluid)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("lat,case", [("d2q9", CASES_2D[2]), ("d3q19", CASES_3D[1]), ("d3q19", CASES_3D[7])])
def test_signed_zero_moments_bitwise(gpu, oracle_port, lat, case, dtype):
    """stream_collide on user-written moments with rho = -0.0 / +0.0 and zero
    stress: the vectorised kernel must fall back to the reference order."""
    name, dims, faces, solid = case
    n = int(np.prod(dims))
    nm = O.moments_layout(lat)
    m0 = np.random.default_rng(9).uniform(-0.01, 0.01, (nm, n)).astype(dtype)
    m0[0] += 1
    m0[0, ::7] = -0.0
    m0[0, 3::11] = 0.0
    m0[:, 5::13] = 0.0
    m0[1:, 6::17] = -0.0
    f0 = O.random_state(lat, dims, 1, dtype)
    fo, mo = f0.copy(), m0.copy()
    oracle_port.single_run(lat, dims, 1.2, faces, fo, mo, 1, 3)
    fg, _ = _gpu_single(lat, dims, 1.2, faces, f0, 1, None, "stream_collide", m0)
    assert_bitwise(fg, fo, "f")


@pytest.mark.parametrize("lat,case", [("d2q9", c) for c in CASES_2D] + [("d3q19", c) for c in CASES_3D]
                         + [("d3q27", c) for c in CASES_3D])
def test_classify_bitwise(gpu, oracle_port, lat, case):
    name, dims, faces, solid = case
    so, sl, nf = oracle_port.classify(lat, dims, faces, solid)
    geo = T.classify_nodes(lat, T.GridDims(*dims), spec_of(faces), solid)
    assert_bitwise(geo.solid, so, "solid")
    assert_bitwise(geo.slow_mask, sl, "slow_mask")
    assert geo.n_fluid == nf


def test_half_periodic_axis_rejected(gpu):
    spec = T.BoundarySpec.all_periodic()
    spec.faces[T.YMin] = T.Face(T.FaceKind.NoSlipWall)
    with pytest.raises(T.InvalidArgument, match="axis 1"):
        T.SingleFluidSim(T.D2Q9, T.GridDims(8, 8, 1), T.CollisionParams(1.0), spec)
    with pytest.raises(T.InvalidArgument):
        T.SingleFluidSim(T.D2Q9, T.GridDims(0, 8, 1), T.CollisionParams(1.0), T.BoundarySpec())
    with pytest.raises(T.InvalidArgument, match="mask size"):
        T.SingleFluidSim(T.D2Q9, T.GridDims(8, 8, 1), T.CollisionParams(1.0), T.BoundarySpec(),
                         solid=np.zeros(10, np.uint8))


def test_cavity_c1_bitwise(gpu, oracle_port):
    """Config 1: D2Q9 lid-driven cavity 256^2, Re 100, 1000 steps, fp64,
    rest init -- bitwise against the oracle."""
    dims = (256, 256, 1)
    omega = T.omega_from_nu(0.064)
    faces = O.lid_cavity(0.025)
    g = T.GridDims(*dims)
    sim = T.SingleFluidSim(T.D2Q9, g, T.CollisionParams(omega), spec_of(faces))
    s = sim.fields()
    T.initialize_regularized(s, sim.geometry(), lambda i, j, k: (1.0, 0, 0, 0, 0, 0, 0, 0, 0, 0), T.D2Q9)
    f0 = s.f.copy()
    sim.run(1000)
    fo = f0.copy()
    oracle_port.single_run("d2q9", dims, omega, faces, fo, None, 1000, 0)
    assert_bitwise(sim.view().f, fo, "cavity f after 1000 steps")
    # reference digest of the same state (bench.hpp:93-99)
    assert T.fnv1a(sim.view().f) == oracle_port.fnv1a(fo)


def test_sim_host_mirror_semantics(gpu, oracle_port):
    """fields() edits are uploaded before the next step; moments lag by one
    step until refresh_moments() (solver.hpp:68-69, 96)."""
    dims = (12, 10, 1)
    sim = T.SingleFluidSim(T.D2Q9, T.GridDims(*dims), T.CollisionParams(1.1), T.BoundarySpec.all_periodic())
    f0 = O.random_state("d2q9", dims, 17)
    sim.fields().f[...] = f0
    sim.run(3)
    fo, mo = f0.copy(), np.zeros((6, f0.shape[1]))
    oracle_port.single_run("d2q9", dims, 1.1, O.periodic(), fo, mo, 3, 0)
    v = sim.view()
    assert_bitwise(v.f, fo, "f")
    assert_bitwise(v.rho, mo[0], "lagged rho")
    sim.refresh_moments()
    oracle_port.single_run("d2q9", dims, 1.1, O.periodic(), fo, mo, 1, 2)
    assert_bitwise(sim.view().rho, mo[0], "refreshed rho")
    assert sim.steps() == 3


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-12), (np.float32, 1e-5)])
def test_conservation_and_totals(gpu, oracle_port, dtype, tol):
    """Mass/momentum conservation on a periodic box (unit_collision_stream.cpp
    :332-379) and device totals vs the serial reference sum."""
    dims = (24, 20, 18)
    sim = T.SingleFluidSim(T.D3Q19, T.GridDims(*dims), T.CollisionParams(1.1), T.BoundarySpec.all_periodic(),
                           dtype=dtype)
    sim.fields().f[...] = O.random_state("d3q19", dims, 91, dtype)
    sim.refresh_moments()
    m0, p0 = sim.totals()
    v = sim.view()
    # the device tree sums in fp64 (deterministic); the reference sums
    # serially in T, whose own rounding error dominates for float storage
    exact = float(np.sum(v.rho.astype(np.float64)))
    assert abs(m0 - exact) / exact < 1e-14
    mref, pref = oracle_port.totals(v.rho, v.mom)
    assert abs(m0 - mref) / mref < (1e-13 if dtype == np.float64 else 1e-5)
    sim.run(200)
    sim.refresh_moments()
    m1, p1 = sim.totals()
    assert abs(m1 - m0) / m0 < tol
    assert np.all(np.abs(p1 - p0) < (1e-10 if dtype == np.float64 else 1e-3))
    rep = sim.stability()
    ref = oracle_port.stability(sim.view().rho, sim.view().mom)
    assert rep.finite and ref["finite"]
    assert rep.max_speed == pytest.approx(ref["max_speed"], rel=1e-12)
    assert rep.min_rho == ref["min_rho"] and rep.max_rho == ref["max_rho"]


def test_stability_locates_nonfinite(gpu):
    dims = (8, 8, 4)
    sim = T.SingleFluidSim(T.D3Q19, T.GridDims(*dims), T.CollisionParams(1.0), T.BoundarySpec.all_periodic())
    s = sim.fields()
    s.f[...] = O.random_state("d3q19", dims, 3)
    s.f[2, 77] = np.nan
    sim.refresh_moments()
    rep = sim.stability()
    assert not rep.finite and rep.first_bad == 77


@pytest.mark.parametrize("lat", ["d2q9", "d3q19", "d3q27"])
def test_fp32_math_mode_within_tolerance(gpu, oracle_port, lat):
    """Opt-in fp32 node arithmetic: tolerance parity:
    max|drho| <= 2e-5, max|du|/|u|max <= 2e-4 after 200 steps."""
    dims = (32, 32, 1) if lat == "d2q9" else (16, 16, 16)
    faces = O.lid_cavity(0.05) if lat == "d2q9" else zwalls_3d()
    f0 = O.random_state(lat, dims, 8, np.float32)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.4, spec_of(faces), np.float32)
    dev.set_math(1)
    dev.upload_f(f0)
    dev.step(200)
    dev.phase("refresh_moments")
    rho, mom = dev.download_field("rho"), dev.download_field("mom")
    fo, mo = f0.copy(), np.zeros((O.moments_layout(lat), f0.shape[1]), np.float32)
    oracle_port.single_run(lat, dims, 1.4, faces, fo, mo, 200, 0)
    oracle_port.single_run(lat, dims, 1.4, faces, fo, mo, 1, 2)
    D = T.lattice_of(lat).dim
    assert np.max(np.abs(rho - mo[0])) <= 2e-5
    umax = np.max(np.abs(mo[1:1 + D]))
    assert np.max(np.abs(mom - mo[1:1 + D])) / umax <= 2e-4
    dev.close()


def test_device_digest_matches_host_definition(gpu):
    dims = (40, 36, 5)
    sim = T.SingleFluidSim(T.D3Q19, T.GridDims(*dims), T.CollisionParams(1.0), T.BoundarySpec.all_periodic(),
                           dtype=np.float32)
    sim.fields().f[...] = O.random_state("d3q19", dims, 11, np.float32)
    sim.run(2)
    dg = sim.plane_digests()[0]
    host = T.chunked_plane_digest(sim.view().f, T.GridDims(*dims))
    assert np.array_equal(dg, host)


@pytest.mark.parametrize("init", ["shear", "taylor_green", "rest"])
def test_device_init_matches_host_formula(gpu, init):
    """Device analytic initialisers agree with the host initialiser to
    libm-vs-CUDA-math rounding (not a parity path: bench inits only)."""
    dims = (32, 16, 8)
    g = T.GridDims(*dims)
    dev = T.DeviceSolver(T.D3Q19, g, 1.6, T.BoundarySpec.all_periodic(), np.float64)
    dev.init_analytic(init, 0.03)
    fdev = dev.download_f()
    s = T.allocate_fields(g, T.D3Q19)

    def st(i, j, k):
        X, Y, Z = (2 * np.pi * (i + 0.5) / dims[0], 2 * np.pi * (j + 0.5) / dims[1], 2 * np.pi * (k + 0.5) / dims[2])
        z = np.zeros_like(X)
        if init == "shear":
            return (1.0, 0.03 * np.sin(2 * np.pi * j / dims[1]), z, z, z, z, z, z, z, z)
        if init == "rest":
            return (1.0, z, z, z, z, z, z, z, z, z)
        U = 0.03
        return (1 + 3 * (U * U / 16) * (np.cos(2 * X) + np.cos(2 * Y)) * (np.cos(2 * Z) + 2),
                U * np.sin(X) * np.cos(Y) * np.cos(Z), -U * np.cos(X) * np.sin(Y) * np.cos(Z), z, z, z, z, z, z, z)

    T.initialize_regularized(s, None, st, T.D3Q19)
    assert np.max(np.abs(fdev - s.f)) < 1e-15
    dev.close()


def test_graph_replay_then_reference_step(gpu, oracle_port):
    """Graph replay (>= 32 steps on a small box), then the two-buffer step
    (which swaps buffers and must drop the captured graph), then more
    replays: every phase bit-exact against the oracle."""
    lat, dims, faces, solid = "d3q19", (12, 10, 8), zwalls_3d(), None
    f0 = O.random_state(lat, dims, 4, np.float64)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.1, spec_of(faces), np.float64)
    dev.upload_f(f0)
    dev.step(40)
    dev.phase("reference_step", 3)
    dev.step(33)
    got = dev.download_f()
    dev.close()
    ref = f0.copy()
    oracle_port.single_run(lat, dims, 1.1, faces, ref, None, 40, 0)
    oracle_port.single_run(lat, dims, 1.1, faces, ref, None, 3, 1)
    oracle_port.single_run(lat, dims, 1.1, faces, ref, None, 33, 0)
    assert_bitwise(got, ref, "f after graph/reference/graph")


WIDE_CASES = [
    ("d3q19", "periodic", (256, 6, 5), O.periodic()),
    ("d3q19", "zwalls", (256, 4, 6), zwalls_3d()),
    ("d3q19", "box", (256, 5, 4), O.closed_box()),
    ("d3q19", "ylid", (512, 3, 4), [("periodic", (0, 0, 0))] * 2 + [("wall", (0, 0, 0)), ("moving", (0.05, 0.0, 0.01))]
     + [("periodic", (0, 0, 0))] * 2),
    ("d3q27", "zwalls", (256, 4, 4), zwalls_3d()),
    ("d2q9", "lid", (256, 8, 1), O.lid_cavity(0.04)),
]


@pytest.mark.parametrize("variant", ["vec"])
@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("case", WIDE_CASES, ids=lambda c: f"{c[0]}-{c[1]}")
def test_box_kernels_bitwise_wide_rows(gpu, oracle_port, case, dtype, variant, monkeypatch):
    """The box-geometry stream-collide kernels on wide rows: bit-exact
    against the oracle, including
    multi-plane CTAs (TSLB_KZ=3) and the wall/wrap row ends."""
    lat, name, dims, faces = case
    monkeypatch.setenv("TSLB_STREAMCOLL", variant)
    monkeypatch.setenv("TSLB_KZ", "3")
    f0 = O.random_state(lat, dims, 7, dtype)
    fo, mo = f0.copy(), np.zeros((O.moments_layout(lat), f0.shape[1]), dtype)
    oracle_port.single_run(lat, dims, 0.83, faces, fo, mo, 4, 0)
    fg, mg = _gpu_single(lat, dims, 0.83, faces, f0, 4, None)
    assert_bitwise(fg, fo, f"{variant} {lat}/{name} f")
    assert_bitwise(mg, mo, f"{variant} {lat}/{name} moments")


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("sched", ["m", "f1"])
def test_slice_sampler_matches_full_download(gpu, axis, sched):
    """download_slice (device-side sampler for the output writers) returns
    exactly the corresponding plane of download_field, for every axis."""
    dims = (32, 16, 6)
    dev = T.DeviceSolver("d3q19", T.GridDims(*dims), 1.3, spec_of(zwalls_3d()), np.float32)
    try:
        dev.set_schedule(sched)
        dev.init_analytic("taylor_green", 0.03)
        dev.step(3)
        for name in ("rho", "mom", "pineq"):
            full = dev.download_field(name).reshape(-1, dims[2], dims[1], dims[0])
            idx = dims[axis] // 2
            sl = dev.download_slice(name, axis, idx)
            want = full[:, idx] if axis == 2 else full[:, :, idx] if axis == 1 else full[:, :, :, idx]
            assert_bitwise(sl, want, f"slice {name} axis {axis}")
    finally:
        dev.close()


def test_invalid_arguments_raise(gpu):
    """EINVAL paths of the C-ABI (fields.hpp:84 / boundary.hpp:65-77 analogues
    and the extension entry points): nothing is created, an exception is
    raised, the error string names the problem."""
    spec = T.BoundarySpec.all_periodic()
    with pytest.raises(T.InvalidArgument):
        T.DeviceSolver("d3q19", T.GridDims(8, 8, 0), 1.0, spec)
    with pytest.raises(T.InvalidArgument):
        T.DeviceSolver("d2q9", T.GridDims(8, 8, 3), 1.0, spec)  # 2-D lattice on a 3-D grid
    for slab in ((4, 8), (-1, 2), (0, 0)):
        with pytest.raises(T.InvalidArgument):
            T.DeviceSolver("d3q19", T.GridDims(8, 8, 8), 1.0, spec, slab=slab)
    dev = T.DeviceSolver("d3q19", T.GridDims(32, 8, 4), 1.0, spec, np.float32, 2, None, T.ColorParams())
    try:
        with pytest.raises(RuntimeError):
            dev.set_schedule("m")  # the M schedule is single-fluid
        with pytest.raises(RuntimeError):
            dev.set_body_force(1e-5, 0.0, 0.0)  # forcing is a single-fluid extension
    finally:
        dev.close()


def test_stability_empty_and_nan_first(gpu):
    """scan_stability edge cases (solver.hpp:39-65): no fluid node -> the
    report's zero fields; a NaN rho on the FIRST fluid node sticks in
    min/max (std::min/std::max never replace it), a later NaN is ignored."""
    dims = (8, 8, 4)
    n = int(np.prod(dims))
    dev = T.DeviceSolver("d3q19", T.GridDims(*dims), 1.0, T.BoundarySpec.all_periodic(), np.float64,
                         solid=np.ones(n, np.uint8))
    try:
        rep = dev.stability()
        assert rep.finite and rep.min_rho == 0.0 and rep.max_rho == 0.0 and rep.max_speed == 0.0
    finally:
        dev.close()
    solid = np.zeros(n, np.uint8)
    solid[:5] = 1  # the first fluid node is 5
    for bad, sticks in ((5, True), (40, False)):
        dev = T.DeviceSolver("d3q19", T.GridDims(*dims), 1.0, T.BoundarySpec.all_periodic(), np.float64,
                             solid=solid)
        try:
            rho = np.linspace(0.9, 1.1, n)
            rho[bad] = np.nan
            dev.upload_field("rho", rho)
            rep = dev.stability()
            assert not rep.finite and rep.first_bad == bad
            if sticks:
                assert np.isnan(rep.min_rho) and np.isnan(rep.max_rho)
            else:
                fl = np.delete(rho[5:], bad - 5)
                assert rep.min_rho == fl.min() and rep.max_rho == fl.max()
        finally:
            dev.close()


def test_host_buffer_validation(gpu):
    """The Python mirror checks every host buffer it hands to the C-ABI."""
    dims = (8, 8, 4)
    dev = T.DeviceSolver("d3q19", T.GridDims(*dims), 1.0, T.BoundarySpec.all_periodic(), np.float32)
    try:
        n = int(np.prod(dims))
        with pytest.raises(_lib.InvalidArgument):
            dev.upload_f(np.zeros((19, n - 1), np.float32))
        for bad in (np.empty((19, n), np.float64), np.empty((19, n + 1), np.float32),
                    np.empty((n, 19), np.float32).T):
            with pytest.raises(_lib.InvalidArgument):
                dev.download_f(out=bad)
        with pytest.raises(_lib.InvalidArgument):
            dev.upload_field("rho", np.zeros(n + 3))
        ok = np.empty((19, n), np.float32)
        assert dev.download_f(out=ok) is ok
    finally:
        dev.close()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("lat,dims,sched,masked", [
    ("d3q19", (32, 16, 6), "m", False), ("d3q19", (32, 16, 6), "f1", False), ("d3q27", (32, 8, 5), "m", False),
    ("d2q9", (45, 17, 1), "m", False), ("d3q19", (12, 10, 9), "f1", True)])
def test_init_state_matches_host_initialize_regularized(gpu, oracle_port, lat, dims, sched, masked, dtype):
    """tslb_cuda_init_state: initialize_regularized on the device from host
    node states (the e2e input path) == the port's initialize_regularized,
    bit for bit, then the same fused steps -- with f(0) pending under M
    (downloaded before the first step) and stored under F1."""
    L = T.lattice_of(lat)
    n = int(np.prod(dims))
    nm = 1 + L.dim + L.npineq
    rng = np.random.default_rng(17)
    st = rng.uniform(-0.02, 0.02, (nm, n))
    st[0] += 1.0
    st[1 + L.dim:] *= 0.01
    st = st.astype(dtype)
    solid = random_solid(dims, 0.15, 3) if masked else None
    state10 = st if L.dim == 3 else np.concatenate([st[:3], np.zeros((1, n), dtype), st[3:5], np.zeros((1, n), dtype),
                                                    st[5:6], np.zeros((2, n), dtype)])
    f0 = oracle_port.init_regularized(lat, dims, state10, solid)
    faces = zwalls_3d() if L.dim == 3 else O.lid_cavity(0.05)
    for read_first in (True, False):
        dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.3, spec_of(faces), dtype, 1, solid)
        try:
            if dev.schedule != sched:
                dev.set_schedule(sched)
            dev.init_state(st)
            if read_first:
                fluid = np.ones(n, bool) if solid is None else solid == 0
                assert_bitwise(dev.download_f(), f0, f"{lat} {sched} f(0)", fluid)
            dev.step(4)
            fg = dev.download_f()
        finally:
            dev.close()
        fo = f0.copy()
        oracle_port.single_run(lat, dims, 1.3, faces, fo, None, 4, 0, solid)
        fluid = np.ones(n, bool) if solid is None else solid == 0
        assert_bitwise(fg, fo, f"{lat} {sched} f(4) after init_state (read f(0) first: {read_first})", fluid)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("lat,dims,sched", [
    ("d3q19", (32, 16, 6), "m"), ("d3q19", (32, 16, 6), "f1"), ("d3q27", (32, 8, 5), "m"), ("d2q9", (45, 17, 1), "m")])
def test_init_equilibrium_is_init_state_with_zero_pi(gpu, oracle_port, lat, dims, sched, dtype):
    """tslb_cuda_init_equilibrium (rho and u only, Pi^neq = 0: the reference
    driver's start, tslb_main.cpp:115-122) == the port's initialize_regularized
    of the same states with zero Pi, bit for bit, before and after steps; on
    one handle after a full init_state (the state buffer changes size) and
    the other way round."""
    L = T.lattice_of(lat)
    n = int(np.prod(dims))
    nm = 1 + L.dim + L.npineq
    rng = np.random.default_rng(23)
    st = rng.uniform(-0.02, 0.02, (nm, n))
    st[0] += 1.0
    st[1 + L.dim:] *= 0.01
    st = st.astype(dtype)
    st0 = st.copy()
    st0[1 + L.dim:] = 0
    zero = np.zeros((1, n), dtype)
    state10 = st0 if L.dim == 3 else np.concatenate([st0[:3], zero, st0[3:5], zero, st0[5:6], zero, zero])
    f0 = oracle_port.init_regularized(lat, dims, state10, None)
    faces = zwalls_3d() if L.dim == 3 else O.lid_cavity(0.05)
    fo = f0.copy()
    oracle_port.single_run(lat, dims, 1.3, faces, fo, None, 3, 0, None)
    dev = T.DeviceSolver(lat, T.GridDims(*dims), 1.3, spec_of(faces), dtype, 1, None)
    try:
        if dev.schedule != sched:
            dev.set_schedule(sched)
        for order in ("state first", "equilibrium first"):
            if order == "state first":
                dev.init_state(st)
                dev.step(1)
                dev.init_equilibrium(np.ascontiguousarray(st[:1 + L.dim]))
            else:
                dev.init_equilibrium(np.ascontiguousarray(st[:1 + L.dim]))
                dev.step(2)
                dev.init_state(st0)
            assert_bitwise(dev.download_f(), f0, f"{lat} {sched} f(0), {order}")
            dev.step(3)
            assert_bitwise(dev.download_f(), fo, f"{lat} {sched} f(3), {order}")
        with pytest.raises(_lib.InvalidArgument):
            dev.init_equilibrium(st)
    finally:
        dev.close()
