"""CPU: the plain-C oracle restatement is bit-identical to the UNMODIFIED
reference headers (oracle/_ref) on the reference's own scenario families
(unit_collision_stream.cpp:269-330, acceptance.cpp:101-135,
unit_multicomponent.cpp), for double and float storage."""
import numpy as np
import pytest

from oracle import oracle as O

from helpers import assert_bitwise, block_solid, corner_box_3d, droplet_state, mixed_2d, random_solid, zwalls_3d

SINGLE = [
    ("d2q9", (16, 16, 1), O.periodic(), None, 1.31),
    ("d2q9", (16, 12, 1), O.closed_box(), None, 0.6),
    ("d2q9", (20, 16, 1), O.lid_cavity(0.05), None, 1.7),
    ("d2q9", (16, 16, 1), mixed_2d(), block_solid((16, 16, 1), (6, 5, 0), (10, 8, 1)), 1.31),
    ("d3q19", (8, 7, 6), zwalls_3d(), None, 0.77),
    ("d3q19", (9, 8, 7), corner_box_3d(), None, 1.9),
    ("d3q19", (10, 9, 8), O.closed_box(), random_solid((10, 9, 8), 0.08, 7), 1.2),
]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("case", SINGLE, ids=lambda c: f"{c[0]}-{c[1]}")
def test_port_equals_reference_single(oracle_port, oracle_ref, case, mode, dtype):
    lat, dims, faces, solid, omega = case
    f = O.random_state(lat, dims, 1, dtype, solid)
    nm = O.moments_layout(lat)
    m = np.zeros((nm, f.shape[1]), dtype)
    if mode == 3:
        m[:] = np.random.default_rng(5).uniform(-0.01, 0.01, m.shape).astype(dtype)
        m[0] += 1
    f1, f2, m1, m2 = f.copy(), f.copy(), m.copy(), m.copy()
    oracle_port.single_run(lat, dims, omega, faces, f1, m1, 4, mode, solid)
    oracle_ref.single_run(lat, dims, omega, faces, f2, m2, 4, mode, solid)
    assert_bitwise(f1, f2, "f")
    assert_bitwise(m1, m2, "moments")


def test_fused_equals_two_buffer_reference(oracle_port):
    """acceptance criterion 1 restated on the port: fused == reference_step."""
    for lat, dims, faces, solid, omega in SINGLE:
        f = O.random_state(lat, dims, 20240817, np.float64, solid)
        a, b = f.copy(), f.copy()
        oracle_port.single_run(lat, dims, omega, faces, a, None, 10, 0, solid)
        oracle_port.single_run(lat, dims, omega, faces, b, None, 10, 1, solid)
        fluid = np.ones(f.shape[1], bool) if solid is None else solid == 0
        assert_bitwise(a, b, f"{lat} fused vs two-buffer", fluid)


TWO = [
    ("d2q9", (24, 20, 1), O.periodic(), None),
    ("d2q9", (24, 20, 1), mixed_2d(), block_solid((24, 20, 1), (3, 2, 0), (7, 5, 1))),
    ("d3q19", (10, 9, 8), zwalls_3d(), None),
]
COLORS = [dict(sigma=0.02), dict(sigma=0.02, linear=True), dict(sigma=0.03, nci_strength=0.1, eps_bulk=0.2)]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("color", COLORS, ids=["squared", "linear", "nci"])
@pytest.mark.parametrize("case", TWO, ids=lambda c: f"{c[0]}-{c[1]}")
def test_port_equals_reference_two(oracle_port, oracle_ref, case, color, dtype):
    lat, dims, faces, solid = case
    st = droplet_state(dims, min(dims[:2]) / 4, dtype, (0.01, -0.005, 0.0))
    fr, fb = oracle_port.init_colors(lat, dims, st, solid)
    a = oracle_port.two_run(lat, dims, 1.2, color, faces, fr1 := fr.copy(), fb1 := fb.copy(), 5, True, 0, solid)
    b = oracle_ref.two_run(lat, dims, 1.2, color, faces, fr2 := fr.copy(), fb2 := fb.copy(), 5, True, 0, solid)
    assert_bitwise(fr1, fr2, "fr")
    assert_bitwise(fb1, fb2, "fb")
    for k in ("rho_r", "rho_b", "rho", "mom", "pineq", "phi", "gradphi", "nci_flag"):
        assert_bitwise(a[k], b[k], k)


@pytest.mark.parametrize("lat,dims,faces,solid", [
    ("d2q9", (8, 6, 1), O.closed_box(), None),
    ("d2q9", (7, 7, 1), O.periodic(), block_solid((7, 7, 1), (3, 3, 0), (4, 4, 1))),
    ("d3q19", (5, 5, 5), O.closed_box(), None),
    ("d3q19", (6, 5, 4), zwalls_3d(), random_solid((6, 5, 4), 0.2, 1)),
])
def test_classify_port_equals_reference(oracle_port, oracle_ref, lat, dims, faces, solid):
    a = oracle_port.classify(lat, dims, faces, solid)
    b = oracle_ref.classify(lat, dims, faces, solid)
    assert_bitwise(a[0], b[0], "solid")
    assert_bitwise(a[1], b[1], "slow")
    assert a[2] == b[2]


def test_half_periodic_axis_rejected_like_reference(oracle_port, oracle_ref):
    f = O.periodic()
    f[2] = ("wall", (0, 0, 0))
    for o in (oracle_port, oracle_ref):
        with pytest.raises(ValueError, match="axis 1"):
            o.classify("d2q9", (8, 8, 1), f)


def test_ref_full_workload_geometry_expansion(oracle_ref):
    """bench.py --impl reference's whole-workload run (tslbref_time_tgv)
    expands classify_nodes' 3x3x3 slow masks instead of classifying 10^9
    nodes serially: the same f afterwards as with the full classification."""
    import ctypes as C
    fn = oracle_ref.lib.tslbref_time_tgv
    fn.argtypes = [C.c_int] * 4 + [C.c_double, C.c_double, C.c_long, C.c_long, C.c_int, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
    digests = []
    for full in (0, 1):
        ti, ts, dg = C.c_double(), C.c_double(), C.c_uint64()
        assert fn(1, 12, 10, 9, 1.6, 0.03, 3, 1, 2, full, C.byref(ti), C.byref(ts), C.byref(dg)) == 0
        digests.append(dg.value)
    assert digests[0] == digests[1]
