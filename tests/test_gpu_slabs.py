"""z-slab decomposition on ONE device through the local-copy transport
(tslb_cuda_link_local / group_step): the same kernels, ghost planes and
masked unpack as the NCCL path, checked bit for bit against the undivided
domain -- SURVEY.md §4's "single-GPU test of the decomposition" and §8(e)'s
GPU-count determinism."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_2304_06437_b200 import _lib
from paper_2304_06437_b200 import tslb as T

from helpers import assert_bitwise, random_solid, spec_of, zwalls_3d

pytestmark = pytest.mark.gpu


def split(nz, parts):
    return [(nz * p // parts, nz * (p + 1) // parts - nz * p // parts) for p in range(parts)]


def run_slabs(lat, dims, omega, faces, f0, steps, parts, solid=None, dtype=np.float64):
    g = T.GridDims(*dims)
    plane = dims[0] * dims[1]
    slabs = [T.DeviceSolver(lat, g, omega, spec_of(faces), dtype, 1, solid, slab=s) for s in split(dims[2], parts)]
    for sv, (z0, nzl) in zip(slabs, split(dims[2], parts)):
        sv.upload_f(np.ascontiguousarray(f0[:, z0 * plane:(z0 + nzl) * plane]))
    arr = (C.c_void_p * parts)(*[s.h.value for s in slabs])
    _lib.call("tslb_cuda_link_local", arr, parts)
    _lib.call("tslb_cuda_group_step", arr, parts, int(steps))
    f = np.concatenate([s.download_f() for s in slabs], axis=1)
    dig = np.concatenate([s.plane_digests()[0] for s in slabs], axis=1)
    for s in slabs:
        s.close()
    return f, dig


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("parts", [2, 3, 4])
@pytest.mark.parametrize("lat,faces,solid_frac", [
    ("d3q19", O.periodic(), 0.0),
    ("d3q19", zwalls_3d(), 0.0),
    ("d3q19", O.closed_box(), 0.0),
    ("d3q19", O.periodic(), 0.1),
    ("d3q27", zwalls_3d(), 0.05),
    ("d3q27", O.periodic(), 0.0),
])
def test_slabs_equal_single_domain(gpu, lat, faces, solid_frac, parts, dtype):
    dims = (12, 10, 12)
    solid = random_solid(dims, solid_frac, 3) if solid_frac else None
    f0 = O.random_state(lat, dims, 20240817, dtype, solid)
    one = T.DeviceSolver(lat, T.GridDims(*dims), 0.9, spec_of(faces), dtype, 1, solid)
    one.upload_f(f0)
    one.step(6)
    ref = one.download_f()
    dig1 = one.plane_digests()[0]
    one.close()
    got, dig = run_slabs(lat, dims, 0.9, faces, f0, 6, parts, solid, dtype)
    fluid = np.ones(f0.shape[1], bool) if solid is None else solid == 0
    assert_bitwise(got, ref, f"{parts} slabs vs one domain", fluid)
    if solid is None:
        # decomposition-independent digest
        assert np.array_equal(dig, dig1)


# --- M schedule on slabs: moment ghost planes instead of population halos ---
M_FACES = [
    ("periodic", O.periodic()),
    ("zwalls", zwalls_3d()),
    ("closed-box", O.closed_box()),
    ("xwall-moving", [("moving", (0.0, 0.02, -0.01)), ("wall", (0, 0, 0))] + [("periodic", (0, 0, 0))] * 4),
]


@pytest.mark.parametrize("lz", ["", "2"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("parts", [2, 3, 4])
@pytest.mark.parametrize("lat", ["d3q19", "d3q27"])
@pytest.mark.parametrize("name,faces", M_FACES, ids=[m[0] for m in M_FACES])
def test_mstep_slabs_equal_oracle(gpu, oracle_port, name, faces, lat, parts, dtype, lz, monkeypatch):
    """M-schedule slabs (boundary chunks, ghost-plane exchange, interior
    chunks; f rebuilt from ghost moments on download) are bit-identical to
    fused_step on the undivided domain, for any slab count."""
    if lz:  # several chunks, and 1-plane boundary chunks (boundary / exchange / interior)
        monkeypatch.setenv("TSLB_LZ", lz)
        monkeypatch.setenv("TSLB_LZB", "1")
    dims = (32, 16, 12)
    f0 = O.random_state(lat, dims, 77, dtype)
    g = T.GridDims(*dims)
    plane = dims[0] * dims[1]
    slabs = [T.DeviceSolver(lat, g, 1.25, spec_of(faces), dtype, 1, None, slab=s) for s in split(dims[2], parts)]
    try:
        assert all(s.schedule == "m" for s in slabs)
        for sv, (z0, nzl) in zip(slabs, split(dims[2], parts)):
            sv.upload_f(np.ascontiguousarray(f0[:, z0 * plane:(z0 + nzl) * plane]))
        arr = (C.c_void_p * parts)(*[s.h.value for s in slabs])
        _lib.call("tslb_cuda_link_local", arr, parts)
        _lib.call("tslb_cuda_group_step", arr, parts, 5)
        mo = np.concatenate([np.concatenate([s.download_field("rho")[None], s.download_field("mom").reshape(3, -1),
                                             s.download_field("pineq").reshape(6, -1)]) for s in slabs], axis=1)
        f = np.concatenate([s.download_f() for s in slabs], axis=1)
    finally:
        for s in slabs:
            s.close()
    ref = f0.copy()
    rmo = np.zeros((10, ref.shape[1]), dtype)
    oracle_port.single_run(lat, dims, 1.25, faces, ref, rmo, 5, 0)
    assert_bitwise(mo, rmo, f"M slabs x{parts} moments")
    assert_bitwise(f, ref, f"M slabs x{parts} f")


# --- the NCCL transport itself, on one device: a single-rank communicator ---
@pytest.mark.parametrize("sched", ["m", "f1"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("lzb", ["", "2"])
def test_nccl_self_exchange_equals_periodic_box(gpu, sched, dtype, lzb, monkeypatch):
    """One slab [0, nzl) of a 2*nzl box attached to a ONE-rank NCCL
    communicator: its up and down neighbour is itself, so every step ships
    its boundary planes (moment planes under M, pushed populations under F1)
    through ncclSend/ncclRecv to itself -- exactly a periodic box of height
    nzl. This exercises the multi-GPU step (boundary chunks, exchange on the
    comm stream, interior chunks, join) on real NCCL with one GPU."""
    monkeypatch.setenv("TSLB_LZ", "2")  # several z chunks per launch
    if lzb:  # M: 2-plane boundary chunks on the comm stream, the interior overlapped
        monkeypatch.setenv("TSLB_LZB", lzb)
    lat, nx, ny, nzl = "d3q19", 32, 16, 8
    f0 = O.random_state(lat, (nx, ny, nzl), 5, dtype)
    spec = spec_of(O.periodic())
    ref = T.DeviceSolver(lat, T.GridDims(nx, ny, nzl), 1.2, spec, dtype)
    slab = T.DeviceSolver(lat, T.GridDims(nx, ny, 2 * nzl), 1.2, spec, dtype, 1, None, slab=(0, nzl))
    try:
        for d in (ref, slab):
            d.set_schedule(sched)
        uid = (C.c_char * 128)()
        _lib.call("tslb_cuda_nccl_unique_id", uid)
        _lib.call("tslb_cuda_attach_nccl", slab.h, uid, 1, 0)
        for d in (ref, slab):
            d.upload_f(f0)
            d.step(7)
        assert_bitwise(slab.download_f(), ref.download_f(), f"NCCL self-exchange ({sched}) f")
        for fld in ("rho", "mom", "pineq"):
            assert_bitwise(slab.download_field(fld), ref.download_field(fld), f"NCCL self-exchange ({sched}) {fld}")
    finally:
        slab.close()
        ref.close()


# --- two-fluid z slabs: phi ghost planes + both species' population halos ---
def _two_cp():
    return T.ColorParams(sigma=0.02, beta=0.7)


def _droplet(dims, dtype):
    from helpers import droplet_state
    st = droplet_state(dims, min(dims[:2]) / 3.5, dtype, (0.01, -0.005, 0.004))
    return Oracle_port().init_colors("d3q19", dims, st, None)


def Oracle_port():
    return O.Oracle("port")


TWO_FACES = [
    ("periodic", O.periodic()),
    ("zwalls", zwalls_3d()),
    ("ywalls-staged", [("periodic", (0, 0, 0))] * 2 + [("wall", (0, 0, 0)), ("moving", (0.02, 0.0, 0.0))]
     + [("periodic", (0, 0, 0))] * 2),
]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("parts", [2, 3])
@pytest.mark.parametrize("name,faces", TWO_FACES, ids=[t[0] for t in TWO_FACES])
def test_two_fluid_slabs_equal_single_domain(gpu, name, faces, parts, dtype):
    dims = (20, 14, 12)
    fr, fb = _droplet(dims, dtype)
    plane = dims[0] * dims[1]
    one = T.DeviceSolver("d3q19", T.GridDims(*dims), 1.25, spec_of(faces), dtype, 2, None, _two_cp())
    one.upload_f(fr, 0)
    one.upload_f(fb, 1)
    one.step(5)
    ref = [one.download_f(0), one.download_f(1)] + [one.download_field(k) for k in ("phi", "gradphi", "rho")]
    one.close()
    slabs = [T.DeviceSolver("d3q19", T.GridDims(*dims), 1.25, spec_of(faces), dtype, 2, None, _two_cp(), slab=s)
             for s in split(dims[2], parts)]
    try:
        for sv, (z0, nzl) in zip(slabs, split(dims[2], parts)):
            sv.upload_f(np.ascontiguousarray(fr[:, z0 * plane:(z0 + nzl) * plane]), 0)
            sv.upload_f(np.ascontiguousarray(fb[:, z0 * plane:(z0 + nzl) * plane]), 1)
        arr = (C.c_void_p * parts)(*[s.h.value for s in slabs])
        _lib.call("tslb_cuda_link_local", arr, parts)
        _lib.call("tslb_cuda_group_step", arr, parts, 5)
        got = [np.concatenate([s.download_f(sp) for s in slabs], axis=1) for sp in (0, 1)]
        got.append(np.concatenate([s.download_field("phi") for s in slabs]))
        got.append(np.concatenate([s.download_field("gradphi").reshape(3, -1) for s in slabs], axis=1))
        got.append(np.concatenate([s.download_field("rho") for s in slabs]))
    finally:
        for s in slabs:
            s.close()
    for g, r, what in zip(got, ref, ["fr", "fb", "phi", "gradphi", "rho"]):
        assert_bitwise(np.reshape(g, np.shape(r)) if what != "gradphi" else g, np.reshape(r, np.shape(g)),
                       f"two-fluid {parts} slabs {what}")


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_two_fluid_nccl_self_exchange(gpu, dtype):
    """Two-fluid slab on a one-rank NCCL communicator == periodic box."""
    dims = (20, 14, 6)
    fr, fb = _droplet(dims, dtype)
    spec = spec_of(O.periodic())
    ref = T.DeviceSolver("d3q19", T.GridDims(*dims), 1.25, spec, dtype, 2, None, _two_cp())
    slab = T.DeviceSolver("d3q19", T.GridDims(dims[0], dims[1], 2 * dims[2]), 1.25, spec, dtype, 2, None, _two_cp(),
                          slab=(0, dims[2]))
    try:
        uid = (C.c_char * 128)()
        _lib.call("tslb_cuda_nccl_unique_id", uid)
        _lib.call("tslb_cuda_attach_nccl", slab.h, uid, 1, 0)
        for d in (ref, slab):
            d.upload_f(fr, 0)
            d.upload_f(fb, 1)
            d.step(6)
        for sp in (0, 1):
            assert_bitwise(slab.download_f(sp), ref.download_f(sp), f"two-fluid NCCL self-exchange species {sp}")
        assert_bitwise(slab.download_field("gradphi"), ref.download_field("gradphi"), "gradphi")
    finally:
        slab.close()
        ref.close()


# --- M on masked slabs: solid bits with ghost planes, solid-aware ghost push ---
@pytest.mark.parametrize("lz", ["", "2"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("parts", [2, 3, 4])
@pytest.mark.parametrize("lat,faces,frac", [
    ("d3q19", O.periodic(), 0.12),
    ("d3q19", zwalls_3d(), 0.3),
    ("d3q27", O.closed_box(), 0.1),
])
def test_mstep_masked_slabs(gpu, oracle_port, lat, faces, frac, parts, dtype, lz, monkeypatch):
    """Masked slabs run the M step too: every node (solid ones included)
    equals the undivided domain under F1, fluid nodes equal the oracle."""
    if lz:
        monkeypatch.setenv("TSLB_LZ", lz)
    dims = (32, 16, 12)
    solid = random_solid(dims, frac, 41)
    f0 = O.random_state(lat, dims, 13, dtype, solid)
    g = T.GridDims(*dims)
    plane = dims[0] * dims[1]
    L = T.lattice_of(lat)
    slabs = [T.DeviceSolver(lat, g, 1.1, spec_of(faces), dtype, 1, solid, slab=s) for s in split(dims[2], parts)]
    try:
        assert all(s.schedule == "m" for s in slabs)
        for sv, (z0, nzl) in zip(slabs, split(dims[2], parts)):
            sv.upload_f(np.ascontiguousarray(f0[:, z0 * plane:(z0 + nzl) * plane]))
        arr = (C.c_void_p * parts)(*[s.h.value for s in slabs])
        _lib.call("tslb_cuda_link_local", arr, parts)
        _lib.call("tslb_cuda_group_step", arr, parts, 5)
        mo = np.concatenate([np.concatenate([s.download_field("rho")[None], s.download_field("mom").reshape(L.dim, -1),
                                             s.download_field("pineq").reshape(L.npineq, -1)]) for s in slabs], axis=1)
        f = np.concatenate([s.download_f() for s in slabs], axis=1)
    finally:
        for s in slabs:
            s.close()
    one = T.DeviceSolver(lat, g, 1.1, spec_of(faces), dtype, 1, solid)
    try:
        one.set_schedule("f1")
        one.upload_f(f0)
        one.step(5)
        fo = one.download_f()
        moo = np.concatenate([one.download_field("rho")[None], one.download_field("mom").reshape(L.dim, -1),
                              one.download_field("pineq").reshape(L.npineq, -1)])
    finally:
        one.close()
    assert_bitwise(f, fo, f"masked M slabs x{parts} f (all nodes)")
    assert_bitwise(mo, moo, f"masked M slabs x{parts} moments (all nodes)")
    ref = f0.copy()
    rmo = np.zeros((O.moments_layout(lat), ref.shape[1]), dtype)
    oracle_port.single_run(lat, dims, 1.1, faces, ref, rmo, 5, 0, solid)
    fluid = solid == 0
    assert_bitwise(f, ref, "masked M slabs f vs oracle", fluid)
    assert_bitwise(mo, rmo, "masked M slabs moments vs oracle", fluid)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_nccl_self_exchange_masked(gpu, dtype, monkeypatch):
    """The masked M slab on real NCCL (one-rank communicator, its own
    neighbour): equals the periodic masked box of the slab's height."""
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
        uid = (C.c_char * 128)()
        _lib.call("tslb_cuda_nccl_unique_id", uid)
        _lib.call("tslb_cuda_attach_nccl", slab.h, uid, 1, 0)
        for d in (ref, slab):
            d.upload_f(f0)
            d.step(7)
        assert_bitwise(slab.download_f(), ref.download_f(), "masked NCCL self-exchange f")
        for fld in ("rho", "mom", "pineq"):
            assert_bitwise(slab.download_field(fld), ref.download_field(fld), f"masked NCCL self-exchange {fld}")
    finally:
        slab.close()
        ref.close()


@pytest.mark.parametrize("sched", ["m", "f1"])
def test_survey_decomposition_512x256x256(gpu, sched):
    """fields bit-identical for 1/2/4/8 slabs at
    512x256x256 (per-plane FNV digests of every population array, D3Q19
    periodic Taylor-Green, fp32 storage, fp64 node math), device-initialised
    on each slab from the global coordinates."""
    dims = (512, 256, 256)
    g = T.GridDims(*dims)
    spec = spec_of(O.periodic())
    steps = 4
    one = T.DeviceSolver("d3q19", g, 1.6, spec, np.float32)
    try:
        one.set_schedule(sched)
        one.init_analytic("taylor_green", 0.03)
        one.step(steps)
        ref = one.plane_digests()
    finally:
        one.close()
    for parts in (2, 4, 8):
        slabs = [T.DeviceSolver("d3q19", g, 1.6, spec, np.float32, 1, None, slab=s) for s in split(dims[2], parts)]
        try:
            for s in slabs:
                s.set_schedule(sched)
                s.init_analytic("taylor_green", 0.03)
            arr = (C.c_void_p * parts)(*[s.h.value for s in slabs])
            _lib.call("tslb_cuda_link_local", arr, parts)
            _lib.call("tslb_cuda_group_step", arr, parts, steps)
            dig = np.concatenate([s.plane_digests() for s in slabs], axis=2)
        finally:
            for s in slabs:
                s.close()
        assert np.array_equal(dig, ref), f"{parts} slabs ({sched}): plane digests differ"


# --- two-fluid slabs with the near-contact scan (NCI): phi and the flags keep
# nci_reach ghost planes; probes cross slab faces; ghost flags are ORed into
# their owners (multicomponent.hpp:202-238, 249-266) ---
def _nci_cp():
    return T.ColorParams(sigma=0.02, beta=0.7, nci_strength=0.01, nci_reach=3)


def _nci_film(dims, dtype):
    """Two red layers (cut to a disc) with thin blue films between them and
    across the periodic z wrap: the scan flags nodes in most planes,
    including the planes next to every slab face of 2 / 3 / 4 slabs."""
    nx, ny, nz = dims
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")

    def layer(z0, z1, w=0.6):
        return 0.5 * (np.tanh((k - z0) / w) - np.tanh((k - z1) / w))
    red = (layer(3.5, 6.6) + layer(9.4, 12.5)) * (np.hypot(i - (nx - 1) / 2, j - (ny - 1) / 2) < 5)
    phi = (2 * np.clip(red, 0, 1) - 1).ravel()
    st = np.zeros((5, phi.size))
    st[0], st[1], st[2], st[3] = 0.5 * (1 + phi), 0.5 * (1 - phi), 0.003, -0.002
    return Oracle_port().init_colors("d3q19", dims, st.astype(dtype))


NCI_FIELDS = ("phi", "gradphi", "rho", "nci_flag", "mom", "pineq")


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("parts", [2, 3, 4])
@pytest.mark.parametrize("name,faces", TWO_FACES[:2], ids=[t[0] for t in TWO_FACES[:2]])
def test_two_fluid_nci_slabs_equal_single_domain(gpu, oracle_port, name, faces, parts, dtype):
    dims, steps = (16, 12, 16), 4
    fr, fb = _nci_film(dims, dtype)
    plane = dims[0] * dims[1]
    one = T.DeviceSolver("d3q19", T.GridDims(*dims), 1.25, spec_of(faces), dtype, 2, None, _nci_cp())
    try:
        one.upload_f(fr, 0)
        one.upload_f(fb, 1)
        one.step(steps)
        ref = {"fr": one.download_f(0), "fb": one.download_f(1)}
        ref.update({k: one.download_field(k) for k in NCI_FIELDS})
    finally:
        one.close()
    assert ref["nci_flag"].sum() > 50, "the state should trigger the near-contact scan"
    slabs = [T.DeviceSolver("d3q19", T.GridDims(*dims), 1.25, spec_of(faces), dtype, 2, None, _nci_cp(), slab=s)
             for s in split(dims[2], parts)]
    try:
        for sv, (z0, nzl) in zip(slabs, split(dims[2], parts)):
            sv.upload_f(np.ascontiguousarray(fr[:, z0 * plane:(z0 + nzl) * plane]), 0)
            sv.upload_f(np.ascontiguousarray(fb[:, z0 * plane:(z0 + nzl) * plane]), 1)
        arr = (C.c_void_p * parts)(*[s.h.value for s in slabs])
        _lib.call("tslb_cuda_link_local", arr, parts)
        _lib.call("tslb_cuda_group_step", arr, parts, steps)
        got = {"fr": np.concatenate([s.download_f(0) for s in slabs], axis=1),
               "fb": np.concatenate([s.download_f(1) for s in slabs], axis=1)}
        for k in NCI_FIELDS:
            parts_k = [s.download_field(k) for s in slabs]
            got[k] = np.concatenate(parts_k, axis=-1)
    finally:
        for s in slabs:
            s.close()
    for k in got:
        assert_bitwise(got[k], ref[k], f"NCI {parts} slabs {k}")
    # and the single domain against the oracle (the reference restatement)
    fro, fbo = fr.copy(), fb.copy()
    cd = dict(sigma=0.02, beta=0.7, nci_strength=0.01, nci_reach=3)
    res = oracle_port.two_run("d3q19", dims, 1.25, cd, faces, fro, fbo, steps)
    assert_bitwise(ref["fr"], fro, "NCI single domain vs oracle fr")
    assert_bitwise(ref["nci_flag"], res["nci_flag"], "NCI single domain vs oracle flags")


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_two_fluid_nci_nccl_self_exchange(gpu, dtype):
    """NCI slab on a one-rank NCCL communicator (its own neighbour above and
    below) == the periodic box: phi ghost planes of depth nci_reach, the
    probes across both faces and the flag OR exchange all go through NCCL."""
    dims = (16, 12, 16)
    fr, fb = _nci_film(dims, dtype)
    spec = spec_of(O.periodic())
    ref = T.DeviceSolver("d3q19", T.GridDims(*dims), 1.25, spec, dtype, 2, None, _nci_cp())
    slab = T.DeviceSolver("d3q19", T.GridDims(dims[0], dims[1], 2 * dims[2]), 1.25, spec, dtype, 2, None, _nci_cp(),
                          slab=(0, dims[2]))
    try:
        uid = (C.c_char * 128)()
        _lib.call("tslb_cuda_nccl_unique_id", uid)
        _lib.call("tslb_cuda_attach_nccl", slab.h, uid, 1, 0)
        for d in (ref, slab):
            d.upload_f(fr, 0)
            d.upload_f(fb, 1)
            d.step(5)
        for sp in (0, 1):
            assert_bitwise(slab.download_f(sp), ref.download_f(sp), f"NCI NCCL self-exchange species {sp}")
        for k in NCI_FIELDS:
            assert_bitwise(slab.download_field(k), ref.download_field(k), f"NCI NCCL self-exchange {k}")
        assert ref.download_field("nci_flag").sum() > 50
    finally:
        slab.close()
        ref.close()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_init_state_on_a_slab(gpu, oracle_port, dtype, monkeypatch):
    """tslb_cuda_init_state on a slab (the local planes' node states) with
    the M step over a one-rank NCCL communicator == the periodic box
    initialised the same way, and == the oracle's initialize_regularized +
    fused_step."""
    monkeypatch.setenv("TSLB_LZB", "2")
    lat, nx, ny, nzl = "d3q19", 32, 8, 8
    n = nx * ny * nzl
    rng = np.random.default_rng(3)
    st = rng.uniform(-0.02, 0.02, (10, n))
    st[0] += 1.0
    st[4:] *= 0.01
    st = st.astype(dtype)
    spec = spec_of(O.periodic())
    ref = T.DeviceSolver(lat, T.GridDims(nx, ny, nzl), 1.2, spec, dtype)
    slab = T.DeviceSolver(lat, T.GridDims(nx, ny, 2 * nzl), 1.2, spec, dtype, 1, None, slab=(0, nzl))
    try:
        uid = (C.c_char * 128)()
        _lib.call("tslb_cuda_nccl_unique_id", uid)
        _lib.call("tslb_cuda_attach_nccl", slab.h, uid, 1, 0)
        for d in (ref, slab):
            d.init_state(st)
            d.step(6)
        fs = slab.download_f()
        assert_bitwise(fs, ref.download_f(), "init_state slab vs box f")
        fo = oracle_port.init_regularized(lat, (nx, ny, nzl), st)
        oracle_port.single_run(lat, (nx, ny, nzl), 1.2, O.periodic(), fo, None, 6, 0)
        assert_bitwise(fs, fo, "init_state slab vs oracle f")
    finally:
        slab.close()
        ref.close()
