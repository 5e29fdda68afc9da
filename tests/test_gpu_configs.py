"""Parity at the BASELINE.json configurations' own sizes.

Each case runs the exact bench path on the device -- device analytic
initialisation, the default schedule, no f until something reads it -- and
the UNMODIFIED reference build (oracle/_ref, WorkerPool over the host cores)
from the same f(0): a second device solver initialised the same way hands
f(0) over (download_f materialises the analytic state). f(N) and the moment
arrays m(N-1) (two-fluid: every field the reference stores) must agree bit
for bit (kernels.hpp:209-215, multicomponent.hpp:405-414).

  C2  D3Q19 Taylor-Green 512^3, fp32 storage (fp64 node math) and fp64 storage
  C4  D3Q19 colour-gradient droplet 512^3, fp32
  C0  the headline workload's lattice/precision/path on a 1024 x 1024 x 64
      periodic box (the full 1024^3 state with the reference's copy exceeds
      the box's host memory)
  C3  D3Q27 Poiseuille channel 1024 x 1024 x 32 (walls, body force) against
      the C restatement -- the reference has no D3Q27 (unpinned by
      construction)

Host memory: the largest case (C2 fp64) holds ~90 GB at its peak.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2304_06437_b200 import tslb as T

from helpers import assert_bitwise

pytestmark = pytest.mark.gpu

WORKERS = os.cpu_count() or 1


def _moments(dev, lat):
    L = T.lattice_of(lat)
    return np.concatenate([dev.download_field("rho")[None], dev.download_field("mom").reshape(L.dim, -1),
                           dev.download_field("pineq").reshape(L.npineq, -1)])


def _channel_spec():
    s = T.BoundarySpec.all_periodic()
    s.faces[T.YMin] = T.Face(T.FaceKind.NoSlipWall)
    s.faces[T.YMax] = T.Face(T.FaceKind.NoSlipWall)
    return s


def _channel_faces():
    f = O.periodic()
    f[2] = ("wall", (0, 0, 0))
    f[3] = ("wall", (0, 0, 0))
    return f


def _single(lat, dims, omega, spec, dtype, init, amp, steps, force=None):
    """(f0, f(N), m(N-1)) of the bench path on the device."""
    g = T.GridDims(*dims)
    dev = T.DeviceSolver(lat, g, omega, spec, dtype)
    try:
        if force:
            dev.set_body_force(*force)
        dev.init_analytic(init, amp)
        f0 = dev.download_f()
    finally:
        dev.close()
    dev = T.DeviceSolver(lat, g, omega, spec, dtype)
    try:
        if force:
            dev.set_body_force(*force)
        assert dev.schedule == "m"
        dev.init_analytic(init, amp)  # bench path: m(0) written directly, f never stored
        dev.step(steps)
        mg = _moments(dev, lat)
        fg = dev.download_f()
    finally:
        dev.close()
    return f0, fg, mg


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
def test_c2_taylor_green_512_vs_reference_build(gpu, oracle_ref, dtype):
    lat, dims, om, steps = "d3q19", (512, 512, 512), 1.6, 5
    f0, fg, mg = _single(lat, dims, om, T.BoundarySpec.all_periodic(), dtype, "taylor_green", 0.03, steps)
    mo = np.zeros_like(mg)
    oracle_ref.single_run(lat, dims, om, O.periodic(), f0, mo, steps, 0, None, WORKERS)
    assert_bitwise(mg, mo, "C2 m(N-1)")
    del mg, mo
    assert_bitwise(fg, f0, "C2 f(N)")


def test_c0_headline_slab_vs_reference_build(gpu, oracle_ref):
    lat, dims, om, steps = "d3q19", (1024, 1024, 64), 1.6, 3
    f0, fg, mg = _single(lat, dims, om, T.BoundarySpec.all_periodic(), np.float32, "taylor_green", 0.03, steps)
    mo = np.zeros_like(mg)
    oracle_ref.single_run(lat, dims, om, O.periodic(), f0, mo, steps, 0, None, WORKERS)
    assert_bitwise(mg, mo, "1024x1024x64 m(N-1)")
    assert_bitwise(fg, f0, "1024x1024x64 f(N)")


def test_c3_channel_d3q27_vs_port(gpu, oracle_port):
    lat, dims, om, steps = "d3q27", (1024, 1024, 32), 1.0, 4
    nu = (1.0 / om - 0.5) / 3.0
    force = (8.0 * nu * 0.05 / float(dims[1]) ** 2, 0.0, 0.0)
    f0, fg, mg = _single(lat, dims, om, _channel_spec(), np.float32, "rest", 0.0, steps, force)
    mo = np.zeros_like(mg)
    oracle_port.set_body_force(*force)
    try:
        oracle_port.single_run(lat, dims, om, _channel_faces(), f0, mo, steps, 0)
    finally:
        oracle_port.set_body_force(0.0, 0.0, 0.0)
    assert_bitwise(mg, mo, "C3 m(N-1)")
    assert_bitwise(fg, f0, "C3 f(N)")


def test_c4_droplet_512_vs_reference_build(gpu, oracle_ref):
    lat, dims, om, steps = "d3q19", (512, 512, 512), 1 / 0.75, 4
    g = T.GridDims(*dims)
    color = T.ColorParams(sigma=0.03, beta=0.7)
    radius = 512 / 6.0

    def dev_():
        d = T.DeviceSolver(lat, g, om, T.BoundarySpec.all_periodic(), np.float32, 2, None, color)
        d.init_analytic("droplet", 0.0, radius)
        return d

    dev = dev_()
    try:
        fr, fb = dev.download_f(0), dev.download_f(1)
    finally:
        dev.close()
    dev = dev_()
    try:
        dev.step(steps)
        got = {k: dev.download_field(k) for k in ("rho_r", "rho_b", "rho", "mom", "pineq", "phi", "gradphi")}
        gr, gb = dev.download_f(0), dev.download_f(1)
    finally:
        dev.close()
    cd = dict(sigma=color.sigma, beta=color.beta, nci_strength=0.0, eps_bulk=color.eps_bulk,
              grad_threshold=color.grad_threshold, nci_reach=color.nci_reach)
    ref = oracle_ref.two_run(lat, dims, om, cd, O.periodic(), fr, fb, steps, False, 0, None, None, WORKERS)
    for k in ("rho_r", "rho_b", "rho", "mom", "pineq", "phi", "gradphi"):
        assert_bitwise(got[k], ref[k], f"C4 {k}")
    del got, ref
    assert_bitwise(gr, fr, "C4 f_red(N)")
    assert_bitwise(gb, fb, "C4 f_blue(N)")
