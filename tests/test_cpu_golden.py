"""CPU: the oracle port reproduces the reference-generated golden fixtures
(tests/golden/, made by make_golden.py from oracle/_ref) bit for bit, and
the reference's own known-answer values."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2304_06437_b200 import tslb as T

import golden_cases as G
from helpers import assert_bitwise


@pytest.mark.parametrize("path", G.single_cases(), ids=os.path.basename)
def test_port_reproduces_single_golden(oracle_port, path):
    d = G.load(path)
    f, m = d["f0"].copy(), np.zeros_like(d["moments"])
    oracle_port.single_run(d["lat"], d["dims"], float(d["omega"]), d["faces"], f, m, int(d["steps"]), 0, d["solid"])
    assert_bitwise(f, d["f"], "f")
    assert_bitwise(m, d["moments"], "moments")
    so, sl, nf = oracle_port.classify(d["lat"], d["dims"], d["faces"], d["solid"])
    assert_bitwise(sl, d["slow_mask"], "slow_mask")
    assert nf == int(d["n_fluid"])


@pytest.mark.parametrize("path", G.two_cases(), ids=os.path.basename)
def test_port_reproduces_two_golden(oracle_port, path):
    d = G.load(path)
    fr, fb = d["fr0"].copy(), d["fb0"].copy()
    out = oracle_port.two_run(d["lat"], d["dims"], float(d["omega"]), G.color_dict(d), d["faces"], fr, fb,
                              int(d["steps"]), False, 0, d["solid"])
    assert_bitwise(fr, d["fr"], "fr")
    assert_bitwise(fb, d["fb"], "fb")
    for k in ("rho_r", "rho_b", "rho", "mom", "pineq", "phi", "gradphi", "nci_flag"):
        assert_bitwise(out[k], d[k], k)


def test_host_initialisers_bitwise_vs_oracle(oracle_port):
    """tslb.initialize_regularized / initialize_colors (numpy, product host
    side) == the oracle's restatement of kernels.hpp:295-311 and
    multicomponent.hpp:427-449, in float and double."""
    for dt in (np.float64, np.float32):
        dims = (12, 10, 6)
        rng = np.random.default_rng(3)
        st = rng.uniform(-0.01, 0.01, (10, 720)).astype(dt)
        st[0] += 1
        s = T.allocate_fields(T.GridDims(*dims), T.D3Q19, dt)
        T.initialize_regularized(s, None, lambda i, j, k: tuple(st), T.D3Q19)
        assert_bitwise(s.f, oracle_port.init_regularized("d3q19", dims, st), "init_regularized")
        cs = rng.uniform(0, 1, (5, 720)).astype(dt)
        cs[2:] *= 0.02
        t = T.allocate_two_fluid(T.GridDims(*dims), T.D3Q19, dt)
        T.initialize_colors(t, None, lambda i, j, k: tuple(cs), T.D3Q19)
        fr, fb = oracle_port.init_colors("d3q19", dims, cs)
        assert_bitwise(t.fr, fr, "fr")
        assert_bitwise(t.fb, fb, "fb")


def test_cavity_digest_matches_survey_probe(oracle_port):
    """D2Q9 cavity 256^2 x 1000 fp64: digest 6902b6f24d59100a, the value the
    survey measured on the reference itself."""
    g = np.load(os.path.join(G.GOLDEN, "cavity_c1_digest.npz"))
    assert int(g["digest"]) == 0x6902B6F24D59100A
    st = np.zeros((10, 256 * 256))
    st[0] = 1.0
    f = oracle_port.init_regularized("d2q9", (256, 256, 1), st)
    oracle_port.single_run("d2q9", (256, 256, 1), T.omega_from_nu(0.064), O.lid_cavity(0.025), f, None, 1000, 0)
    assert oracle_port.fnv1a(f) == 0x6902B6F24D59100A


def test_known_answers():
    # census (unit_analysis_bench.cpp:274-290)
    c = T.count_kernel_cost(T.D3Q19, 8)
    assert (c.flops, c.bytes) == (377, 464)
    assert T.count_kernel_cost(T.D3Q19, 4).bytes == 232
    c2 = T.count_kernel_cost(T.D2Q9, 8)
    assert (c2.flops, c2.bytes) == (172, 240)
    # FNV-1a of "a" (unit_analysis_bench.cpp:313-322)
    assert T.fnv1a(b"a") == 0xAF63DC4C8601EC8C
    # roofline bound 2.079e12 style: min(peak, bw * I)
    # ledger (unit_lattice_fields.cpp:190-215): 15/21 and 29/42 arrays
    for L, fused, flip in ((T.D2Q9, 15, 21), (T.D3Q19, 29, 42)):
        assert L.q + 1 + L.dim + L.npineq == fused and 2 * L.q + 1 + L.dim == flip


@pytest.mark.parametrize("lat", ["d2q9", "d3q19", "d3q27"])
def test_lattice_moment_conditions(lat):
    """validate_moments (lattice.hpp:155-244) on all three velocity sets,
    including the new D3Q27 tables and its B weights."""
    L = T.lattice_of(lat)
    c = np.array(L.c, float)
    t = np.array([a / b for a, b in L.t_rat])
    b = np.array([a / bb for a, bb in L.b_rat])
    D = L.dim
    cs2, cs4 = 1 / 3, 1 / 9
    assert abs(t.sum() - 1) < 1e-14
    assert np.abs(t @ c).max() < 1e-15
    assert np.abs(np.einsum("a,ai,aj->ij", t, c, c)[:D, :D] - cs2 * np.eye(D)).max() < 1e-15
    iso = np.einsum("a,ai,aj,ak,al->ijkl", t, c, c, c, c)[:D, :D, :D, :D]
    I = np.eye(D)
    want = cs4 * (np.einsum("ij,kl->ijkl", I, I) + np.einsum("ik,jl->ijkl", I, I) + np.einsum("il,jk->ijkl", I, I))
    assert np.abs(iso - want).max() < 1e-15
    opp = L.opp
    assert all(opp[opp[a]] == a and np.all(c[opp[a]] == -c[a]) for a in range(L.q))
    assert abs(b.sum() - cs2) < 1e-15 and np.abs(b @ c).max() < 1e-15
    assert np.abs(np.einsum("a,ai,aj->ij", b, c, c)[:D, :D] - cs2 * np.eye(D)).max() < 1e-15
