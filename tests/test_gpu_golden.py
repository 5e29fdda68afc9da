"""GPU: the CUDA path reproduces the reference-generated golden fixtures bit
for bit (these travel with the repo; /root/reference is not on the box)."""
import os

import numpy as np
import pytest

from paper_2304_06437_b200 import tslb as T

import golden_cases as G
from helpers import assert_bitwise, spec_of

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("path", G.single_cases(), ids=os.path.basename)
def test_gpu_reproduces_single_golden(gpu, path):
    d = G.load(path)
    dev = T.DeviceSolver(d["lat"], T.GridDims(*d["dims"]), float(d["omega"]), spec_of(d["faces"]), d["f0"].dtype, 1,
                         d["solid"])
    dev.upload_f(d["f0"])
    dev.step(int(d["steps"]))
    fluid = np.ones(d["f0"].shape[1], bool) if d["solid"] is None else d["solid"] == 0
    assert_bitwise(dev.download_f(), d["f"], "f", fluid)
    L = T.lattice_of(d["lat"])
    mo = np.concatenate([dev.download_field("rho")[None], dev.download_field("mom").reshape(L.dim, -1),
                         dev.download_field("pineq").reshape(L.npineq, -1)])
    assert_bitwise(mo, d["moments"], "moments", fluid)
    geo = dev.geometry()
    assert_bitwise(geo.slow_mask, d["slow_mask"], "slow_mask")
    assert geo.n_fluid == int(d["n_fluid"])
    dev.close()


@pytest.mark.parametrize("path", G.two_cases(), ids=os.path.basename)
def test_gpu_reproduces_two_golden(gpu, path):
    d = G.load(path)
    c = G.color_dict(d)
    cp = T.ColorParams(sigma=c["sigma"], beta=c["beta"], nci_strength=c["nci_strength"], nci_reach=c["nci_reach"],
                       eps_bulk=c["eps_bulk"], grad_threshold=c["grad_threshold"],
                       form=T.PerturbationForm.Linear if c["linear"] else T.PerturbationForm.Squared)
    dev = T.DeviceSolver(d["lat"], T.GridDims(*d["dims"]), float(d["omega"]), spec_of(d["faces"]), d["fr0"].dtype, 2,
                         d["solid"], cp)
    dev.upload_f(d["fr0"], 0)
    dev.upload_f(d["fb0"], 1)
    dev.step(int(d["steps"]))
    fluid = np.ones(d["fr0"].shape[1], bool) if d["solid"] is None else d["solid"] == 0
    assert_bitwise(dev.download_f(0), d["fr"], "fr", fluid)
    assert_bitwise(dev.download_f(1), d["fb"], "fb", fluid)
    for k in ("rho_r", "rho_b", "rho", "phi", "nci_flag"):
        assert_bitwise(dev.download_field(k), d[k], k, None if k == "nci_flag" else fluid)
    for k in ("mom", "pineq", "gradphi"):
        assert_bitwise(np.reshape(dev.download_field(k), d[k].shape), d[k], k, fluid)
    dev.close()


def test_gpu_cavity_digest(gpu):
    """C1 end to end on the GPU: digest equals the reference's 6902b6f24d59100a."""
    g = T.GridDims(256, 256, 1)
    sim = T.SingleFluidSim(T.D2Q9, g, T.CollisionParams(T.omega_from_nu(0.064)), T.BoundarySpec.lid_cavity(0.025))
    T.initialize_regularized(sim.fields(), sim.geometry(), lambda i, j, k: (1.0, 0, 0, 0, 0, 0, 0, 0, 0, 0), T.D2Q9)
    sim.run(1000)
    assert T.fnv1a(sim.view().f) == 0x6902B6F24D59100A
