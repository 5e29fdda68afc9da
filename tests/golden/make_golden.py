"""Generate golden fixtures from the UNMODIFIED reference build.

    make -C oracle ref && python tests/golden/make_golden.py

Runs oracle/_ref/libtslb_ref.so (the reference headers compiled with the
reference's Release flags, oracle/Makefile) on small seeded inputs and stores
inputs and outputs as tests/golden/*.npz. These fixtures travel with the repo
to the GPU box, where /root/reference does not exist: the GPU tests and the
oracle port are both checked against them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import oracle as O  # noqa: E402

from helpers import block_solid, corner_box_3d, droplet_state, mixed_2d, random_solid, zwalls_3d  # noqa: E402

SINGLE = {
    "d2q9_periodic": ("d2q9", (16, 16, 1), O.periodic(), None, 1.31, 5),
    "d2q9_lid": ("d2q9", (20, 16, 1), O.lid_cavity(0.05), None, 1.7, 7),
    "d2q9_mixed_block": ("d2q9", (16, 16, 1), mixed_2d(), block_solid((16, 16, 1), (6, 5, 0), (10, 8, 1)), 1.31, 5),
    "d3q19_zwalls": ("d3q19", (8, 7, 6), zwalls_3d(), None, 0.77, 4),
    "d3q19_corner_box": ("d3q19", (9, 8, 7), corner_box_3d(), None, 1.9, 4),
    "d3q19_box_random": ("d3q19", (10, 9, 8), O.closed_box(), random_solid((10, 9, 8), 0.08, 7), 1.2, 4),
}
TWO = {
    "d2q9_two_periodic_nci": ("d2q9", (24, 20, 1), O.periodic(), None, dict(sigma=0.03, nci_strength=0.1,
                                                                            eps_bulk=0.2)),
    "d2q9_two_mixed_block": ("d2q9", (24, 20, 1), mixed_2d(), block_solid((24, 20, 1), (3, 2, 0), (7, 5, 1)),
                             dict(sigma=0.02)),
    "d3q19_two_zwalls_linear": ("d3q19", (10, 9, 8), zwalls_3d(), None, dict(sigma=0.02, linear=True)),
}


def main():
    ref = O.Oracle("ref")
    port = O.Oracle("port")
    for name, (lat, dims, faces, solid, omega, steps) in SINGLE.items():
        for dt in (np.float64, np.float32):
            f0 = O.random_state(lat, dims, 2024, dt, solid)
            f = f0.copy()
            m = np.zeros((O.moments_layout(lat), f.shape[1]), dt)
            ref.single_run(lat, dims, omega, faces, f, m, steps, 0, solid)
            so, sl, nf = ref.classify(lat, dims, faces, solid)
            kinds, uw = O.faces_arrays(faces)
            np.savez_compressed(os.path.join(HERE, f"{name}_{np.dtype(dt).name}.npz"), lat=lat, dims=dims,
                                kinds=kinds, uw=uw, solid=np.zeros(0, np.uint8) if solid is None else solid,
                                omega=omega, steps=steps, f0=f0, f=f, moments=m, slow_mask=sl, n_fluid=nf)
    for name, (lat, dims, faces, solid, color) in TWO.items():
        for dt in (np.float64, np.float32):
            st = droplet_state(dims, min(dims[:2]) / 4, dt, (0.01, -0.005, 0.002 if dims[2] > 1 else 0.0))
            fr0, fb0 = port.init_colors(lat, dims, st, solid)
            fr, fb = fr0.copy(), fb0.copy()
            out = ref.two_run(lat, dims, 1.2, color, faces, fr, fb, 6, False, 0, solid)
            kinds, uw = O.faces_arrays(faces)
            np.savez_compressed(os.path.join(HERE, f"{name}_{np.dtype(dt).name}.npz"), lat=lat, dims=dims,
                                kinds=kinds, uw=uw, solid=np.zeros(0, np.uint8) if solid is None else solid,
                                omega=1.2, steps=6, color=np.array([color.get("sigma", 0.01), color.get("beta", 0.7),
                                                                    color.get("nci_strength", 0.0),
                                                                    color.get("eps_bulk", 0.02), 1e-6]),
                                color_i=np.array([color.get("nci_reach", 3), 1 if color.get("linear") else 0]),
                                state=st, fr0=fr0, fb0=fb0, fr=fr, fb=fb,
                                **{k: out[k] for k in ("rho_r", "rho_b", "rho", "mom", "pineq", "phi", "gradphi",
                                                       "nci_flag")})
    # cavity C1 digest after 1000 steps (6902b6f24d59100a)
    f = np.zeros((9, 256 * 256))
    st = np.zeros((10, 256 * 256))
    st[0] = 1.0
    f = port.init_regularized("d2q9", (256, 256, 1), st)
    ref.single_run("d2q9", (256, 256, 1), 1.0 / (0.064 / (1.0 / 3.0) + 0.5), O.lid_cavity(0.025), f, None, 1000, 0,
                   None, workers=os.cpu_count())
    np.savez_compressed(os.path.join(HERE, "cavity_c1_digest.npz"), digest=np.uint64(ref.fnv1a(f)),
                        rho_sum=f.sum())
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
