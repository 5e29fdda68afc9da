"""2-D small-domain paths across domain sizes (measurement only): the
persistent launch with temporal blocking, without it (one grid barrier per
pass), and per-pass launches replayed from CUDA graphs (TSLB_PERSIST=0);
D2Q9 periodic Taylor-Green and lid cavity, fp64."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

from paper_2304_06437_b200 import tslb as T  # noqa: E402


def run(n, faces, tb, steps=400, persist=True):
    os.environ["TSLB_TB2D"] = "1" if tb else "0"
    os.environ["TSLB_PERSIST"] = "1" if persist else "0"
    spec = T.BoundarySpec.all_periodic() if faces == "periodic" else T.BoundarySpec.lid_cavity(0.05)
    dev = T.DeviceSolver("d2q9", T.GridDims(n, n, 1), 1.6, spec, np.float64)
    try:
        dev.init_analytic("taylor_green", 0.03)
        dev.step(8)
        ms = min(dev.time_steps(steps) for _ in range(3))
        return n * n * steps / (ms / 1e3) / 1e9
    finally:
        dev.close()


SIZES = [int(v) for v in os.environ.get("TB2D_SIZES", "128,256,384,512,768,1024").split(",")]
for n in SIZES:
    for faces in ("periodic", "lid"):
        a, b, c = run(n, faces, True), run(n, faces, False), run(n, faces, False, persist=False)
        print(json.dumps({"n": n, "faces": faces, "tb_glups": round(a, 3), "per_pass_glups": round(b, 3),
                          "launches_glups": round(c, 3)}))
