"""Loader for the reference-generated fixtures in tests/golden/."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FACE_NAMES = {0: "periodic", 1: "wall", 2: "moving"}


def single_cases():
    return sorted(p for p in glob.glob(os.path.join(GOLDEN, "d*_*.npz")) if "_two_" not in p)


def two_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "d*_two_*.npz")))


def load(path):
    z = np.load(path)
    d = {k: z[k] for k in z.files}
    d["lat"] = str(d["lat"])
    d["dims"] = tuple(int(v) for v in d["dims"])
    d["faces"] = [(FACE_NAMES[int(k)], tuple(d["uw"][3 * i:3 * i + 3])) for i, k in enumerate(d["kinds"])]
    d["solid"] = None if d["solid"].size == 0 else d["solid"]
    return d


def color_dict(d):
    c, ci = d["color"], d["color_i"]
    return dict(sigma=c[0], beta=c[1], nci_strength=c[2], eps_bulk=c[3], grad_threshold=c[4], nci_reach=int(ci[0]),
                linear=bool(ci[1]))
