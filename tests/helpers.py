"""Shared test helpers: geometry presets in both the oracle and the product
vocabulary, seeded states, bitwise comparison."""
import numpy as np

from oracle import oracle as O
from paper_2304_06437_b200 import tslb as T

KIND = {"periodic": T.FaceKind.Periodic, "wall": T.FaceKind.NoSlipWall, "moving": T.FaceKind.MovingWall}


def spec_of(faces) -> T.BoundarySpec:
    return T.BoundarySpec([T.Face(KIND[k], tuple(u)) for k, u in faces])


def mixed_2d(u=0.04):
    f = O.periodic()
    f[2] = ("wall", (0, 0, 0))
    f[3] = ("moving", (u, 0.0, 0.0))
    return f


def zwalls_3d(u=(0.03, 0.01, 0.0)):
    f = O.periodic()
    f[4] = ("wall", (0, 0, 0))
    f[5] = ("moving", u)
    return f


def corner_box_3d():
    f = O.closed_box()
    f[3] = ("moving", (0.04, 0.0, 0.01))
    f[1] = ("moving", (0.0, 0.02, 0.0))
    return f


def block_solid(dims, lo, hi):
    nx, ny, nz = dims
    s = np.zeros((nz, ny, nx), np.uint8)
    s[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = 1
    return s.ravel()


def random_solid(dims, frac, seed):
    rng = np.random.default_rng(seed)
    return (rng.random(int(np.prod(dims))) < frac).astype(np.uint8)


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint8 if a.dtype.itemsize == 1 else np.dtype(f"u{a.dtype.itemsize}"))


def assert_bitwise(a, b, what="", mask=None):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    ba, bb = bits(a), bits(b)
    if mask is not None:
        ba = ba[..., mask]
        bb = bb[..., mask]
    neq = ba != bb
    if neq.any():
        idx = np.argwhere(neq)[:5]
        af = a[..., mask] if mask is not None else a
        bf = b[..., mask] if mask is not None else b
        ex = [(tuple(i), af[tuple(i)], bf[tuple(i)]) for i in idx]
        raise AssertionError(f"{what}: {int(neq.sum())} of {neq.size} values differ bitwise, e.g. {ex}")


def droplet_state(dims, R, dtype, u=(0.0, 0.0, 0.0), width=3.0):
    nx, ny, nz = dims
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    cz = (nz - 1) / 2 if nz > 1 else 0.0
    r = np.sqrt((i - (nx - 1) / 2) ** 2 + (j - (ny - 1) / 2) ** 2 + (k - cz) ** 2).ravel()
    phi = np.tanh(2 * (R - r) / width)
    st = np.zeros((5, r.size))
    st[0] = 0.5 * (1 + phi)
    st[1] = 0.5 * (1 - phi)
    st[2], st[3], st[4] = u
    return st.astype(dtype)
