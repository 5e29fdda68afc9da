"""z-slab decomposition plan (multi-GPU) -- host-side logic.

SURVEY.md §8(e): the domain is split along z (slowest axis, so each plane of
each SoA array is one contiguous nx*ny run). Each rank owns planes
[z0, z0 + nzl) and carries one ghost plane below and above in its population
arrays. The fused stream-collide pushes populations with c_z = +1 out of the
top plane into the upper ghost plane (c_z = -1: lower ghost plane); the halo
exchange ships those planes to the neighbour's boundary plane, where they are
the only writer of those slots -- the reference's one-writer-per-slot rule
(kernels.hpp:149-153) carried across GPUs.

A received slot is valid only if the sender really pushed into it: its
source node (one plane away, shifted by -c) must be fluid and the push must
not have crossed an x/y wall (then the sender bounced instead). With solids
or x/y walls the received plane is therefore staged and unpacked under that
mask; for periodic x/y and no solids every slot is written and the receive
lands in place.

This module is the plan; the device implementation (csrc/tslb_capi.cu,
csrc/tslb_exchange.cu) follows it, and tests/test_cpu_slabs_gloo.py checks
the plan with two gloo ranks against the undivided oracle.
"""
from __future__ import annotations

import numpy as np

from . import tslb as T

WRAP, WALL, GHOST = "wrap", "wall", "ghost"


def split(nz: int, world: int) -> list[tuple[int, int]]:
    """Contiguous z ranges per rank (same rule as the reference's
    partition_range, parallel.hpp:20-23)."""
    if world < 1 or nz < world:
        raise ValueError(f"cannot split {nz} planes over {world} ranks")
    return [(nz * r // world, nz * (r + 1) // world - nz * r // world) for r in range(world)]


def face_modes(kinds, z0: int, nzl: int, nz: int) -> list[str]:
    """Face behaviour of one slab: x/y faces as in the box; a z face is a
    wall only at a global wall end, otherwise a ghost (exchanged) face."""
    per = [WRAP if k == T.FaceKind.Periodic else WALL for k in kinds]
    if nzl == nz:
        return per
    zlo = WALL if (z0 == 0 and kinds[4] != T.FaceKind.Periodic) else GHOST
    zhi = WALL if (z0 + nzl == nz and kinds[5] != T.FaceKind.Periodic) else GHOST
    return per[:4] + [zlo, zhi]


def neighbours(modes, rank: int, world: int) -> tuple[int, int]:
    """(down, up) ranks for the ghost faces, -1 where the face is a wall."""
    down = (rank - 1) % world if modes[4] == GHOST else -1
    up = (rank + 1) % world if modes[5] == GHOST else -1
    return down, up


def exchange_dirs(lat) -> tuple[list, list]:
    """Directions crossing the z faces: (c_z = +1, c_z = -1) lists of
    (a, cx, cy)."""
    L = T.lattice_of(lat)
    up = [(a, c[0], c[1]) for a, c in enumerate(L.c) if c[2] == 1]
    dn = [(a, c[0], c[1]) for a, c in enumerate(L.c) if c[2] == -1]
    return up, dn


def needs_staging(modes, has_solid: bool) -> bool:
    return has_solid or modes[0] == WALL or modes[2] == WALL


def accept_mask(nx: int, ny: int, cx: int, cy: int, modes, src_solid_plane=None, dst_solid_plane=None):
    """Boolean (ny, nx) mask of destination slots that the neighbour really
    wrote for a direction with in-plane components (cx, cy)."""
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    si, sj = i - cx, j - cy
    ok = np.ones((ny, nx), bool)
    for s, n, lo, hi in ((si, nx, 0, 1), (sj, ny, 2, 3)):
        out = (s < 0) | (s >= n)
        if modes[lo] == WALL:
            ok &= ~out
        s %= n
    if src_solid_plane is not None:
        ok &= ~np.asarray(src_solid_plane, bool).reshape(ny, nx)[sj % ny, si % nx]
    if dst_solid_plane is not None:
        ok &= ~np.asarray(dst_solid_plane, bool).reshape(ny, nx)
    return ok


# --- M schedule: the exchange is the slabs' boundary moment planes ----------
def pack_moment_planes(mo: np.ndarray, nm: int, plane: int, nzl: int) -> np.ndarray:
    """The send buffer of the M-step halo exchange (the device's h->sx,
    csrc/tslb_capi.cu pack_moments): [2][NM][plane] -- every moment array's
    plane 0 (for the slab below) and plane nzl - 1 (for the slab above) --
    one contiguous message per face."""
    m = np.asarray(mo).reshape(nm, -1)[:, :nzl * plane].reshape(nm, nzl, plane)
    return np.ascontiguousarray(np.stack([m[:, 0], m[:, nzl - 1]]))


def moment_ghost_messages(packed: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(to the slab below, to the slab above): the receiver stores the first
    as its upper ghost planes gm[1], the second as its lower gm[0]
    (layout [2][NM][plane], below / above)."""
    return packed[0], packed[1]
