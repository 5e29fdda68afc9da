"""CPU, multi-process: the z-slab decomposition plan (paper_2304_06437_b200/
slabs.py) with real ranks on the gloo backend.

Each rank advances its slab plus ghost planes with the CPU oracle, ships the
ghost planes to its z neighbours with torch.distributed send/recv, and
accepts them under the plan's mask; after K steps the gathered slabs must be
bit-identical to the undivided domain (GPU-count determinism, SURVEY.md
§8(e)). The device implementation of the same plan is checked on one GPU by
tests/test_gpu_slabs.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2304_06437_b200 import slabs as S
from paper_2304_06437_b200 import tslb as T

from helpers import random_solid, spec_of, zwalls_3d

ORACLE_FACE = {S.WRAP: "periodic", S.WALL: "wall"}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, case, steps, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lat, dims, faces, solid, seed = case
        nx, ny, nz = dims
        plane = nx * ny
        L = T.lattice_of(lat)
        kinds = [T.FaceKind.Periodic if k == "periodic" else T.FaceKind.NoSlipWall if k == "wall"
                 else T.FaceKind.MovingWall for k, _ in faces]
        z0, nzl = S.split(nz, world)[rank]
        modes = S.face_modes(kinds, z0, nzl, nz)
        down, up = S.neighbours(modes, rank, world)
        glo, ghi = modes[4] == S.GHOST, modes[5] == S.GHOST
        # extended slab: [ghost below] owned [ghost above]
        planes = ([z0 - 1] if glo else []) + list(range(z0, z0 + nzl)) + ([z0 + nzl] if ghi else [])
        zl = len(planes)
        owned0 = 1 if glo else 0
        f0 = O.random_state(lat, dims, seed, np.float64, solid)
        gsolid = np.zeros(nx * ny * nz, np.uint8) if solid is None else solid
        f = np.concatenate([f0[:, (p % nz) * plane:(p % nz + 1) * plane] for p in planes], axis=1).copy()
        sol = np.concatenate([gsolid[(p % nz) * plane:(p % nz + 1) * plane] for p in planes]).copy()
        # z faces of the extended slab: ghost ends are periodic if both ends
        # are ghosts, else a resting wall (it only bounces ghost-node pushes);
        # a real wall end keeps its kind and velocity
        ext_faces = list(faces)
        zghost = ("periodic" if (glo and ghi) else "wall", (0.0, 0.0, 0.0))
        if glo:
            ext_faces[4] = zghost
        if ghi:
            ext_faces[5] = zghost
        edims = (nx, ny, zl)
        orc = O.Oracle("port")
        up_dirs, dn_dirs = S.exchange_dirs(L)
        staged = S.needs_staging(modes, solid is not None)

        def pl(k):
            return slice(k * plane, (k + 1) * plane)

        for _ in range(steps):
            orc.single_run(lat, edims, 0.9, ext_faces, f, None, 1, 0, sol if solid is not None else None)
            reqs = []
            if ghi:
                msg = np.ascontiguousarray(np.stack([f[a, pl(zl - 1)] for a, _, _ in up_dirs]))
                reqs.append(dist.isend(torch.from_numpy(msg), dst=up, tag=1))
            if glo:
                msg = np.ascontiguousarray(np.stack([f[a, pl(0)] for a, _, _ in dn_dirs]))
                reqs.append(dist.isend(torch.from_numpy(msg), dst=down, tag=2))
            rlo = torch.zeros((len(up_dirs), plane), dtype=torch.float64)
            rhi = torch.zeros((len(dn_dirs), plane), dtype=torch.float64)
            if glo:
                reqs.append(dist.irecv(rlo, src=down, tag=1))
            if ghi:
                reqs.append(dist.irecv(rhi, src=up, tag=2))
            for r in reqs:
                r.wait()
            if glo:  # c_z = +1 populations from below land in the first owned plane
                src = sol[pl(0)] if solid is not None else None
                dst = sol[pl(owned0)] if solid is not None else None
                for e, (a, cx, cy) in enumerate(up_dirs):
                    m = S.accept_mask(nx, ny, cx, cy, modes, src, dst).ravel() if staged else np.ones(plane, bool)
                    tgt = f[a, pl(owned0)]
                    tgt[m] = rlo.numpy()[e][m]
            if ghi:
                k = owned0 + nzl - 1
                src = sol[pl(zl - 1)] if solid is not None else None
                dst = sol[pl(k)] if solid is not None else None
                for e, (a, cx, cy) in enumerate(dn_dirs):
                    m = S.accept_mask(nx, ny, cx, cy, modes, src, dst).ravel() if staged else np.ones(plane, bool)
                    tgt = f[a, pl(k)]
                    tgt[m] = rhi.numpy()[e][m]
        mine = np.ascontiguousarray(f[:, owned0 * plane:(owned0 + nzl) * plane])
        out_q.put((rank, z0, nzl, mine))
    finally:
        dist.destroy_process_group()


CASES = [
    ("d3q19", (10, 9, 8), None, None, 11),
    ("d3q19", (10, 9, 8), "zwalls", None, 12),
    ("d3q19", (10, 9, 9), "box", 0.08, 13),
    ("d3q27", (8, 7, 8), "periodic", 0.1, 14),
]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[2]}-{c[3]}")
def test_slab_plan_with_gloo_ranks(case, world):
    lat, dims, fk, frac, seed = case
    faces = {None: O.periodic(), "periodic": O.periodic(), "zwalls": zwalls_3d(), "box": O.closed_box()}[fk]
    solid = random_solid(dims, frac, seed) if frac else None
    steps = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, (lat, dims, faces, solid, seed), steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    parts.sort(key=lambda t: t[1])
    got = np.concatenate([p[3] for p in parts], axis=1)
    ref = O.random_state(lat, dims, seed, np.float64, solid)
    O.Oracle("port").single_run(lat, dims, 0.9, faces, ref, None, steps, 0, solid)
    fluid = np.ones(ref.shape[1], bool) if solid is None else solid == 0
    assert np.array_equal(got[:, fluid].view(np.uint64), ref[:, fluid].view(np.uint64))


def test_split_and_modes():
    assert S.split(10, 3) == [(0, 3), (3, 3), (6, 4)]
    per = [T.FaceKind.Periodic] * 6
    assert S.face_modes(per, 0, 5, 10)[4:] == [S.GHOST, S.GHOST]
    walls = [T.FaceKind.Periodic] * 4 + [T.FaceKind.NoSlipWall] * 2
    assert S.face_modes(walls, 0, 5, 10)[4:] == [S.WALL, S.GHOST]
    assert S.face_modes(walls, 5, 5, 10)[4:] == [S.GHOST, S.WALL]
    assert S.neighbours(S.face_modes(per, 0, 5, 10), 0, 2) == (1, 1)
    assert S.neighbours(S.face_modes(walls, 0, 5, 10), 0, 2) == (-1, 1)
    up, dn = S.exchange_dirs(T.D3Q19)
    assert len(up) == len(dn) == 5
    assert len(S.exchange_dirs(T.D3Q27)[0]) == 9


# --- the M schedule's plan: moment ghost planes, one packed message per face
def _rank_main_m(rank, world, port, case, steps, out_q):
    """One rank of the M-schedule plan: the slab keeps its moments m(t) and
    the neighbours' boundary moment planes (gm, [2][NM][plane]); a step is
    f(t+1) = stream_collide(m(t)) over [ghost below] owned [ghost above]
    (only owned planes kept), m(t+1) = compute_moments(f(t+1)), then the
    packed boundary planes go to the neighbours. The oracle's phases stand in
    for the M kernel (tests/test_gpu_slabs.py runs the device one)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lat, dims, faces, solid, seed = case
        nx, ny, nz = dims
        plane = nx * ny
        L = T.lattice_of(lat)
        nm = O.moments_layout(lat)
        kinds = [T.FaceKind.Periodic if k == "periodic" else T.FaceKind.NoSlipWall if k == "wall"
                 else T.FaceKind.MovingWall for k, _ in faces]
        z0, nzl = S.split(nz, world)[rank]
        modes = S.face_modes(kinds, z0, nzl, nz)
        down, up = S.neighbours(modes, rank, world)
        glo, ghi = modes[4] == S.GHOST, modes[5] == S.GHOST
        planes = ([z0 - 1] if glo else []) + list(range(z0, z0 + nzl)) + ([z0 + nzl] if ghi else [])
        zl, owned0 = len(planes), (1 if glo else 0)
        gsolid = np.zeros(nx * ny * nz, np.uint8) if solid is None else solid
        sol = np.concatenate([gsolid[(p % nz) * plane:(p % nz + 1) * plane] for p in planes]).copy()
        ext_faces = list(faces)
        zghost = ("periodic" if (glo and ghi) else "wall", (0.0, 0.0, 0.0))
        if glo:
            ext_faces[4] = zghost
        if ghi:
            ext_faces[5] = zghost
        edims = (nx, ny, zl)
        orc = O.Oracle("port")
        ssol = sol if solid is not None else None
        own = slice(owned0 * plane, (owned0 + nzl) * plane)
        f0 = O.random_state(lat, dims, seed, np.float64, solid)
        fe = np.concatenate([f0[:, (p % nz) * plane:(p % nz + 1) * plane] for p in planes], axis=1).copy()
        me = np.zeros((nm, zl * plane))
        gm = np.zeros((2, nm, plane))

        def exchange():
            packed = S.pack_moment_planes(np.ascontiguousarray(me[:, own]), nm, plane, nzl)
            to_dn, to_up = S.moment_ghost_messages(packed)
            reqs = []
            if ghi:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(to_up)), dst=up, tag=1))
            if glo:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(to_dn)), dst=down, tag=2))
            rlo, rhi = torch.zeros((nm, plane), dtype=torch.float64), torch.zeros((nm, plane), dtype=torch.float64)
            if glo:
                reqs.append(dist.irecv(rlo, src=down, tag=1))
            if ghi:
                reqs.append(dist.irecv(rhi, src=up, tag=2))
            for r in reqs:
                r.wait()
            gm[0], gm[1] = rlo.numpy(), rhi.numpy()
            if glo:
                me[:, :plane] = gm[0]
            if ghi:
                me[:, (zl - 1) * plane:] = gm[1]

        # first step's moments pass (m(0) of the owned planes) + exchange
        orc.single_run(lat, edims, 0.9, ext_faces, fe, me, 1, 2, ssol)
        exchange()
        for _ in range(steps - 1):
            orc.single_run(lat, edims, 0.9, ext_faces, fe, me, 1, 3, ssol)  # f(t+1) = stream_collide(m(t))
            orc.single_run(lat, edims, 0.9, ext_faces, fe, me, 1, 2, ssol)  # m(t+1)
            exchange()
        m_lag = np.ascontiguousarray(me[:, own])            # the lagged moments m(steps - 1)
        orc.single_run(lat, edims, 0.9, ext_faces, fe, me, 1, 3, ssol)  # f(steps), materialised
        out_q.put((rank, z0, nzl, np.ascontiguousarray(fe[:, own]), m_lag))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[2]}-{c[3]}")
def test_m_slab_plan_with_gloo_ranks(case, world):
    """The M-schedule decomposition (packed moment planes per face, the
    device's exchange_moments_nccl) with real gloo ranks: f(N) and the
    lagged moments gathered over the slabs equal the undivided fused_step."""
    lat, dims, fk, frac, seed = case
    faces = {None: O.periodic(), "periodic": O.periodic(), "zwalls": zwalls_3d(), "box": O.closed_box()}[fk]
    solid = random_solid(dims, frac, seed) if frac else None
    steps = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main_m, args=(r, world, port, (lat, dims, faces, solid, seed), steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    parts.sort(key=lambda t: t[1])
    got_f = np.concatenate([p[3] for p in parts], axis=1)
    got_m = np.concatenate([p[4] for p in parts], axis=1)
    ref = O.random_state(lat, dims, seed, np.float64, solid)
    mo = np.zeros((O.moments_layout(lat), ref.shape[1]))
    O.Oracle("port").single_run(lat, dims, 0.9, faces, ref, mo, steps, 0, solid)
    fluid = np.ones(ref.shape[1], bool) if solid is None else solid == 0
    assert np.array_equal(got_f[:, fluid].view(np.uint64), ref[:, fluid].view(np.uint64))
    assert np.array_equal(got_m[:, fluid].view(np.uint64), mo[:, fluid].view(np.uint64))


def test_pack_moment_planes_layout():
    nm, plane, nzl = 10, 6, 4
    mo = np.arange(nm * nzl * plane, dtype=np.float64).reshape(nm, nzl * plane)
    p = S.pack_moment_planes(mo, nm, plane, nzl)
    assert p.shape == (2, nm, plane)
    assert np.array_equal(p[0], mo[:, :plane]) and np.array_equal(p[1], mo[:, (nzl - 1) * plane:])
    dn, upm = S.moment_ghost_messages(p)
    assert np.array_equal(dn, p[0]) and np.array_equal(upm, p[1])
