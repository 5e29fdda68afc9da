#!/usr/bin/env python
"""Throughput of the thread-safe LB hot path (BASELINE.json metric:
"GLUPS and % of HBM roofline (D3Q19 1024^3) at 1/2/4/8 B200 vs CPU ref").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload tgv-d3q19|tgv-c5|channel-d3q27|droplet-d3q19|tgv-d2q9|porous-d3q19|cavity-d2q9]
                    [--math f64|f32] [--schedule auto|m|f1]

Default workload (the metric's): D3Q19 single-phase periodic Taylor-Green
vortex, 1024^3 nodes per GPU, fp32 storage, fp64 node arithmetic (the
reference's float build, bit for bit), M step = ONE moment-resident kernel
per step (k_mstep: populations rebuilt and streamed in shared memory, 80 B
per lattice update). `--gpus N` without a torchrun environment re-launches
this command as N ranks (one process per GPU, torch.distributed.run on
127.0.0.1); under torchrun WORLD_SIZE must equal N. N > 1: weak scaling, one
1024^3 z slab per GPU of a 1024 x 1024 x (1024 N) periodic box, boundary
chunks + NCCL halo exchange on the comm stream overlapped with the interior
chunk. `--workload tgv-c5` is BASELINE config 5 (strong scaling: the fixed
2048 x 1024 x 1024 domain split into N slabs). The state (86 GB per GPU) is
far larger than the 126 MB L2, so no L2 flush is needed.

The other workloads are BASELINE.json's configs 1, 3 and 4 and extra cases,
for the record; the driver's headline is the default.

--impl reference times the reference's own CPU implementation
(oracle/_ref/libtslb_ref.so = the unmodified tslb headers, WorkerPool over
all host cores; the plain-C oracle port if that build is absent): the WHOLE
per-GPU workload when the host has the memory (1024^3: 130 GB), else a
1024 x 1024 x 16 slab sample of it.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
L2_NOTE = "state >> 126 MB L2, no flush needed"
METRIC = "GLUPS and % of HBM roofline (D3Q19 1024^3) at 1/2/4/8 B200 vs CPU ref"

# per-GPU workloads (BASELINE.json configs)
WORKLOADS = {
    "tgv-d3q19": dict(lat="d3q19", dims=(1024, 1024, 1024), faces="periodic", comps=1, init="taylor_green",
                      amp=0.03, omega=1.6, storage="f32",
                      desc="D3Q19 periodic Taylor-Green {n}"),
    "channel-d3q27": dict(lat="d3q27", dims=(1024, 1024, 1024), faces="channel", comps=1, init="rest", amp=0.0,
                          omega=1.0, storage="f32", umax=0.05,
                          desc="D3Q27 Poiseuille channel {n}: no-slip walls at y, body force along x for "
                               "u_max 0.05 (single-fluid forcing extension), rest init"),
    "droplet-d3q19": dict(lat="d3q19", dims=(512, 512, 512), faces="periodic", comps=2, init="droplet",
                          radius=512 / 6.0, omega=1 / 0.75, storage="f32", sigma=0.03, beta=0.7,
                          desc="D3Q19 two-component colour-gradient droplet {n}, R = 85.33, sigma 0.03, beta 0.7"),
    "tgv-d2q9": dict(lat="d2q9", dims=(4096, 4096, 1), faces="periodic", comps=1, init="taylor_green", amp=0.03,
                     omega=1.6, storage="f32", desc="D2Q9 periodic Taylor-Green {n} (the paper's 2-D size)"),
    "porous-d3q19": dict(lat="d3q19", dims=(512, 512, 512), faces="periodic", comps=1, init="rest", amp=0.0,
                         omega=1.0, storage="f32", force=(1e-6, 0.0, 0.0), spheres=(12.0, 0.25, 5),
                         desc="D3Q19 periodic porous medium {n}: random overlapping spheres (r 12, ~25 % solid, "
                              "bounce-back), body force along x, rest init"),
    "cavity-d2q9": dict(lat="d2q9", dims=(256, 256, 1), faces="lid", comps=1, init="rest", amp=0.0,
                        omega=1 / (0.064 * 3 + 0.5), storage="f64",
                        desc="D2Q9 lid-driven cavity {n}, Re 100, fp64"),
    # BASELINE config 5: one fixed domain split into N z slabs (strong scaling)
    "tgv-c5": dict(lat="d3q19", dims=(2048, 1024, 1024), faces="periodic", comps=1, init="taylor_green",
                   amp=0.03, omega=1.6, storage="f32", strong=True,
                   desc="D3Q19 periodic Taylor-Green 2048x1024x1024 (BASELINE config 5): {n}"),
}


def peaks():
    try:
        with open(PEAKS) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured", p
    except Exception:
        return 6650.0, "fallback", {}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        self.t.join(1)
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) > 8:
                for nm, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference arm / cpu baseline
# ---------------------------------------------------------------------------
def tgv_state(dims, nz_global, z0, dtype):
    from paper_2304_06437_b200 import tslb as T
    nx, ny, nz = dims
    g = T.GridDims(nx, ny, nz)
    s = T.allocate_fields(g, T.D3Q19, dtype)
    U = 0.03

    def st(i, j, k):
        X = 2 * np.pi * (i + 0.5) / nx
        Y = 2 * np.pi * (j + 0.5) / ny
        Z = 2 * np.pi * (k + z0 + 0.5) / nz_global
        z = np.zeros(i.shape)
        rho = 1 + 3 * (U * U / 16) * (np.cos(2 * X) + np.cos(2 * Y)) * (np.cos(2 * Z) + 2)
        return (rho, U * np.sin(X) * np.cos(Y) * np.cos(Z), -U * np.cos(X) * np.sin(Y) * np.cos(Z), z, z, z, z, z, z, z)

    T.initialize_regularized(s, None, st, T.D3Q19)
    return s.f


def cpu_reference(steps, warmup, sample_nz=16, workers=None):
    """Time the reference CPU path on a 1024 x 1024 x sample_nz periodic slab
    of the Taylor-Green workload (fp32 storage). Returns (GLUPS, info)."""
    import ctypes as C

    from oracle import oracle as O
    workers = workers or os.cpu_count() or 1
    dims = (1024, 1024, sample_nz)
    f = tgv_state(dims, 1024, 0, np.float32)
    kinds, uw = O.faces_arrays(O.periodic())
    if os.path.exists(O.REF_SO):
        o = O.Oracle("ref")
        secs = C.c_double()
        rc = o.lib.tslbref_time_steps(1, 1, *dims, 1.6, O._ptr(kinds), O._ptr(uw), O._ptr(f), int(steps),
                                      int(warmup), int(workers), C.byref(secs))
        o._check(rc)
        kind, cores, t = "reference", workers, secs.value
    else:
        o = O.Oracle("port")
        o.single_run("d3q19", dims, 1.6, O.periodic(), f, None, warmup, 0)
        t0 = time.perf_counter()
        o.single_run("d3q19", dims, 1.6, O.periodic(), f, None, steps, 0)
        kind, cores, t = "port", 1, time.perf_counter() - t0
    glups = dims[0] * dims[1] * dims[2] * steps / t / 1e9
    sample = (f"D3Q19 periodic Taylor-Green slab {dims[0]}x{dims[1]}x{dims[2]} fp32 (fp64 node math), {steps} steps "
              f"after {warmup} warm-up, WorkerPool({cores})")
    return glups, dict(kind=kind, cores=cores, sample=sample, seconds=t)


def mem_available():
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def cpu_reference_full(dims, steps, warmup, workers=None):
    """The reference CPU path on the WHOLE per-GPU workload: the reference's
    fused_step (WorkerPool over every host core) on the nx x ny x nz
    periodic Taylor-Green state of the reference's own
    initialize_regularized (oracle/ref_capi.cpp tslbref_time_tgv).
    Returns (GLUPS, info) or None when the host cannot hold the state."""
    import ctypes as C

    from oracle import oracle as O
    if not os.path.exists(O.REF_SO):
        return None
    n = int(np.prod(dims))
    need = n * (29 * 4 + 5)  # f + moments (fp32), slow mask, solid mask
    if mem_available() < 1.08 * need:
        return None
    workers = workers or os.cpu_count() or 1
    lib = C.CDLL(O.REF_SO)
    fn = lib.tslbref_time_tgv
    fn.argtypes = [C.c_int] * 4 + [C.c_double, C.c_double, C.c_long, C.c_long, C.c_int, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
    ti, ts, dg = C.c_double(), C.c_double(), C.c_uint64()
    if fn(1, *dims, 1.6, 0.03, int(steps), int(warmup), int(workers), 0, C.byref(ti), C.byref(ts), C.byref(dg)):
        lib.tslbref_last_error.restype = C.c_char_p
        raise RuntimeError(lib.tslbref_last_error().decode())
    what = "x".join(str(v) for v in dims)
    sample = (f"the whole workload: D3Q19 periodic Taylor-Green {what} fp32 (fp64 node math), {steps} steps after "
              f"{warmup} warm-up, WorkerPool({workers})")
    return n * steps / ts.value / 1e9, dict(kind="reference", cores=workers, sample=sample, seconds=ts.value,
                                            init_seconds=round(ti.value, 1), digest=f"{dg.value:016x}")


def cpu_reference_workload(name, W, dims, steps, warmup, sample_nz=16, workers=None):
    """The reference CPU path (oracle/_ref: the reference headers, WorkerPool
    over the host cores) on a bounded sample of a non-default workload:
    2-D workloads whole, 3-D workloads as an nx x ny x sample_nz slab
    (periodic in z) of the same faces / mask / colour state. The reference
    has no D3Q27: the channel row times D3Q19 on the same slab (BASELINE.md
    §3, C3). Returns (GLUPS, info) or raises."""
    import ctypes as C

    from oracle import oracle as O
    if not os.path.exists(O.REF_SO):
        raise FileNotFoundError("oracle/_ref not built")
    workers = workers or os.cpu_count() or 1
    lat = "d3q19" if W["lat"] == "d3q27" else W["lat"]
    nx, ny, nz = dims
    sdims = (nx, ny, nz) if nz == 1 else (nx, ny, min(sample_nz, nz))
    n = int(np.prod(sdims))
    steps = max(steps, min(2000, int(2e8 // n)))  # small grids: enough steps for a stable timing
    dt = np.float32 if W["storage"] == "f32" else np.float64
    faces = {"periodic": O.periodic(), "lid": O.lid_cavity(0.025)}.get(W["faces"])
    if faces is None:  # channel: no-slip walls at y
        faces = O.periodic()
        faces[2] = ("wall", (0, 0, 0))
        faces[3] = ("wall", (0, 0, 0))
    kinds, uw = O.faces_arrays(faces)
    info = O.lattice_info(lat)
    o = O.Oracle("ref")
    secs = C.c_double()
    scalar = 0 if dt == np.float64 else 1
    if W["comps"] == 2:
        z0 = (nz - sdims[2]) // 2  # a slab through the droplet centre
        k, j, i = np.meshgrid(np.arange(sdims[2]) + z0, np.arange(ny), np.arange(nx), indexing="ij")
        r = np.sqrt((i - 0.5 * nx + 0.5) ** 2 + (j - 0.5 * ny + 0.5) ** 2 + (k - 0.5 * nz + 0.5) ** 2).ravel()
        prof = 0.5 * (1 + np.tanh(W["radius"] - r))
        st = np.zeros((5, n), dt)
        st[0], st[1] = prof, 1 - prof
        fr, fb = O.Oracle("port").init_colors(lat, sdims, st)
        cp = np.array([W.get("sigma", 0.01), W.get("beta", 0.7), 0.0, 0.02, 1e-6], np.float64)
        ip = np.array([3, 0], np.int32)
        o._check(o.lib.tslbref_time_two(O.LATTICES[lat], scalar, *sdims, float(W["omega"]), O._ptr(cp),
                                        O._ptr(ip), O._ptr(kinds), O._ptr(uw), O._ptr(fr), O._ptr(fb), int(steps),
                                        int(warmup), int(workers), C.byref(secs)))
    else:
        solid = None
        if "spheres" in W:
            solid = np.ascontiguousarray(sphere_pack(dims, *W["spheres"])[:n])
        f = np.repeat(info["t"].astype(dt)[:, None], n, axis=1)  # rest equilibrium
        if solid is not None:
            f[:, solid != 0] = 0
        f = np.ascontiguousarray(f)
        o._check(o.lib.tslbref_time_steps_ex(O.LATTICES[lat], scalar, *sdims, float(W["omega"]), O._ptr(kinds),
                                             O._ptr(uw), O._ptr(solid), O._ptr(f), int(steps), int(warmup),
                                             int(workers), C.byref(secs)))
    t = secs.value
    glups = n * steps / t / 1e9
    what = "x".join(str(v) for v in sdims)
    sample = (f"{lat.upper()} {what} sample of the {name} workload ({W['storage']}), {steps} steps after "
              f"{warmup} warm-up, WorkerPool({workers})" + (" -- D3Q19 stands in: the reference has no D3Q27"
                                                            if W["lat"] == "d3q27" else ""))
    return glups, dict(kind="reference", cores=workers, sample=sample, seconds=t)


def host_info():
    """CPU model, logical CPUs, sockets and physical cores (lscpu's fields,
    read from /proc/cpuinfo)."""
    model, phys = "", set()
    cur = {}
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                k, _, v = line.partition(":")
                k, v = k.strip(), v.strip()
                if k == "model name" and not model:
                    model = v
                elif k in ("physical id", "core id"):
                    cur[k] = v
                elif not k and cur:
                    phys.add((cur.get("physical id"), cur.get("core id")))
                    cur = {}
        if cur:
            phys.add((cur.get("physical id"), cur.get("core id")))
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count(), "sockets": len({p for p, _ in phys}) or None,
            "physical_cores": len(phys) or None}


# ---------------------------------------------------------------------------
def spec_of(T, kind):
    if kind == "periodic":
        return T.BoundarySpec.all_periodic()
    if kind == "lid":
        return T.BoundarySpec.lid_cavity(0.025)
    s = T.BoundarySpec.all_periodic()  # channel: no-slip walls at y
    s.faces[T.YMin] = T.Face(T.FaceKind.NoSlipWall)
    s.faces[T.YMax] = T.Face(T.FaceKind.NoSlipWall)
    return s


def sphere_pack(dims, radius, frac, seed):
    """Solid mask of random overlapping periodic spheres, about `frac` of the
    nodes solid (x fastest, the solver's node order)."""
    nx, ny, nz = dims
    rng = np.random.default_rng(seed)
    vol = 4.0 / 3.0 * np.pi * radius ** 3
    count = int(round(-np.log(1.0 - frac) * nx * ny * nz / vol))
    s = np.zeros((nz, ny, nx), np.uint8)
    r = int(np.ceil(radius))
    off = np.arange(-r, r + 1)
    d2 = off[:, None, None] ** 2 + off[None, :, None] ** 2 + off[None, None, :] ** 2
    ball = (d2 <= radius * radius).astype(np.uint8)
    for c in rng.random((count, 3)) * np.array([nz, ny, nx]):
        iz, iy, ix = (np.floor(c).astype(int)[:, None] + off[None, :]) % np.array([[nz], [ny], [nx]])
        s[np.ix_(iz, iy, ix)] |= ball
    return s.ravel()


def kernel_bytes(lat, comps, es, solid=False):
    """Algorithmic bytes per node of each kernel class;
    masked geometries add the solid mask (1 B), the per-node direction masks
    of the F1 stream-collide (4 B) and the M step's solid bits (4 B)."""
    q, D = lat.q, lat.dim
    npi = D * (D + 1) // 2
    nm = 1 + D + npi
    if comps == 1:
        # F1: moments pass + stream-collide; M: one moment-resident pass
        sb = 1 if solid else 0
        return {"moments": (q + nm) * es + sb, "streamcoll": (nm + q) * es + 5 * sb, "mstep": 2 * nm * es + 4 * sb}
    return {"cg_moments": (2 * q + 3 + nm) * es, "cg_gradient": (1 + D) * es,
            "cg_streamcoll": (3 + D + npi + D + 2 * q) * es}


def step_bytes(lat, comps, es, schedule="f1", solid=False):
    kb = kernel_bytes(lat, comps, es, solid)
    if comps == 1:
        return kb["mstep"] if schedule == "m" else kb["moments"] + kb["streamcoll"]
    return sum(kb.values())


def _json_stdout():
    """stdout carries exactly one JSON line: anything else written to fd 1
    (NCCL's version banner, library chatter) is sent to stderr; the returned
    stream is the original stdout."""
    sys.stdout.flush()
    keep = os.dup(1)
    os.dup2(2, 1)
    return os.fdopen(keep, "w", buffering=1)


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _relaunch(n):
    """`bench.py --gpus N` outside torchrun: re-run this command as N ranks
    (one process per GPU) under torch.distributed.run and return its exit
    code; rank 0 prints the JSON line."""
    # (torch.distributed.run's parser would take "--n" for an abbreviation of
    # its own options even after the script path: pass it as "--cube")
    argv = ["--cube" + a[3:] if a == "--n" or a.startswith("--n=") else a for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *argv]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


def launch_check(world, rank):
    """--launch-check: the ranks this command started, gathered over gloo
    (CPU; no GPU needed) -- the test of the N-rank launch path."""
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
        ranks = [None] * world
        dist.all_gather_object(ranks, (rank, os.getpid()))
        dist.destroy_process_group()
    else:
        ranks = [(rank, os.getpid())]
    return {"launch_check": True, "n_gpus": world, "ranks": [r for r, _ in ranks],
            "pids_distinct": len({p for _, p in ranks}) == world}


def main():
    # --gpus N without a torchrun environment: one process per GPU
    world_env = os.environ.get("WORLD_SIZE")
    pre = argparse.ArgumentParser(add_help=False)
    pre.add_argument("--gpus", type=int, default=1)
    ngpus = pre.parse_known_args()[0].gpus
    if world_env is None and ngpus > 1:
        sys.exit(_relaunch(ngpus))
    if world_env is not None and int(world_env) != ngpus:
        raise SystemExit(f"bench.py: --gpus {ngpus} but WORLD_SIZE={world_env}: launch one rank per GPU")
    out_stream = _json_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="tgv-d3q19", choices=sorted(WORKLOADS))
    ap.add_argument("--n", "--cube", dest="n", type=int, default=0, help="override the per-GPU cube edge (3D)")
    ap.add_argument("--dims", default="", help="override the per-GPU extent nx,ny,nz (3D)")
    ap.add_argument("--math", default="f64", choices=["f64", "f32"])
    ap.add_argument("--schedule", default="auto", choices=["auto", "m", "f1"])
    ap.add_argument("--storage", default="native", choices=["native", "f16"],
                    help="f16: the M steps keep the moments as scaled fp16 (mixed precision, fp32 node math)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sample-nz", type=int, default=16)
    ap.add_argument("--sample-only", action="store_true",
                    help="--impl reference: time the 1024 x 1024 x sample_nz slab even if the host holds the "
                         "whole workload")
    ap.add_argument("--launch-check", action="store_true",
                    help="report the ranks this command launched (gloo, CPU) and exit")
    ap.add_argument("--nccl-self", action="store_true",
                    help="N=1 probe of the multi-GPU step: the GPU's domain is a z slab of a twice-as-tall box on "
                         "a one-rank NCCL communicator (its own up/down neighbour), so every step runs the "
                         "boundary chunks, the NCCL halo exchange on the comm stream and the overlapped interior")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "ipc"],
                    help="slab halo transport for N > 1 (and the self-exchange probe): NCCL send/recv, or ipc -- "
                         "the boundary planes copied straight into the neighbours' ghost buffers through CUDA IPC "
                         "mappings (M single-fluid steps)")
    ap.add_argument("--ipc-self", action="store_true",
                    help="like --nccl-self, over the peer-memory transport (the slab's own handle on both faces)")
    args = ap.parse_args()
    if args.ipc_self:
        args.nccl_self, args.transport = True, "ipc"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.launch_check:
        info = launch_check(world, rank)
        if rank == 0:
            print(json.dumps(info), file=out_stream)
        return
    W = dict(WORKLOADS[args.workload])
    dims = W["dims"]
    strong = W.get("strong", False)
    if args.n and dims[2] > 1:
        dims = (args.n, args.n, args.n)
    if args.dims and dims[2] > 1:
        dims = tuple(int(v) for v in args.dims.split(","))
    if strong:
        # the fixed global domain (--n / --dims: its extent), one z slab per rank
        if dims[2] % world:
            raise SystemExit(f"{args.workload}: nz = {dims[2]} does not split into {world} slabs")
        dims = (dims[0], dims[1], dims[2] // world)
    default = args.workload == "tgv-d3q19" and not args.nccl_self
    scaling = "strong" if strong else "weak"
    probe = f", {'IPC' if args.transport == 'ipc' else 'NCCL'} self-exchange probe" if args.nccl_self else ""
    metric = METRIC if default else f"GLUPS ({args.workload}{probe})"

    if args.impl == "reference":
        if rank != 0:
            return
        steps, warm = args.steps, args.warmup
        # the whole per-GPU workload when the host holds it (1024^3: 130 GB),
        # else a 1024 x 1024 x 16 slab sample of it
        full = None
        if default and not args.sample_only:
            full = cpu_reference_full(dims, steps, warm)
        if full:
            glups, info = full
        else:
            warm = max(1, min(warm, 2))
            glups, info = cpu_reference(steps, warm, args.sample_nz)
        # the host, and a 1-worker row beside the all-cores one
        g1, info1 = cpu_reference(1, 1, args.sample_nz, workers=1)
        n_desc = "x".join(str(v) for v in dims)
        cfg = ({"workload": WORKLOADS["tgv-d3q19"]["desc"].format(n=n_desc) + " per GPU", "lattice": "d3q19",
                "nodes": int(np.prod(dims)), "storage": "f32", "node_math": "f64", "l2": L2_NOTE,
                "parallelism": "single GPU"}
               if full else
               {"workload": f"D3Q19 periodic Taylor-Green, sample of the {dims[0]}^3 fp32 workload",
                "lattice": "d3q19", "storage": "f32", "sample": info["sample"]})
        out = {"metric": METRIC, "value": round(glups, 6), "unit": "GLUPS", "n_gpus": args.gpus, "steps": steps,
               "warmup": warm, "ms_per_step": round(info["seconds"] / steps * 1e3, 3), "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "impl": "reference", "same_config": bool(full),
               "config": cfg,
               "cpu_baseline": {"value": round(glups, 6), "unit": "GLUPS", "cores": info["cores"],
                                "kind": info["kind"], "sample": info["sample"]},
               "e2e": {"value": round(glups, 6), "unit": "GLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
               "cpu_1worker": {"value": round(g1, 6), "unit": "GLUPS", "cores": info1["cores"],
                               "kind": info1["kind"], "sample": info1["sample"]},
               "host": host_info()}
        if full:
            out["reference_run"] = {"init_seconds": info["init_seconds"], "f_digest": info["digest"]}
        print(json.dumps(out), file=out_stream)
        return

    import torch

    from paper_2304_06437_b200 import _lib
    from paper_2304_06437_b200 import tslb as T

    dist = None
    # TSLB_BENCH_ONE_GPU=1 (functional checks of the N-rank path on a one-GPU
    # box; timings meaningless): every rank on device 0, peer-memory transport
    one_gpu = os.environ.get("TSLB_BENCH_ONE_GPU") == "1"
    if one_gpu and args.transport != "ipc":
        raise SystemExit("TSLB_BENCH_ONE_GPU needs --transport ipc (NCCL refuses two ranks on one device)")
    dev_id = local if world > 1 and not one_gpu else 0
    backend = "nccl" if args.transport == "nccl" else "gloo"  # (ipc: the process group is control plane only)
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(dev_id)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_id))
        else:
            dist.init_process_group("gloo")
    torch.cuda.set_device(dev_id)

    lat = T.lattice_of(W["lat"])
    dtype = np.float32 if W["storage"] == "f32" else np.float64
    es = np.dtype(dtype).itemsize
    if world > 1 and lat.dim != 3:
        raise SystemExit("multi-GPU slabs: 3-D workloads only")
    nx, ny, nzp = dims
    self_x = args.nccl_self and world == 1 and lat.dim == 3
    nz_g = nzp * (2 if self_x else world)
    g = T.GridDims(nx, ny, nz_g)
    spec = spec_of(T, W["faces"])
    color = T.ColorParams(sigma=W.get("sigma", 0.01), beta=W.get("beta", 0.7)) if W["comps"] == 2 else None
    slab = (rank * nzp, nzp) if world > 1 or self_x else None
    solid = None
    if "spheres" in W:
        if world > 1:
            raise SystemExit("masked geometries run on whole domains (one GPU)")
        solid = sphere_pack(dims, *W["spheres"])
    sim = T.DeviceSolver(lat, g, W["omega"], spec, dtype, W["comps"], solid, color, dev_id, slab=slab)
    if args.math == "f32":
        sim.set_math(_lib.MATH_F32)
    if args.storage == "f16":
        sim.set_moment_storage("f16")  # (fp32 node math with it)
        args.math = "f32"
    if args.schedule != "auto" and W["comps"] == 1:
        sim.set_schedule(args.schedule)
    if "umax" in W:
        # Poiseuille: u_max = F H^2 / (8 nu), H = ny (halfway bounce-back)
        nu = (1.0 / W["omega"] - 0.5) / 3.0
        sim.set_body_force(8.0 * nu * W["umax"] / float(ny) ** 2, 0.0, 0.0)
    if "force" in W:
        sim.set_body_force(*W["force"])
    if (world > 1 or self_x) and args.transport == "ipc":
        # peer-memory transport: every rank's handle to every rank
        own = sim.ipc_handle()
        hs = [own]
        if dist:
            hs = [None] * world
            dist.all_gather_object(hs, own)
        zper = spec.faces[T.ZMin].kind == T.FaceKind.Periodic
        below = hs[(rank - 1) % world] if (rank > 0 or zper) else None
        above = hs[(rank + 1) % world] if (rank < world - 1 or zper) else None
        sim.attach_ipc(below, above)
    elif world > 1 or self_x:
        import ctypes as C
        uid = (C.c_char * 128)()
        if rank == 0:
            _lib.check(_lib.load().tslb_cuda_nccl_unique_id(uid))
        if dist:
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=0)
            uid = (C.c_char * 128).from_buffer_copy(obj[0])
        _lib.check(_lib.load().tslb_cuda_attach_nccl(sim.h, uid, world, rank))
    if W["init"] == "droplet":
        sim.init_analytic("droplet", 0.0, W["radius"])
    else:
        sim.init_analytic(W["init"], W.get("amp", 0.0))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (untimed)
    sim.step(args.warmup)
    barrier()
    launches0 = sim.launch_count()
    clocks = Clocks() if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    sim.profile(True)
    barrier()
    ms = sim.time_steps(args.steps)
    barrier()
    prof = sim.profile_read()
    sim.profile(False)
    launches = sim.launch_count() - launches0
    clk = clocks.stop() if clocks else None
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    nodes = nx * ny * nzp * world  # (the self-exchange probe steps one slab)
    glups = nodes * args.steps / (ms / 1e3) / 1e9

    # roofline of the dominant kernel: algorithmic bytes per launch / mean
    # launch duration (CUDA events on the solver stream, timed region)
    masked = solid is not None
    per_node = kernel_bytes(lat, W["comps"], es, masked)
    if args.storage == "f16":  # fp16 moments in and out of the M step
        per_node["mstep"] = 2 * (1 + lat.dim + lat.dim * (lat.dim + 1) // 2) * 2
    if W["comps"] == 2 and "cg_moments" not in prof:
        # the one-pass step (k_cg_fused, profiled as the recolouring class):
        # both species in and out, the colour moment arrays out, the flags
        npi = lat.dim * (lat.dim + 1) // 2
        per_node = {"cg_streamcoll": 4 * lat.q * es + (4 + lat.dim + npi) * es + 1}
    elif W["comps"] == 2 and "cg_gradient" not in prof:
        # gradient folded into the recolouring stream-collide: it reads phi
        # (its stencil from cache) instead of the stored gradient
        npi = lat.dim * (lat.dim + 1) // 2
        per_node = {"cg_moments": per_node["cg_moments"], "cg_streamcoll": (3 + lat.dim + npi + 1 + 2 * lat.q) * es}
    dom = max((k for k in per_node if k in prof), key=lambda k: prof[k][0])
    k_ms, k_n = prof[dom]
    local_nodes = nx * ny * nzp
    # algorithmic bytes over the class's summed launch time: one launch per
    # step on a whole domain (= bytes per launch / mean launch time); slabs
    # split the step into boundary and interior chunk launches
    achieved = per_node[dom] * local_nodes * args.steps / (k_ms / 1e3) / 1e9
    hbm, peak_kind, _ = peaks()
    sched = sim.schedule if W["comps"] == 1 else "f1"
    sb = step_bytes(lat, W["comps"], es, sched, masked) if W["comps"] == 1 else sum(per_node.values())
    if args.storage == "f16":
        sb = per_node["mstep"]
    step_bw = glups * sb / world  # per-GPU GB/s of the whole step
    traffic, tsrc, limiter, fp64_ops = None, None, None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            # (masked geometries carry the solid bits: their own capture)
            skey = W["storage"] if args.storage == "native" else "f16"
            tr = json.load(fh).get(f"{lat.name}/{skey}/{dom}{'+solid' if masked else ''}")
        if tr and args.workload not in tr.get("workloads", [args.workload]):
            tr = None
        if tr:
            traffic, tsrc = round(tr["bytes_per_node"] * local_nodes / 1e9, 3), tr["source"]
            limiter = tr.get("limiter")
            fp64_ops = tr.get("fp64_ops_per_lu") if args.math == "f64" else None
    except (OSError, ValueError):
        pass
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 4), "traffic": traffic, "traffic_unit": "GB per launch",
            "traffic_source": tsrc, "limiter": limiter, "kernel": f"k_{dom}",
            "kernel_bytes_per_node": per_node[dom], "peak_kind": peak_kind,
            "per_kernel_ms": {k: round(v[0] / v[1], 4) for k, v in prof.items()},
            "kernel_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in prof.items()},
            "launches_per_step": {k: round(v[1] / args.steps, 2) for k, v in prof.items()},
            "step_bytes_per_lu": sb, "step_frac": round(step_bw / hbm, 4),
            "step_frac_of_8TBs": round(step_bw / 8000.0, 4)}
    if fp64_ops:
        # the pipe that binds the fp64-arithmetic M kernel: executed DADD+DMUL
        # per LU (ncu SASS mix) against 64 fp64 lanes/clk/SM at the sampled clock
        mhz = (clk or {}).get("sm_mhz") or 1965.0
        peak_t = 148 * 64 * mhz * 1e6 / 1e12
        ach_t = fp64_ops * glups / world * 1e9 / 1e12
        roof["fp64_pipe"] = {"ops_per_lu": fp64_ops, "achieved_tops": round(ach_t, 2),
                             "peak_tops": round(peak_t, 2), "frac": round(ach_t / peak_t, 4),
                             "source": "profiles/traffic.json"}
    if W["comps"] == 1:
        # the F1 schedule's ceiling: every population through HBM twice
        # (census bytes, bench.hpp:62-63); M beats it by moving fewer bytes
        f1b = kernel_bytes(lat, 1, es, masked)["moments"] + kernel_bytes(lat, 1, es, masked)["streamcoll"]
        roof["f1_bytes_per_lu"] = f1b
        roof["f1_roofline_glups"] = round(hbm / f1b, 3)
        roof["vs_f1_roofline"] = round(glups / world / (hbm / f1b), 4)

    e2e = None
    if default and not args.no_e2e and world == 1:
        e2e = run_e2e(sim, lat, (nx, ny, nzp), args.steps, dtype, W.get("amp", 0.03))
    elif default and not args.no_e2e:
        # the loop stages each rank's whole state in pinned host memory
        # (~99 GB per 1024^3 slab): not attempted N times on one host
        e2e = {"value": None, "unit": "GLUPS", "reason": "measured at N=1 only (pinned host staging of the "
                                                           "full state per rank)"}

    cpu = None
    if not default and rank == 0 and not args.no_cpu and world == 1 and not args.nccl_self:
        try:
            cg, info = cpu_reference_workload(args.workload, W, dims, max(2, min(args.steps, 5)), 1, args.sample_nz)
            cpu = {"value": round(cg, 6), "unit": "GLUPS", "cores": info["cores"], "kind": info["kind"],
                   "sample": info["sample"], "host": host_info()}
        except Exception as e:  # report, never fake
            cpu = {"value": None, "unit": "GLUPS", "cores": 0, "kind": "unavailable", "sample": str(e)[:200]}
    if default and rank == 0 and not args.no_cpu and world == 1:
        try:
            cg, info = cpu_reference(max(2, min(args.steps, 5)), 1, args.sample_nz)
            cpu = {"value": round(cg, 6), "unit": "GLUPS", "cores": info["cores"], "kind": info["kind"],
                   "sample": info["sample"], "host": host_info()}
        except Exception as e:  # report, never fake
            cpu = {"value": None, "unit": "GLUPS", "cores": 0, "kind": "unavailable", "sample": str(e)[:200]}

    if rank == 0:
        n_desc = f"{nx}x{ny}x{nzp}" if lat.dim == 3 else f"{nx}x{ny}"
        out = {"metric": metric, "value": round(glups, 4), "unit": "GLUPS", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
               "scaling": scaling, "vs_baseline": None,
               "dtype": ("f64" if args.math == "f64" else "f32") if W["comps"] == 1 else W["storage"],
               "data": "synthetic",
               "config": {"workload": W["desc"].format(n=n_desc) + (" per GPU" if lat.dim == 3 else "")
                          + (f" (global {nx}x{ny}x{nz_g}, {world} z slabs)" if world > 1 else ""),
                          "lattice": lat.name, "nodes": nodes,
                          "storage": W["storage"] if args.storage == "native"
                          else "f16 moments (scaled), f32 populations",
                          **({"solid_fraction": round(float(solid.mean()), 4)} if masked else {}),
                          "node_math": (args.math if W["comps"] == 1 else W["storage"] + " (as the reference)"),
                          "l2": L2_NOTE if nodes > 10 ** 7 else "L2-resident (correctness config)",
                          "parallelism": (f"z-slab x{world} ({'NCCL' if args.transport == 'nccl' else 'peer-memory'} "
                                          f"halos{', all ranks on one device' if one_gpu else ''})") if world > 1 else
                          ("one z slab on a 1-rank NCCL communicator (self halo exchange)" if args.transport == "nccl"
                           else "one z slab exchanging with itself over the peer-memory (CUDA IPC) transport")
                          if self_x
                          else "single GPU"},
               # (how this arm computes the workload; `config` is what both arms run)
               "schedule": ({"m": "M: moment-resident single pass (populations rebuilt in shared "
                                  "memory; f materialised on read)",
                             "f1": "F1: moments + fused stream-collide"}[sched] if W["comps"] == 1
                            else "one pass: colour moments + gradient + prepare + stream-collide-recolour "
                                 "(ping-pong populations)" if "cg_moments" not in prof
                            else "colour moments + fused gradient/prepare/stream-collide-recolour"
                            if "cg_gradient" not in prof
                            else "colour moments + gradient + fused prepare/stream-collide-recolour"),
               "roofline": roof, "gpu_launches": launches, "clocks": clk, "e2e": e2e, "cpu_baseline": cpu}
        print(json.dumps(out), file=out_stream)
    # (a neighbour may still copy into this rank's buffers until every rank
    # is done)
    if dist:
        dist.barrier()
    sim.close()
    if dist:
        dist.destroy_process_group()


def tgv_state_host(dims, amp, tdt):
    """The Taylor-Green node states (rho, u[3]; Pi^neq = 0 as in the
    reference driver's prepare_node(rho, u, 0, ...), tslb_main.cpp:115-122)
    of an nx*ny*nz box in a pinned host tensor (1 + D, n), computed on the
    device plane chunk by plane chunk (untimed set-up of the e2e loop)."""
    import torch
    nx, ny, nz = dims
    plane = nx * ny
    st = torch.zeros((4, plane * nz), dtype=tdt, pin_memory=True)
    dev = torch.device("cuda")
    two_pi = 2.0 * np.pi
    X = two_pi * (torch.arange(nx, device=dev, dtype=torch.float64) + 0.5) / nx
    Y = two_pi * (torch.arange(ny, device=dev, dtype=torch.float64) + 0.5) / ny
    sx, cx, c2x = torch.sin(X), torch.cos(X), torch.cos(2 * X)
    sy, cy, c2y = torch.sin(Y), torch.cos(Y), torch.cos(2 * Y)
    step = max(1, (1 << 26) // plane)
    for k0 in range(0, nz, step):
        k1 = min(nz, k0 + step)
        Z = two_pi * (torch.arange(k0, k1, device=dev, dtype=torch.float64) + 0.5) / nz
        cz, c2z = torch.cos(Z)[:, None, None], torch.cos(2 * Z)[:, None, None]
        rho = 1.0 + 3.0 * (amp * amp / 16.0) * (c2x[None, None, :] + c2y[None, :, None]) * (c2z + 2.0)
        ux = amp * sx[None, None, :] * cy[None, :, None] * cz
        uy = -amp * cx[None, None, :] * sy[None, :, None] * cz
        sl = slice(k0 * plane, k1 * plane)
        st[0, sl].copy_(rho.reshape(-1).to(tdt))
        st[1, sl].copy_(ux.reshape(-1).to(tdt))
        st[2, sl].copy_(uy.reshape(-1).to(tdt))
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return st


def gpu_local_cpus(dev=0):
    """The host CPUs of the GPU's NUMA node (sysfs), or None (one node, or
    no information: the single-socket GPU VMs of this pool). On a
    multi-socket host the e2e loop allocates its pinned buffers from there:
    pages land on the allocating CPU's node, and DMA from the other socket's
    memory would cross the socket link."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(dev)
        addr = f"{int(pr.pci_domain_id):04x}:{int(pr.pci_bus_id):02x}:{int(pr.pci_device_id):02x}.0"
        with open(f"/sys/bus/pci/devices/{addr}/numa_node") as fh:
            node = int(fh.read().strip())
        if node < 0:
            return None
        with open(f"/sys/devices/system/node/node{node}/cpulist") as fh:
            cpus = set()
            for part in fh.read().strip().split(","):
                lo, _, hi = part.partition("-")
                cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:  # (no NUMA information: leave the affinity alone)
        return None


def run_e2e(sim, lat, dims, steps, dtype, amp):
    """The reference driver loop (tslb_main.cpp run_single) through the public
    C-ABI with HOST buffers: the initial rho and u go up from pinned host
    memory into the device initialize_regularized with Pi^neq = 0
    (tslb_cuda_init_equilibrium -- the reference driver's start,
    tslb_main.cpp:115-122 -- chunked upload overlapped with the
    initialisation), `steps` steps each
    followed by a totals() sample read back to the host, then refresh and
    download rho and u (the output frame). Host wall time around it. The
    host buffers live on the GPU's NUMA node (gpu_local_cpus)."""
    import torch

    nn = int(np.prod(dims))
    esz = np.dtype(dtype).itemsize
    tdt = torch.float32 if esz == 4 else torch.float64
    nm = 1 + lat.dim
    saved = os.sched_getaffinity(0)
    local = gpu_local_cpus()
    if local:
        os.sched_setaffinity(0, local)
    try:
        return _run_e2e(sim, lat, dims, steps, dtype, amp, nn, esz, tdt, nm, local)
    finally:
        os.sched_setaffinity(0, saved)


def _run_e2e(sim, lat, dims, steps, dtype, amp, nn, esz, tdt, nm, local):
    import ctypes as C

    import torch

    from paper_2304_06437_b200 import _lib
    try:
        host_state = tgv_state_host(dims, amp, tdt)
        out = torch.empty((1 + lat.dim, nn), dtype=tdt, pin_memory=True)
    except Exception as e:
        return {"value": None, "unit": "GLUPS", "error": f"pinned host alloc failed: {e}"[:200]}
    lib = _lib.load()
    mass = C.c_double()
    mom = (C.c_double * 3)()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(lib.tslb_cuda_init_equilibrium(sim.h, C.c_void_p(host_state.data_ptr())))
    t1 = time.perf_counter()
    for _ in range(steps):
        _lib.check(lib.tslb_cuda_step(sim.h, 1))
        _lib.check(lib.tslb_cuda_totals(sim.h, C.byref(mass), mom))
    t2 = time.perf_counter()
    _lib.check(lib.tslb_cuda_refresh_moments(sim.h))
    t3 = time.perf_counter()
    _lib.check(lib.tslb_cuda_download_field(sim.h, 0, C.c_void_p(out.data_ptr())))
    _lib.check(lib.tslb_cuda_download_field(sim.h, 1, C.c_void_p(out[1:].data_ptr())))
    t = time.perf_counter() - t0
    phases = {"init_equilibrium": round(t1 - t0, 3), "steps_and_totals": round(t2 - t1, 3), "refresh": round(t3 - t2, 3),
              "download": round(t0 + t - t3, 3)}
    h2d = nm * nn * esz
    d2h = (1 + lat.dim) * nn * esz + steps * 32
    return {"value": round(nn * steps / t / 1e9, 4), "unit": "GLUPS", "h2d_bytes_per_step": int(h2d / steps),
            "d2h_bytes_per_step": int(d2h / steps), "seconds": round(t, 3), "phase_seconds": phases,
            "host_cpus": f"{len(local)} on the GPU's NUMA node" if local else "all",
            "loop": "rho, u (pinned) -> init_equilibrium (device initialize_regularized, Pi^neq = 0, upload "
                    "overlapped) -> "
                    "steps x (step + totals readback) -> refresh, download rho,u"}


if __name__ == "__main__":
    main()
