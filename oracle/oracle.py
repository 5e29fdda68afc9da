"""ctypes front-end for the CPU checkers -- TEST INFRASTRUCTURE ONLY.

Two checkers share one calling convention (see tslb_oracle.h):

* ``Oracle("port")``  -> oracle/build/liboracle.so, the plain-C restatement
  (tslb_oracle.c), which also covers D3Q27 (no reference code exists for it).
* ``Oracle("ref")``   -> oracle/_ref/libtslb_ref.so, the UNMODIFIED reference
  headers compiled by oracle/Makefile (only where /root/reference exists, or
  where the prebuilt .so travelled with the repo snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module. The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtslb_ref.so")
REF_INC = "/root/reference/proj/include"

LATTICES = {"d2q9": 0, "d3q19": 1, "d3q27": 2}
FACE = {"periodic": 0, "wall": 1, "moving": 2}


def build(ref: bool = True) -> None:
    """Compile the port (always) and the reference wrapper (if its sources exist)."""
    targets = ["port"]
    if ref and os.path.exists(os.path.join(REF_INC, "tslb", "kernels.hpp")):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def lattice_info(lat: str):
    o = Oracle("port")
    q, dim = C.c_int(), C.c_int()
    c = np.zeros(27 * 3, np.int32)
    opp = np.zeros(27, np.int32)
    t = np.zeros(27)
    b = np.zeros(27)
    o.lib.tslbo_lattice_info(LATTICES[lat], C.byref(q), C.byref(dim), _ptr(c), _ptr(opp), _ptr(t), _ptr(b))
    qq = q.value
    return dict(q=qq, dim=dim.value, c=c[: 3 * qq].reshape(qq, 3).copy(), opp=opp[:qq].copy(), t=t[:qq].copy(), b=b[:qq].copy())


def faces_arrays(faces):
    """faces: list of 6 (kind, (ux, uy, uz)) -> (int32[6], float64[18])."""
    kinds = np.array([FACE[k] if isinstance(k, str) else int(k) for k, _ in faces], np.int32)
    uw = np.array([float(v) for _, u in faces for v in u], np.float64)
    return kinds, uw


def periodic():
    return [("periodic", (0.0, 0.0, 0.0))] * 6


def closed_box():
    return [("wall", (0.0, 0.0, 0.0))] * 6


def lid_cavity(u):
    f = closed_box()
    f[3] = ("moving", (u, 0.0, 0.0))
    return f


class Oracle:
    """One CPU checker (``kind`` = "port" or "ref")."""

    _cache: dict = {}

    def __init__(self, kind: str = "port"):
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run oracle.build())")
        if path not in Oracle._cache:
            Oracle._cache[path] = C.CDLL(path)
        self.lib = Oracle._cache[path]
        self.kind = kind
        self.pre = "tslbo_" if kind == "port" else "tslbref_"
        vp, i, d, l = C.c_void_p, C.c_int, C.c_double, C.c_long
        self._fn("single_run").argtypes = [i, i, i, i, i, d, vp, vp, vp, vp, vp, l] + ([i, i] if kind == "ref" else [i])
        self._fn("two_run").argtypes = [i, i, i, i, i, d, vp, vp, vp, vp, vp, vp, vp, vp, vp, l] + ([i, i, i, vp] if kind == "ref" else [i, i, vp])
        self._fn("classify").argtypes = [i, i, i, i, vp, vp, vp, vp, vp, vp]
        self._fn("last_error").restype = C.c_char_p
        self._fn("fnv1a").restype = C.c_uint64
        self._fn("fnv1a").argtypes = [vp, C.c_size_t, C.c_uint64]
        if kind == "port":
            self._fn("init_regularized").argtypes = [i, i, i, i, i, vp, vp, vp]
            self._fn("init_colors").argtypes = [i, i, i, i, i, vp, vp, vp, vp]
            self._fn("totals").argtypes = [i, i, C.c_uint64, vp, vp, vp, vp, vp]
            self._fn("stability").argtypes = [i, i, C.c_uint64, vp, vp, vp, vp, vp, vp, vp]
            self._fn("census").argtypes = [i, i, vp, vp]
        else:
            self._fn("time_steps").argtypes = [i, i, i, i, i, d, vp, vp, vp, l, l, i, vp]
            self._fn("time_steps_ex").argtypes = [i, i, i, i, i, d, vp, vp, vp, vp, l, l, i, vp]
            self._fn("time_two").argtypes = [i, i, i, i, i, d, vp, vp, vp, vp, vp, vp, l, l, i, vp]
            self._fn("bench").argtypes = [i, i, i, i, i, d, l, l, i, vp, vp, vp]

    def _fn(self, name):
        return getattr(self.lib, self.pre + name)

    def _check(self, rc):
        if rc != 0:
            raise ValueError(self._fn("last_error")().decode())

    # -- geometry ---------------------------------------------------------
    def classify(self, lat, dims, faces, solid=None):
        nx, ny, nz = dims
        n = nx * ny * nz
        kinds, uw = faces_arrays(faces)
        so = np.zeros(n, np.uint8)
        sl = np.zeros(n, np.uint32)
        nf = C.c_uint64()
        sol = None if solid is None else np.ascontiguousarray(solid, np.uint8)
        self._check(self._fn("classify")(LATTICES[lat], nx, ny, nz, _ptr(kinds), _ptr(uw), _ptr(sol), _ptr(so), _ptr(sl), C.byref(nf)))
        return so, sl, int(nf.value)

    def set_body_force(self, fx=0.0, fy=0.0, fz=0.0):
        """Body-force extension of the port (not in the reference)."""
        if self.kind != "port":
            raise ValueError("the reference has no single-fluid body force")
        self.lib.tslbo_set_body_force(C.c_double(fx), C.c_double(fy), C.c_double(fz))

    # -- single fluid -----------------------------------------------------
    def single_run(self, lat, dims, omega, faces, f, moments=None, steps=1, mode=0, solid=None, workers=1):
        """Advance f (q, n) in place; returns (f, moments)."""
        nx, ny, nz = dims
        scalar = 0 if f.dtype == np.float64 else 1
        kinds, uw = faces_arrays(faces)
        sol = None if solid is None else np.ascontiguousarray(solid, np.uint8)
        assert f.flags.c_contiguous
        if moments is not None:
            assert moments.flags.c_contiguous and moments.dtype == f.dtype
        args = [LATTICES[lat], scalar, nx, ny, nz, float(omega), _ptr(kinds), _ptr(uw), _ptr(sol), _ptr(f), _ptr(moments), int(steps)]
        args += [workers, mode] if self.kind == "ref" else [mode]
        self._check(self._fn("single_run")(*args))
        return f, moments

    # -- two fluid --------------------------------------------------------
    def two_run(self, lat, dims, omega, color, faces, fr, fb, steps=1, refresh=False, mode=0, solid=None, phi=None, workers=1):
        """color: dict(sigma, beta, nci_strength, eps_bulk, grad_threshold, nci_reach, linear)."""
        nx, ny, nz = dims
        n = nx * ny * nz
        dt = fr.dtype if fr is not None else phi.dtype
        scalar = 0 if dt == np.float64 else 1
        info = lattice_info(lat)
        D = info["dim"]
        np_ = D * (D + 1) // 2
        kinds, uw = faces_arrays(faces)
        cp = np.array([color.get("sigma", 0.01), color.get("beta", 0.7), color.get("nci_strength", 0.0),
                       color.get("eps_bulk", 0.02), color.get("grad_threshold", 1e-6)], np.float64)
        ip = np.array([color.get("nci_reach", 3), 1 if color.get("linear", False) else 0], np.int32)
        out = np.zeros((3 + D + np_ + 1 + D, n), dt)
        flags = np.zeros(n, np.uint8)
        sol = None if solid is None else np.ascontiguousarray(solid, np.uint8)
        args = [LATTICES[lat], scalar, nx, ny, nz, float(omega), _ptr(cp), _ptr(ip), _ptr(kinds), _ptr(uw), _ptr(sol),
                _ptr(fr), _ptr(fb), _ptr(out), _ptr(flags), int(steps)]
        if self.kind == "ref":
            args += [workers, int(refresh), mode, _ptr(phi)]
        else:
            args += [int(refresh), mode, _ptr(phi)]
        self._check(self._fn("two_run")(*args))
        names = ["rho_r", "rho_b", "rho"] + [f"mom{d}" for d in range(D)] + [f"pineq{p}" for p in range(np_)] + ["phi"] + [f"grad{d}" for d in range(D)]
        res = {k: out[i] for i, k in enumerate(names)}
        res["mom"] = out[3:3 + D]
        res["pineq"] = out[3 + D:3 + D + np_]
        res["gradphi"] = out[4 + D + np_:]
        res["nci_flag"] = flags
        return res

    # -- port-only helpers --------------------------------------------------
    def init_regularized(self, lat, dims, state, solid=None):
        """state (10, n) of the storage dtype -> f (q, n)."""
        nx, ny, nz = dims
        info = lattice_info(lat)
        state = np.ascontiguousarray(state)
        f = np.zeros((info["q"], nx * ny * nz), state.dtype)
        scalar = 0 if state.dtype == np.float64 else 1
        sol = None if solid is None else np.ascontiguousarray(solid, np.uint8)
        self._check(self._fn("init_regularized")(LATTICES[lat], scalar, nx, ny, nz, _ptr(sol), _ptr(state), _ptr(f)))
        return f

    def init_colors(self, lat, dims, state, solid=None):
        nx, ny, nz = dims
        info = lattice_info(lat)
        state = np.ascontiguousarray(state)
        fr = np.zeros((info["q"], nx * ny * nz), state.dtype)
        fb = np.zeros_like(fr)
        scalar = 0 if state.dtype == np.float64 else 1
        sol = None if solid is None else np.ascontiguousarray(solid, np.uint8)
        self._check(self._fn("init_colors")(LATTICES[lat], scalar, nx, ny, nz, _ptr(sol), _ptr(state), _ptr(fr), _ptr(fb)))
        return fr, fb

    def totals(self, rho, mom, solid=None):
        scalar = 0 if rho.dtype == np.float64 else 1
        mass = C.c_double()
        m = np.zeros(3)
        mom = np.ascontiguousarray(mom)
        sol = None if solid is None else np.ascontiguousarray(solid, np.uint8)
        self._check(self._fn("totals")(scalar, mom.shape[0], rho.size, _ptr(sol), _ptr(rho), _ptr(mom), C.byref(mass), _ptr(m)))
        return mass.value, m

    def stability(self, rho, mom, solid=None):
        scalar = 0 if rho.dtype == np.float64 else 1
        fin = C.c_int()
        ms, lo, hi = C.c_double(), C.c_double(), C.c_double()
        mom = np.ascontiguousarray(mom)
        sol = None if solid is None else np.ascontiguousarray(solid, np.uint8)
        self._check(self._fn("stability")(scalar, mom.shape[0], rho.size, _ptr(sol), _ptr(rho), _ptr(mom), C.byref(fin), C.byref(ms), C.byref(lo), C.byref(hi)))
        return dict(finite=bool(fin.value), max_speed=ms.value, min_rho=lo.value, max_rho=hi.value)

    def census(self, lat, elem_bytes):
        fl, by = C.c_double(), C.c_double()
        self._fn("census")(LATTICES[lat], elem_bytes, C.byref(fl), C.byref(by))
        return fl.value, by.value

    def fnv1a(self, arr, h=0xCBF29CE484222325):
        arr = np.ascontiguousarray(arr)
        return int(self._fn("fnv1a")(_ptr(arr), arr.nbytes, h))


def moments_layout(lat):
    info = lattice_info(lat)
    D = info["dim"]
    return 1 + D + D * (D + 1) // 2


def random_state(lat, dims, seed, dtype=np.float64, solid=None):
    """Near-equilibrium random f in the spirit of the reference fixtures
    (unit_collision_stream.cpp:36-58): rho~U(.92,1.08), u~U(-.04,.04),
    f = feq * (1 + U(-.02,.02)); numpy RNG (not mt19937), values computed in
    double then rounded to the storage dtype."""
    info = lattice_info(lat)
    n = int(np.prod(dims))
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.92, 1.08, n)
    u = rng.uniform(-0.04, 0.04, (3, n))
    if info["dim"] == 2:
        u[2] = 0.0
    c = info["c"].astype(np.float64)
    t = info["t"]
    cu = c @ u
    usq = 1.5 * (u * u).sum(0)
    feq = t[:, None] * (rho[None, :] + 3 * cu + 4.5 * cu * cu - usq[None, :])
    f = feq * (1.0 + rng.uniform(-0.02, 0.02, feq.shape))
    if solid is not None:
        f[:, np.asarray(solid, bool)] = 0.0
    return np.ascontiguousarray(f.astype(dtype))
