"""Python mirror of the reference's solver/lattice interface, over the C-ABI.

Names, argument meaning and error behaviour follow the reference tslb
headers (proj/include/tslb/*.hpp) so that tests read like the reference's
own (tests/unit_*.cpp). The C++ drop-in for C++ callers is include/tslb/;
this module is the same contract for Python callers and for bench.py.

Template parameters become arguments: ``SingleFluidSim<D3Q19, float>`` is
``SingleFluidSim(D3Q19, g, prm, spec, dtype=np.float32)``.

Host-visible semantics kept from the reference:
  * after ``step()`` f is f(t+1) while the moment arrays still hold m(t)
    (solver.hpp:68-69); ``refresh_moments()`` gives m(t+1);
  * two-fluid: after a step ``mom``/``pineq`` hold u_eq / Pi^neq, after
    ``refresh_moments`` the bare j / raw second moment (solver.hpp:163-166);
  * ``fields()`` returns host arrays the caller may modify; modifications are
    uploaded before the next device operation (``view()`` is read-only).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _lib
from ._lib import InvalidArgument, TslbCudaError

# ---------------------------------------------------------------------------
# lattices (lattice.hpp:15-75; D3Q27 new)
# ---------------------------------------------------------------------------


class LatticeKind:
    D2Q9 = _lib.D2Q9
    D3Q19 = _lib.D3Q19
    D3Q27 = _lib.D3Q27


@dataclass(frozen=True)
class Lattice:
    kind: int
    name: str
    dim: int
    c: tuple
    t_rat: tuple
    b_rat: tuple

    @property
    def q(self) -> int:
        return len(self.c)

    @property
    def opp(self) -> list[int]:
        return [0] + [a + 1 if a % 2 == 1 else a - 1 for a in range(1, self.q)]

    @property
    def npineq(self) -> int:
        return self.dim * (self.dim + 1) // 2


_AX = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
_FD = [(1, 1, 0), (-1, -1, 0), (1, -1, 0), (-1, 1, 0), (1, 0, 1), (-1, 0, -1), (1, 0, -1), (-1, 0, 1),
       (0, 1, 1), (0, -1, -1), (0, 1, -1), (0, -1, 1)]
_CR = [(1, 1, 1), (-1, -1, -1), (1, 1, -1), (-1, -1, 1), (1, -1, 1), (-1, 1, -1), (-1, 1, 1), (1, -1, -1)]

D2Q9 = Lattice(LatticeKind.D2Q9, "d2q9", 2,
               tuple([(0, 0, 0)] + _AX[:4] + [(1, 1, 0), (-1, -1, 0), (1, -1, 0), (-1, 1, 0)]),
               tuple([(4, 9)] + [(1, 9)] * 4 + [(1, 36)] * 4),
               tuple([(-4, 27)] + [(2, 27)] * 4 + [(5, 108)] * 4))
D3Q19 = Lattice(LatticeKind.D3Q19, "d3q19", 3, tuple([(0, 0, 0)] + _AX + _FD),
                tuple([(1, 3)] + [(1, 18)] * 6 + [(1, 36)] * 12),
                tuple([(-1, 3)] + [(1, 18)] * 6 + [(1, 36)] * 12))
D3Q27 = Lattice(LatticeKind.D3Q27, "d3q27", 3, tuple([(0, 0, 0)] + _AX + _FD + _CR),
                tuple([(8, 27)] + [(2, 27)] * 6 + [(1, 54)] * 12 + [(1, 216)] * 8),
                tuple([(-1, 3)] + [(1, 18)] * 6 + [(1, 36)] * 12 + [(0, 1)] * 8))
LATTICES = {0: D2Q9, 1: D3Q19, 2: D3Q27, "d2q9": D2Q9, "d3q19": D3Q19, "d3q27": D3Q27}


def lattice_of(x) -> Lattice:
    return x if isinstance(x, Lattice) else LATTICES[x]


def lattice_name(k) -> str:
    return lattice_of(k).name


def dispatch_lattice(kind, fn: Callable):
    """solver.hpp:20-24 -- call fn with the lattice for a runtime kind."""
    return fn(lattice_of(kind))


def weights(lat: Lattice, dtype=np.float64) -> np.ndarray:
    dt = np.dtype(dtype).type
    return np.array([dt(n) / dt(d) for n, d in lat.t_rat], dtype=dtype)


def cs2(dtype=np.float64):
    dt = np.dtype(dtype).type
    return dt(1) / dt(3)


# ---------------------------------------------------------------------------
# fields, geometry, parameters (fields.hpp, boundary.hpp, collision.hpp,
# multicomponent.hpp:24-33)
# ---------------------------------------------------------------------------


@dataclass
class GridDims:
    nx: int = 0
    ny: int = 0
    nz: int = 1

    def n(self) -> int:
        return self.nx * self.ny * self.nz

    def valid(self) -> bool:
        return self.nx > 0 and self.ny > 0 and self.nz > 0

    def tuple(self):
        return (self.nx, self.ny, self.nz)


def linear_index(g: GridDims, i: int, j: int, k: int) -> int:
    return i + g.nx * (j + g.ny * k)


def wrap(i: int, n: int) -> int:
    return i % n


class FaceKind:
    Periodic = _lib.FACE_PERIODIC
    NoSlipWall = _lib.FACE_WALL
    MovingWall = _lib.FACE_MOVING


XMin, XMax, YMin, YMax, ZMin, ZMax = range(6)


@dataclass
class Face:
    kind: int = FaceKind.Periodic
    u_wall: tuple = (0.0, 0.0, 0.0)


@dataclass
class BoundarySpec:
    faces: list = field(default_factory=lambda: [Face() for _ in range(6)])

    @staticmethod
    def all_periodic() -> "BoundarySpec":
        return BoundarySpec()

    @staticmethod
    def closed_box() -> "BoundarySpec":
        return BoundarySpec([Face(FaceKind.NoSlipWall) for _ in range(6)])

    @staticmethod
    def lid_cavity(u_lid: float) -> "BoundarySpec":
        s = BoundarySpec.closed_box()
        s.faces[YMax] = Face(FaceKind.MovingWall, (u_lid, 0.0, 0.0))
        return s

    def arrays(self):
        kinds = np.array([f.kind for f in self.faces], np.int32)
        uw = np.array([float(v) for f in self.faces for v in f.u_wall], np.float64)
        return kinds, uw


@dataclass
class CollisionParams:
    omega: float = 1.0
    rho0: float = 1.0
    # single-fluid body force: an extension (the reference has none)
    force: tuple = (0.0, 0.0, 0.0)

    def tau(self) -> float:
        return 1.0 / self.omega

    def nu(self) -> float:
        return (1.0 / 3.0) * (self.tau() - 0.5)


def omega_from_nu(nu: float) -> float:
    return 1.0 / (nu / (1.0 / 3.0) + 0.5)


def omega_from_tau(tau: float) -> float:
    return 1.0 / tau


def nu_from_omega(omega: float) -> float:
    return (1.0 / 3.0) * (1.0 / omega - 0.5)


class PerturbationForm:
    Squared = 0
    Linear = 1


@dataclass
class ColorParams:
    sigma: float = 0.01
    beta: float = 0.7
    nci_strength: float = 0.0
    nci_reach: int = 3
    eps_bulk: float = 0.02
    grad_threshold: float = 1e-6
    form: int = PerturbationForm.Squared

    def arrays(self):
        return (np.array([self.sigma, self.beta, self.nci_strength, self.eps_bulk, self.grad_threshold], np.float64),
                np.array([self.nci_reach, self.form], np.int32))


@dataclass
class FieldSet:
    dims: GridDims
    q: int
    dim: int
    f: np.ndarray       # (q, n)
    rho: np.ndarray     # (n,)
    mom: np.ndarray     # (dim, n)
    pineq: np.ndarray   # (np, n)

    def n(self) -> int:
        return self.dims.n()

    def npineq(self) -> int:
        return self.dim * (self.dim + 1) // 2

    def copy(self) -> "FieldSet":
        return FieldSet(self.dims, self.q, self.dim, self.f.copy(), self.rho.copy(), self.mom.copy(), self.pineq.copy())


@dataclass
class TwoFluidFieldSet:
    dims: GridDims
    q: int
    dim: int
    fr: np.ndarray
    fb: np.ndarray
    rho_r: np.ndarray
    rho_b: np.ndarray
    rho: np.ndarray
    mom: np.ndarray
    pineq: np.ndarray
    phi: np.ndarray
    gradphi: np.ndarray
    nci_flag: np.ndarray

    def n(self) -> int:
        return self.dims.n()


def allocate_fields(g: GridDims, lat, dtype=np.float64) -> FieldSet:
    """fields.hpp:82-97"""
    if not g.valid():
        raise InvalidArgument("allocate_fields: bad dims")
    L = lattice_of(lat)
    n = g.n()
    return FieldSet(g, L.q, L.dim, np.zeros((L.q, n), dtype), np.zeros(n, dtype), np.zeros((L.dim, n), dtype),
                    np.zeros((L.npineq, n), dtype))


def allocate_two_fluid(g: GridDims, lat, dtype=np.float64) -> TwoFluidFieldSet:
    """fields.hpp:99-125"""
    if not g.valid():
        raise InvalidArgument("allocate_two_fluid: bad dims")
    L = lattice_of(lat)
    n = g.n()
    z = lambda *s: np.zeros(s, dtype)
    return TwoFluidFieldSet(g, L.q, L.dim, z(L.q, n), z(L.q, n), z(n), z(n), z(n), z(L.dim, n), z(L.npineq, n), z(n),
                            z(L.dim, n), np.zeros(n, np.uint8))


@dataclass
class NodeGeometry:
    dims: GridDims
    solid: np.ndarray
    slow_mask: np.ndarray
    n_fluid: int


@dataclass
class StabilityReport:
    finite: bool = True
    max_speed: float = 0.0
    min_rho: float = 0.0
    max_rho: float = 0.0
    first_bad: int = -1

    def stable(self) -> bool:
        return self.finite and self.max_speed < 0.3 * 0.57735026918962576


def _scalar_id(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return _lib.F64
    if dt == np.float32:
        return _lib.F32
    raise InvalidArgument(f"unsupported scalar type {dt}")


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# device solver handle (thin RAII over tslb_cuda_create/destroy)
# ---------------------------------------------------------------------------


class DeviceSolver:
    """Owns one C-ABI handle. All methods raise on a nonzero status."""

    def __init__(self, lat, g: GridDims, omega: float, spec: BoundarySpec, dtype=np.float64, components: int = 1,
                 solid=None, color: ColorParams | None = None, device: int = 0, slab: tuple | None = None):
        lib = _lib.load()
        self.lat = lattice_of(lat)
        self.dims = g
        self.dtype = np.dtype(dtype)
        self.components = components
        kinds, uw = spec.arrays()
        cpd, cpi = (color or ColorParams()).arrays()
        sol = None
        if solid is not None:
            sol = np.ascontiguousarray(np.asarray(solid, np.uint8))
            if sol.size != g.n():
                raise InvalidArgument("classify_nodes: mask size mismatch")
        h = C.c_void_p()
        if slab is None:
            rc = lib.tslb_cuda_create(self.lat.kind, _scalar_id(dtype), components, g.nx, g.ny, g.nz, float(omega),
                                      _ptr(kinds), _ptr(uw), _ptr(sol), _ptr(cpd), _ptr(cpi), device, C.byref(h))
            self.z0, self.nzl = 0, g.nz
        else:
            z0, nzl = slab
            rc = lib.tslb_cuda_create_slab(self.lat.kind, _scalar_id(dtype), components, g.nx, g.ny, g.nz, z0, nzl,
                                           float(omega), _ptr(kinds), _ptr(uw), _ptr(sol), _ptr(cpd), _ptr(cpi),
                                           device, C.byref(h))
            self.z0, self.nzl = z0, nzl
        _lib.check(rc)
        self.h = h
        self.n = g.nx * g.ny * self.nzl

    def close(self):
        if getattr(self, "h", None):
            _lib.load().tslb_cuda_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _call(self, name, *args):
        _lib.check(getattr(_lib.load(), name)(self.h, *args))

    # data movement
    def upload_f(self, f, species=0):
        f = np.ascontiguousarray(f, self.dtype)
        if f.shape != (self.lat.q, self.n):
            raise _lib.InvalidArgument(f"upload_f: expected shape {(self.lat.q, self.n)}, got {f.shape}")
        self._call("tslb_cuda_upload_f", species, _ptr(f))

    def download_f(self, species=0, out=None):
        """f of one species as (q, n); `out` (optional) must be a C-contiguous
        array of the solver's dtype and exactly that shape -- the C-ABI
        writes q * n elements into it."""
        if out is None:
            out = np.empty((self.lat.q, self.n), self.dtype)
        elif (not isinstance(out, np.ndarray) or out.dtype != self.dtype or out.shape != (self.lat.q, self.n)
              or not out.flags.c_contiguous or not out.flags.writeable):
            raise _lib.InvalidArgument(
                f"download_f: out must be a writeable C-contiguous {np.dtype(self.dtype).name} array of shape "
                f"{(self.lat.q, self.n)}")
        self._call("tslb_cuda_download_f", species, _ptr(out))
        return out

    _FIELD_SHAPE = dict(rho=1, mom="D", pineq="P", rho_r=1, rho_b=1, phi=1, gradphi="D", nci_flag=1, solid=1,
                        slow_mask=1)

    def _fshape(self, name):
        k = self._FIELD_SHAPE[name]
        cnt = self.lat.dim if k == "D" else self.lat.npineq if k == "P" else 1
        dt = np.uint8 if name in ("nci_flag", "solid") else np.uint32 if name == "slow_mask" else self.dtype
        return cnt, dt

    def download_field(self, name):
        cnt, dt = self._fshape(name)
        out = np.empty((cnt, self.n), dt)
        self._call("tslb_cuda_download_field", _lib.FIELD[name], _ptr(out))
        return out[0] if cnt == 1 else out

    def download_slice(self, name, axis: int, index: int) -> np.ndarray:
        """One 2-D slice of a field (device-side sampler, tslb_cuda.h):
        returns (arrays, rows, cols) with the fastest axis last."""
        cnt, dt = self._fshape(name)
        ext = [self.dims.nx, self.dims.ny, self.nzl]
        rows_cols = {2: (ext[1], ext[0]), 1: (ext[2], ext[0]), 0: (ext[2], ext[1])}[axis]
        out = np.empty((cnt, *rows_cols), dt)
        self._call("tslb_cuda_download_slice", _lib.FIELD[name], int(axis), int(index), _ptr(out))
        return out

    def upload_field(self, name, arr):
        cnt, dt = self._fshape(name)
        a = np.asarray(arr, dt)
        if a.size != cnt * self.n:
            raise _lib.InvalidArgument(f"upload_field({name}): expected {cnt * self.n} values, got {a.size}")
        a = np.ascontiguousarray(a.reshape(cnt, self.n))
        self._call("tslb_cuda_upload_field", _lib.FIELD[name], _ptr(a))

    def geometry(self) -> NodeGeometry:
        solid = np.empty(self.n, np.uint8)
        slow = np.empty(self.n, np.uint32)
        nf = C.c_uint64()
        self._call("tslb_cuda_download_geometry", _ptr(solid), _ptr(slow), C.byref(nf))
        return NodeGeometry(GridDims(self.dims.nx, self.dims.ny, self.nzl), solid, slow, int(nf.value))

    # stepping & phases
    def step(self, n=1):
        self._call("tslb_cuda_step", int(n))

    def step_async(self, n=1):
        self._call("tslb_cuda_step_async", int(n))

    def synchronize(self):
        self._call("tslb_cuda_synchronize")

    def time_steps(self, n) -> float:
        ms = C.c_double()
        self._call("tslb_cuda_time_steps", int(n), C.byref(ms))
        return ms.value

    def phase(self, name, *args):
        self._call("tslb_cuda_" + name, *args)

    def set_math(self, mode: int):
        self._call("tslb_cuda_set_math", mode)

    def set_schedule(self, schedule: str):
        """"f1" (moments pass + fused stream-collide) or "m" (moment-resident
        single pass); same results bit for bit."""
        self._call("tslb_cuda_set_schedule", {"f1": _lib.SCHED_F1, "m": _lib.SCHED_M}[schedule])

    def set_moment_storage(self, kind: str):
        """"f16": the M steps keep the moments as scaled fp16 (40 B per
        lattice update) with fp32 node arithmetic -- a tolerance mode
        (tslb_cuda.h); "native": the storage scalar."""
        self._call("tslb_cuda_set_moment_storage", {"native": _lib.STORE_NATIVE, "f16": _lib.STORE_F16}[kind])

    def set_body_force(self, fx=0.0, fy=0.0, fz=0.0):
        """Single-fluid body force (extension)."""
        f = np.array([fx, fy, fz], np.float64)
        self._call("tslb_cuda_set_body_force", _ptr(f))

    @property
    def schedule(self) -> str:
        v = C.c_int()
        self._call("tslb_cuda_get_schedule", C.byref(v))
        return "m" if v.value == _lib.SCHED_M else "f1"

    def init_analytic(self, kind: str, amplitude=0.0, radius=0.0):
        self._call("tslb_cuda_init_analytic", _lib.INIT[kind], float(amplitude), float(radius))

    def init_state(self, state):
        """initialize_regularized on the device from host node states: an
        array (1 + D + np, n) of the storage dtype -- rho, u[D], Pi[np] per
        node (kernels.hpp:296-311). Pinned host memory (e.g. a torch tensor
        with pin_memory) is taken as is, by pointer."""
        self._init_states("tslb_cuda_init_state", state, 1 + self.lat.dim + self.lat.npineq)

    def init_equilibrium(self, state):
        """The same from rho and u alone, Pi^neq = 0 (the reference driver's
        prepare_node(rho, u, 0, ...), tslb_main.cpp:115-122): an array
        (1 + D, n) of the storage dtype."""
        self._init_states("tslb_cuda_init_equilibrium", state, 1 + self.lat.dim)

    # peer-memory slab transport (tslb_cuda_ipc_handle / tslb_cuda_attach_ipc)
    IPC_HANDLE_BYTES = 64

    def ipc_handle(self) -> bytes:
        """This slab's CUDA IPC handle (ghost planes + flag words), to send
        to the z neighbours' processes."""
        buf = (C.c_char * self.IPC_HANDLE_BYTES)()
        self._call("tslb_cuda_ipc_handle", buf)
        return bytes(buf)

    def attach_ipc(self, below: bytes | None, above: bytes | None):
        """Map the neighbours' handles (None for a wall face); the slab then
        steps with the peer-memory transport."""
        def arg(b):
            if b is None:
                return None
            if len(b) != self.IPC_HANDLE_BYTES:
                raise _lib.InvalidArgument(f"attach_ipc: a handle is {self.IPC_HANDLE_BYTES} bytes")
            return C.create_string_buffer(bytes(b), self.IPC_HANDLE_BYTES)
        self._call("tslb_cuda_attach_ipc", arg(below), arg(above))

    def _init_states(self, fn, state, nm):
        name = fn[len("tslb_cuda_"):]
        if hasattr(state, "data_ptr"):  # a torch tensor (pinned host buffer)
            if tuple(state.shape) != (nm, self.n) or not state.is_contiguous() or state.element_size() != \
                    np.dtype(self.dtype).itemsize or state.is_cuda:
                raise _lib.InvalidArgument(f"{name}: expected a contiguous host tensor of shape {(nm, self.n)}")
            self._call(fn, C.c_void_p(state.data_ptr()))
            return
        a = np.ascontiguousarray(state, self.dtype)
        if a.shape != (nm, self.n):
            raise _lib.InvalidArgument(f"{name}: expected shape {(nm, self.n)}, got {a.shape}")
        self._call(fn, _ptr(a))

    # diagnostics
    def totals(self):
        mass = C.c_double()
        mom = np.zeros(3)
        self._call("tslb_cuda_totals", C.byref(mass), _ptr(mom))
        return mass.value, mom

    def stability(self) -> StabilityReport:
        fin = C.c_int()
        ms, lo, hi = C.c_double(), C.c_double(), C.c_double()
        fb = C.c_int64()
        self._call("tslb_cuda_stability", C.byref(fin), C.byref(ms), C.byref(lo), C.byref(hi), C.byref(fb))
        return StabilityReport(bool(fin.value), ms.value, lo.value, hi.value, int(fb.value))

    def color_masses(self):
        r, b = C.c_double(), C.c_double()
        self._call("tslb_cuda_color_masses", C.byref(r), C.byref(b))
        return r.value, b.value

    def plane_digests(self) -> np.ndarray:
        out = np.zeros(self.components * self.lat.q * self.nzl, np.uint64)
        self._call("tslb_cuda_plane_digests", _ptr(out))
        return out.reshape(self.components, self.lat.q, self.nzl)

    def profile(self, on=True):
        self._call("tslb_cuda_profile", int(on))

    def profile_read(self):
        ms = np.zeros(len(_lib.KCLASS))
        cnt = np.zeros(len(_lib.KCLASS), np.int64)
        self._call("tslb_cuda_profile_read", _ptr(ms), _ptr(cnt))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(_lib.KCLASS) if cnt[i]}

    def steps_done(self) -> int:
        v = C.c_long()
        self._call("tslb_cuda_steps_done", C.byref(v))
        return v.value

    def launch_count(self) -> int:
        v = C.c_int64()
        self._call("tslb_cuda_launch_count", C.byref(v))
        return v.value

    def memory_bytes(self) -> int:
        v = C.c_uint64()
        self._call("tslb_cuda_memory_bytes", C.byref(v))
        return v.value


# ---------------------------------------------------------------------------
# host-side node algebra (initialisers only; T arithmetic in numpy, same
# operand order as collision.hpp so inits are bit-identical to the reference)
# ---------------------------------------------------------------------------


def prepare_node(rho, ux, uy, uz, pxx, pyy, pzz, pxy, pxz, pyz, dtype=np.float64):
    """collision.hpp:72-89 on arrays (or scalars) of the storage dtype."""
    dt = np.dtype(dtype).type
    a = [np.asarray(v, dtype=dtype) for v in (rho, ux, uy, uz, pxx, pyy, pzz, pxy, pxz, pyz)]
    rho, ux, uy, uz, pxx, pyy, pzz, pxy, pxz, pyz = a
    return dict(rho=rho, ux=ux, uy=uy, uz=uz, usq15=dt(1.5) * (ux * ux + uy * uy + uz * uz), pxx=pxx, pyy=pyy,
                pzz=pzz, pxy2=pxy + pxy, pxz2=pxz + pxz, pyz2=pyz + pyz, trcs2=cs2(dtype) * (pxx + pyy + pzz))


def _dotc(c, x, y, z, dtype):
    s = np.zeros_like(np.asarray(x, dtype=dtype))
    for comp, v in zip(c, (x, y, z)):
        if comp == 1:
            s = s + v
        elif comp == -1:
            s = s - v
    return s


def equilibrium_dir(lat, a, m, dtype=np.float64):
    L = lattice_of(lat)
    dt = np.dtype(dtype).type
    t = dt(L.t_rat[a][0]) / dt(L.t_rat[a][1])
    cu = _dotc(L.c[a], m["ux"], m["uy"], m["uz"], dtype)
    return t * (m["rho"] + dt(3) * cu + dt(4.5) * cu * cu - m["usq15"])


def regularized_dir(lat, a, m, dtype=np.float64):
    L = lattice_of(lat)
    dt = np.dtype(dtype).type
    t = dt(L.t_rat[a][0]) / dt(L.t_rat[a][1])
    cx, cy, cz = L.c[a]
    s = np.zeros_like(m["rho"])
    if cx != 0:
        s = s + m["pxx"]
    if cy != 0:
        s = s + m["pyy"]
    if cz != 0:
        s = s + m["pzz"]
    for p, key in ((cx * cy, "pxy2"), (cx * cz, "pxz2"), (cy * cz, "pyz2")):
        if p == 1:
            s = s + m[key]
        elif p == -1:
            s = s - m[key]
    return t * dt(4.5) * (s - m["trcs2"])


def _coords(g: GridDims):
    k, j, i = np.meshgrid(np.arange(g.nz), np.arange(g.ny), np.arange(g.nx), indexing="ij")
    return i.ravel(), j.ravel(), k.ravel()


def initialize_regularized(s: FieldSet, geo: NodeGeometry | None, node_state: Callable, lat=None):
    """kernels.hpp:295-311. node_state(i, j, k) is called ONCE with coordinate
    arrays and returns the 10 prepare_node arguments (arrays or scalars) in
    the storage dtype: rho ux uy uz pxx pyy pzz pxy pxz pyz."""
    L = lattice_of(lat) if lat is not None else (D2Q9 if s.dim == 2 else (D3Q19 if s.q == 19 else D3Q27))
    dtype = s.f.dtype
    i, j, k = _coords(s.dims)
    st = node_state(i, j, k)
    n = s.n()
    args = [np.broadcast_to(np.asarray(v, dtype=dtype), (n,)) for v in st]
    m = prepare_node(*args, dtype=dtype)
    fluid = np.ones(n, bool) if geo is None else geo.solid == 0
    for a in range(L.q):
        v = equilibrium_dir(L, a, m, dtype) + regularized_dir(L, a, m, dtype)
        s.f[a, fluid] = v[fluid]


def initialize_colors(s: TwoFluidFieldSet, geo: NodeGeometry | None, node_state: Callable, lat=None):
    """multicomponent.hpp:427-449. node_state(i, j, k) -> (rho_r, rho_b, ux,
    uy, uz) arrays in the storage dtype."""
    L = lattice_of(lat) if lat is not None else (D2Q9 if s.dim == 2 else (D3Q19 if s.q == 19 else D3Q27))
    dtype = s.fr.dtype
    i, j, k = _coords(s.dims)
    n = s.n()
    rr, rb, ux, uy, uz = [np.broadcast_to(np.asarray(v, dtype=dtype), (n,)) for v in node_state(i, j, k)]
    r = rr + rb
    z = np.zeros(n, dtype)
    m = prepare_node(r, ux, uy, uz, z, z, z, z, z, z, dtype=dtype)
    frac = rr / r
    fluid = np.ones(n, bool) if geo is None else geo.solid == 0
    for a in range(L.q):
        fe = equilibrium_dir(L, a, m, dtype)
        s.fr[a, fluid] = (frac * fe)[fluid]
        s.fb[a, fluid] = (fe - frac * fe)[fluid]


# ---------------------------------------------------------------------------
# solvers
# ---------------------------------------------------------------------------


class _SimBase:
    def __init__(self, lat, g: GridDims, prm: CollisionParams, spec: BoundarySpec, solid, dtype, components, cp,
                 device):
        self.lattice = lattice_of(lat)
        self._dims = g
        self._prm = prm
        self._spec = spec
        self._cp = cp
        self.dtype = np.dtype(dtype)
        self.dev = DeviceSolver(self.lattice, g, prm.omega, spec, dtype, components, solid, cp, device)
        if components == 1 and any(float(v) != 0.0 for v in getattr(prm, "force", (0.0, 0.0, 0.0))):
            self.dev.set_body_force(*prm.force)
        self._geo = None
        self._steps = 0
        self._host_dirty = False
        self._host = None

    # reference accessors (solver.hpp:115-122)
    def dims(self) -> GridDims:
        return self._dims

    def params(self) -> CollisionParams:
        return self._prm

    def boundary(self) -> BoundarySpec:
        return self._spec

    def steps(self) -> int:
        return self._steps

    def geometry(self) -> NodeGeometry:
        if self._geo is None:
            self._geo = self.dev.geometry()
        return self._geo

    def _flush(self):
        if self._host_dirty:
            self._upload_all()
            self._host_dirty = False

    def fields(self):
        """Mutable host view: synchronised from the device, uploaded back
        before the next device operation (non-const Sim::fields())."""
        self._flush()
        self._host = self._download_all()
        self._host_dirty = True
        return self._host

    def view(self):
        """Read-only snapshot (const Sim::fields())."""
        self._flush()
        return self._download_all()

    def step(self):
        self._flush()
        self.dev.step(1)
        self._steps += 1

    def run(self, n: int):
        self._flush()
        self.dev.step(int(n))
        self._steps += int(n)

    def refresh_moments(self):
        self._flush()
        self.dev.phase("refresh_moments")

    def stability(self) -> StabilityReport:
        self._flush()
        return self.dev.stability()

    def plane_digests(self):
        self._flush()
        return self.dev.plane_digests()

    def close(self):
        self.dev.close()


class SingleFluidSim(_SimBase):
    """solver.hpp:70-132"""

    def __init__(self, lat, g: GridDims, prm: CollisionParams, spec: BoundarySpec, solid=None, dtype=np.float64,
                 device: int = 0):
        super().__init__(lat, g, prm, spec, solid, dtype, 1, None, device)

    def _download_all(self) -> FieldSet:
        d = self.dev
        return FieldSet(self._dims, self.lattice.q, self.lattice.dim, d.download_f(0), d.download_field("rho"),
                        d.download_field("mom").reshape(self.lattice.dim, -1),
                        d.download_field("pineq").reshape(self.lattice.npineq, -1))

    def _upload_all(self):
        s = self._host
        self.dev.upload_f(s.f)
        self.dev.upload_field("rho", s.rho)
        self.dev.upload_field("mom", s.mom)
        self.dev.upload_field("pineq", s.pineq)

    def totals(self):
        """Total mass and momentum over fluid nodes (device fp64 tree)."""
        self._flush()
        return self.dev.totals()


class TwoFluidSim(_SimBase):
    """solver.hpp:135-202"""

    def __init__(self, lat, g: GridDims, prm: CollisionParams, cp: ColorParams, spec: BoundarySpec, solid=None,
                 dtype=np.float64, device: int = 0):
        super().__init__(lat, g, prm, spec, solid, dtype, 2, cp, device)

    def colors(self) -> ColorParams:
        return self._cp

    def _download_all(self) -> TwoFluidFieldSet:
        d = self.dev
        L = self.lattice
        return TwoFluidFieldSet(self._dims, L.q, L.dim, d.download_f(0), d.download_f(1), d.download_field("rho_r"),
                                d.download_field("rho_b"), d.download_field("rho"),
                                d.download_field("mom").reshape(L.dim, -1),
                                d.download_field("pineq").reshape(L.npineq, -1), d.download_field("phi"),
                                d.download_field("gradphi").reshape(L.dim, -1), d.download_field("nci_flag"))

    def _upload_all(self):
        s = self._host
        d = self.dev
        d.upload_f(s.fr, 0)
        d.upload_f(s.fb, 1)
        for k in ("rho_r", "rho_b", "rho", "mom", "pineq", "phi", "gradphi", "nci_flag"):
            d.upload_field(k, getattr(s, k))

    def color_masses(self):
        self._flush()
        return self.dev.color_masses()


# ---------------------------------------------------------------------------
# free functions on host FieldSets (kernels.hpp / multicomponent.hpp API):
# upload, run the device phase, download. Not the hot path -- for tests and
# drivers that manipulate FieldSets directly, as the reference tests do.
# ---------------------------------------------------------------------------


def classify_nodes(lat, g: GridDims, spec: BoundarySpec, solid=None) -> NodeGeometry:
    """boundary.hpp:61-111 (device classify, bit-exact)."""
    d = DeviceSolver(lat, g, 1.0, spec, np.float32, 1, solid)
    try:
        return d.geometry()
    finally:
        d.close()


def _single_call(lat, s: FieldSet, spec, prm, solid, fn):
    d = DeviceSolver(lat, s.dims, prm.omega if prm else 1.0, spec or BoundarySpec(), s.f.dtype, 1, solid)
    try:
        d.upload_f(s.f)
        d.upload_field("rho", s.rho)
        d.upload_field("mom", s.mom)
        d.upload_field("pineq", s.pineq)
        fn(d)
        s.f[...] = d.download_f(0)
        s.rho[...] = d.download_field("rho")
        s.mom[...] = d.download_field("mom").reshape(s.mom.shape)
        s.pineq[...] = d.download_field("pineq").reshape(s.pineq.shape)
    finally:
        d.close()


def _solid_of(geo):
    return None if geo is None else geo.solid


def compute_moments(lat, s: FieldSet, geo: NodeGeometry | None = None):
    _single_call(lat, s, None, None, _solid_of(geo), lambda d: d.phase("compute_moments"))


def stream_collide_fused(lat, s: FieldSet, geo, spec: BoundarySpec, prm: CollisionParams):
    _single_call(lat, s, spec, prm, _solid_of(geo), lambda d: d.phase("stream_collide"))


def fused_step(lat, s: FieldSet, geo, spec: BoundarySpec, prm: CollisionParams, steps: int = 1):
    _single_call(lat, s, spec, prm, _solid_of(geo), lambda d: d.step(steps))


def reference_step(lat, s: FieldSet, geo, spec: BoundarySpec, prm: CollisionParams, steps: int = 1):
    _single_call(lat, s, spec, prm, _solid_of(geo), lambda d: d.phase("reference_step", int(steps)))


def stream_only(lat, s: FieldSet, geo, spec: BoundarySpec):
    _single_call(lat, s, spec, None, _solid_of(geo), lambda d: d.phase("stream_only"))


# ---------------------------------------------------------------------------
# census and digests (bench.hpp:24-109)
# ---------------------------------------------------------------------------


@dataclass
class KernelCost:
    flops: float
    bytes: float
    intensity: float


def count_kernel_cost(lat, elem_bytes: int) -> KernelCost:
    """bench.hpp:30-66, same counting rules (extends to D3Q27)."""
    L = lattice_of(lat)
    D = L.dim
    npi = D * (D + 1) // 2
    p1, p2 = 0.0, 12.0
    for c in L.c:
        nm = sum(1 for v in c if v != 0)
        pairs = sum(1 for ax in range(3) for bx in range(ax + 1, 3) if c[ax] != 0 and c[bx] != 0)
        p1 += 1 + 2 * nm + pairs
        p2 += 6 if nm == 0 else ((nm - 1) + 7) + ((nm + pairs - 1) + 3) + 2
    p1 += 1 + 3 * D + 2 * (npi - D)
    fl = p1 + p2
    by = 2.0 * (L.q + 1 + D + npi) * elem_bytes
    return KernelCost(fl, by, fl / by)


FNV_BASIS = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3


def fnv1a(data: bytes | np.ndarray, h: int = FNV_BASIS) -> int:
    """bench.hpp:83-91 (host, byte-serial; vectorised over nothing -- use for
    small states)."""
    b = np.ascontiguousarray(data).view(np.uint8).ravel() if isinstance(data, np.ndarray) else np.frombuffer(data, np.uint8)
    for v in b.tolist():
        h ^= v
        h = (h * FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
    return h


def chunked_plane_digest(arrays: np.ndarray, dims: GridDims, chunk: int = 16384) -> np.ndarray:
    """Host definition of the device plane digest (tslb_reduce.cu): per plane
    of each array, FNV-1a over the FNV-1a hashes of its 16 KiB chunks."""
    arrays = np.ascontiguousarray(arrays)
    q = arrays.shape[0]
    plane = dims.nx * dims.ny
    out = np.zeros((q, dims.nz), np.uint64)
    for a in range(q):
        for k in range(dims.nz):
            pb = arrays[a, k * plane:(k + 1) * plane].view(np.uint8)
            h = FNV_BASIS
            for c0 in range(0, pb.size, chunk):
                hc = fnv1a(pb[c0:c0 + chunk])
                h = fnv1a(np.array([hc], np.uint64), h)
            out[a, k] = h
    return out


def fold_digest(plane_digests: np.ndarray) -> int:
    """Global digest = FNV-1a over the plane digests in (species, a, z) order."""
    return fnv1a(np.ascontiguousarray(plane_digests, np.uint64).ravel())
