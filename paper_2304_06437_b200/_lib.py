"""ctypes binding of the C-ABI in include/tslb_cuda.h.

The product path has exactly one implementation: libtslb_cuda.so (sm_100a).
If the library is missing or no CUDA device is visible, every entry point
raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libtslb_cuda.so")

# include/tslb_cuda.h enums
D2Q9, D3Q19, D3Q27 = 0, 1, 2
F64, F32 = 0, 1
FACE_PERIODIC, FACE_WALL, FACE_MOVING = 0, 1, 2
MATH_F64, MATH_F32 = 0, 1
FIELD = dict(rho=0, mom=1, pineq=2, rho_r=3, rho_b=4, phi=5, gradphi=6, nci_flag=7, solid=8, slow_mask=9)
INIT = dict(rest=0, shear=1, taylor_green=2, droplet=3)
KCLASS = ["moments", "streamcoll", "cg_moments", "cg_gradient", "cg_streamcoll", "exchange", "mstep"]
SCHED_F1, SCHED_M = 0, 1
STORE_NATIVE, STORE_F16 = 0, 1


class TslbCudaError(RuntimeError):
    """Raised for any nonzero status of the C-ABI."""


class InvalidArgument(TslbCudaError, ValueError):
    """TSLB_EINVAL -- the reference's std::invalid_argument."""


_lib = None


def load(path: str | None = None) -> C.CDLL:
    """Load (once) and type the shared library. Raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    # TSLB_LIB: a measurement variant (same-box A/B runs, scripts/gpu_ab_libs.sh)
    p = path or os.environ.get("TSLB_LIB") or LIB_PATH
    if not os.path.exists(p):
        raise TslbCudaError(
            f"{p} is missing: build it with `python -m paper_2304_06437_b200.build` "
            "(there is no CPU fallback for the product path)")
    lib = C.CDLL(p)
    vp, i, d, l = C.c_void_p, C.c_int, C.c_double, C.c_long
    H = C.c_void_p
    sig = {
        "tslb_cuda_abi_version": ([], i),
        "tslb_cuda_last_error": ([], C.c_char_p),
        "tslb_cuda_device_count": ([vp], i),
        "tslb_cuda_create": ([i, i, i, i, i, i, d, vp, vp, vp, vp, vp, i, vp], i),
        "tslb_cuda_create_slab": ([i, i, i, i, i, i, i, i, d, vp, vp, vp, vp, vp, i, vp], i),
        "tslb_cuda_destroy": ([H], i),
        "tslb_cuda_set_math": ([H, i], i),
        "tslb_cuda_set_schedule": ([H, i], i),
        "tslb_cuda_get_schedule": ([H, vp], i),
        "tslb_cuda_set_body_force": ([H, vp], i),
        "tslb_cuda_download_slice": ([H, i, i, i, vp], i),
        "tslb_cuda_describe": ([H, vp, vp], i),
        "tslb_cuda_memory_bytes": ([H, vp], i),
        "tslb_cuda_upload_f": ([H, i, vp], i),
        "tslb_cuda_download_f": ([H, i, vp], i),
        "tslb_cuda_upload_field": ([H, i, vp], i),
        "tslb_cuda_download_field": ([H, i, vp], i),
        "tslb_cuda_download_geometry": ([H, vp, vp, vp], i),
        "tslb_cuda_init_analytic": ([H, i, d, d], i),
        "tslb_cuda_init_state": ([H, vp], i),
        "tslb_cuda_init_equilibrium": ([H, vp], i),
        "tslb_cuda_set_moment_storage": ([H, i], i),
        "tslb_cuda_step": ([H, l], i),
        "tslb_cuda_step_async": ([H, l], i),
        "tslb_cuda_synchronize": ([H], i),
        "tslb_cuda_steps_done": ([H, vp], i),
        "tslb_cuda_time_steps": ([H, l, vp], i),
        "tslb_cuda_compute_moments": ([H], i),
        "tslb_cuda_stream_collide": ([H], i),
        "tslb_cuda_reference_step": ([H, l], i),
        "tslb_cuda_stream_only": ([H], i),
        "tslb_cuda_color_moments": ([H], i),
        "tslb_cuda_gradient_and_nci": ([H], i),
        "tslb_cuda_prepare_stress": ([H], i),
        "tslb_cuda_stream_collide_recolor": ([H], i),
        "tslb_cuda_refresh_moments": ([H], i),
        "tslb_cuda_totals": ([H, vp, vp], i),
        "tslb_cuda_stability": ([H, vp, vp, vp, vp, vp], i),
        "tslb_cuda_color_masses": ([H, vp, vp], i),
        "tslb_cuda_plane_digests": ([H, vp], i),
        "tslb_cuda_profile": ([H, i], i),
        "tslb_cuda_profile_read": ([H, vp, vp], i),
        "tslb_cuda_launch_count": ([H, vp], i),
        "tslb_cuda_nccl_unique_id": ([vp], i),
        "tslb_cuda_attach_nccl": ([H, vp, i, i], i),
        "tslb_cuda_link_local": ([vp, i], i),
        "tslb_cuda_group_step": ([vp, i, l], i),
        "tslb_cuda_ipc_handle": ([H, vp], i),
        "tslb_cuda_attach_ipc": ([H, vp, vp], i),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.tslb_cuda_abi_version() != 3:
        raise TslbCudaError("libtslb_cuda.so ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().tslb_cuda_last_error().decode()
        if rc == 1:
            raise InvalidArgument(msg)
        raise TslbCudaError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def header_symbols(header: str | None = None) -> list[str]:
    import re
    h = header or os.path.join(os.path.dirname(PKG), "include", "tslb_cuda.h")
    txt = open(h).read()
    return sorted(set(re.findall(r"\b(tslb_cuda_[a-z0-9_]+)\s*\(", txt)))
