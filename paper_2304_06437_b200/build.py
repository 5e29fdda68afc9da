"""In-tree build of libtslb_cuda.so (nvcc, sm_100a only).

Compiles every csrc/*.cu in parallel with
    -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false
(--fmad=false is part of the parity contract: no contracted multiply-adds,
so the kernels reproduce the reference's evaluation order bit for bit) and
links them with the static CUDA runtime. Rebuilds only stale objects.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
INC = os.path.join(os.path.dirname(PKG), "include")
LIB = os.path.join(PKG, "libtslb_cuda.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", *GENCODE, "-lineinfo", "--fmad=false",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", f"-I{INC}", "-Wno-deprecated-gpu-targets"]


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(INC, "tslb_cuda.h"))
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, obj, extra=()):
    cmd = [NVCC, *FLAGS, *extra, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def build(verbose: bool = False, out: str | None = None, defines: tuple = ()) -> str:
    """Build the product library (default), or -- with `defines` -- a
    measurement variant (-D flags) into `out` with its own object directory
    (same-box A/B runs load it through TSLB_LIB; the product .so is untouched)."""
    lib = out or LIB
    # (variant builds only: TSLB_NVCC_EXTRA adds raw nvcc flags)
    raw = os.environ.get("TSLB_NVCC_EXTRA", "").split() if out else []
    tag = "_".join([d.replace("=", "-") for d in defines] + [str(abs(hash(" ".join(raw))) % 10 ** 8)] * bool(raw))
    obj_dir = OBJ if not (defines or raw) else os.path.join(OBJ, "v_" + tag)
    extra = [f"-D{d}" for d in defines] + raw
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))
    hdrs = _headers()
    jobs = []
    objs = []
    for s in srcs:
        o = os.path.join(obj_dir, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if _stale(o, [s, *hdrs]):
            jobs.append((s, o))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            for o in ex.map(lambda so: _compile(*so, extra), jobs):
                if verbose:
                    print("compiled", o, file=sys.stderr)
    if jobs or _stale(lib, objs):
        os.makedirs(os.path.dirname(os.path.abspath(lib)), exist_ok=True)
        cmd = [NVCC, "-shared", *GENCODE, "-Wno-deprecated-gpu-targets", "-o", lib, *objs,
               "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib


if __name__ == "__main__":
    # python build.py [OUT.so -DNAME[=V] ...]: a measurement variant
    args = sys.argv[1:]
    if args:
        print(build(verbose=True, out=args[0], defines=tuple(a[2:] for a in args[1:] if a.startswith("-D"))))
    else:
        print(build(verbose=True))
