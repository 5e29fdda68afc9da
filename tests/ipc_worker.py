"""One rank of a multi-process z-slab run over the peer-memory transport
(tslb_cuda_ipc_handle / tslb_cuda_attach_ipc), for tests/test_gpu_ipc.py:
every rank is its own process, so the CUDA IPC mapping, the cross-process
flag words and the parity double buffering are exercised exactly as with one
process per GPU (here all ranks share one device).

    python tests/ipc_worker.py RANK PARTS OUTDIR LAT NX NY NZ DTYPE STEPS MID FACES
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from oracle import oracle as O  # noqa: E402
from paper_2304_06437_b200 import tslb as T  # noqa: E402

from helpers import spec_of, zwalls_3d  # noqa: E402

FACES = {"periodic": O.periodic, "zwalls": zwalls_3d}


def split(nz, parts):
    return [(nz * p // parts, nz * (p + 1) // parts - nz * p // parts) for p in range(parts)]


def wait_for(path, timeout=120.0):
    t0 = time.time()
    while not os.path.exists(path):
        if time.time() - t0 > timeout:
            raise TimeoutError(path)
        time.sleep(0.02)


def main():
    rank, parts, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    lat = sys.argv[4]
    dims = tuple(int(v) for v in sys.argv[5:8])
    dtype = np.float32 if sys.argv[8] == "f32" else np.float64
    steps, mid = int(sys.argv[9]), int(sys.argv[10])
    faces = FACES[sys.argv[11]]()
    f0 = O.random_state(lat, dims, 91, dtype)
    plane = dims[0] * dims[1]
    z0, nzl = split(dims[2], parts)[rank]
    sv = T.DeviceSolver(lat, T.GridDims(*dims), 1.25, spec_of(faces), dtype, 1, None, slab=(z0, nzl))
    try:
        assert sv.schedule == "m"
        sv.upload_f(np.ascontiguousarray(f0[:, z0 * plane:(z0 + nzl) * plane]))
        # handles over the file system (any host channel does)
        tmp = os.path.join(out, f"h{rank}.tmp")
        with open(tmp, "wb") as fh:
            fh.write(sv.ipc_handle())
        os.replace(tmp, os.path.join(out, f"h{rank}.bin"))
        hs = []
        for r in range(parts):
            wait_for(os.path.join(out, f"h{r}.bin"))
            with open(os.path.join(out, f"h{r}.bin"), "rb") as fh:
                hs.append(fh.read())
        periodic_z = sys.argv[11] == "periodic"
        below = hs[(rank - 1) % parts] if (rank > 0 or periodic_z) else None
        above = hs[(rank + 1) % parts] if (rank < parts - 1 or periodic_z) else None
        sv.attach_ipc(below, above)
        sv.step(mid)
        f_mid = sv.download_f()  # f materialised from the ghost moments mid-run
        sv.step(steps - mid)
        rho = sv.download_field("rho")
        mom = sv.download_field("mom").reshape(3, -1)
        pin = sv.download_field("pineq").reshape(6, -1)
        f = sv.download_f()
        np.savez(os.path.join(out, f"out{rank}.npz"), f=f, f_mid=f_mid, m=np.concatenate([rho[None], mom, pin]))
        # the neighbours still copy into this rank's block until their last
        # step is done: free it only after every rank has finished
        open(os.path.join(out, f"done{rank}"), "w").close()
        for r in range(parts):
            wait_for(os.path.join(out, f"done{r}"))
    finally:
        sv.close()


if __name__ == "__main__":
    main()
