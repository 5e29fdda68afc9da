import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TSLB_STREAMCOLL", "tma")
from oracle import oracle as O
from paper_2304_06437_b200 import tslb as T
dims = tuple(int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (256, 4, 4)))
dt = np.float32 if (len(sys.argv) < 5 or sys.argv[4] == "f32") else np.float64
f0 = O.random_state("d3q19", dims, 1, dt)
dev = T.DeviceSolver(T.D3Q19, T.GridDims(*dims), 1.1, T.BoundarySpec.all_periodic(), dt)
dev.upload_f(f0)
dev.step(1)
g = dev.download_f()
ref = f0.copy()
O.Oracle("port").single_run("d3q19", dims, 1.1, O.periodic(), ref, None, 1, 0)
print("bitwise equal:", np.array_equal(g.view(np.uint8), ref.view(np.uint8)), "maxdiff", float(np.abs(g - ref).max()))
