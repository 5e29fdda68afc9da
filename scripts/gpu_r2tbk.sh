#!/bin/bash
# 2-D temporal blocking: passes per block K (build variants), cavity 256^2 and a 1024^2 TGV (persistent limit 2^20 nodes)
set -u
mkdir -p gpurun_out
bash scripts/gpu_ab_libs.sh r2tbk "tbk2 tbk4 tbk6 tbk8" --workload cavity-d2q9 --steps 2000 --warmup 64
python - <<PY
import json
for l in open("gpurun_out/r2tbk.txt"):
    n, j = l.split(" ", 1)
    try:
        d = json.loads(j); print(n, d["value"], d["ms_per_step"])
    except Exception as e: print(n, "?", l[:200])
PY
