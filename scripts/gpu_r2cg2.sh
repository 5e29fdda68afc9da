#!/bin/bash
# two-fluid recolouring, two nodes per thread under register caps (same box A/B)
set -u
mkdir -p gpurun_out
bash scripts/gpu_ab_libs.sh r2cg2 "cgbase cg2m5 cg2m6 cg2m8" --workload droplet-d3q19
python - <<PY
import json
for l in open("gpurun_out/r2cg2.txt"):
    n, j = l.split(" ", 1)
    try:
        d = json.loads(j); print(n, d["value"], d["ms_per_step"], d.get("clocks", {}).get("sm_mhz"))
    except Exception as e: print(n, "?", l[:200])
PY
