#!/bin/bash
# two-fluid kernels: x nodes per block (128 / 256 / 512), droplet 512^3, same box
set -u
mkdir -p gpurun_out
bash scripts/gpu_ab_libs.sh r2bx "bx128 bx256 bx512" --workload droplet-d3q19 --steps 10
python - <<PY
import json
for l in open("gpurun_out/r2bx.txt"):
    n, j = l.split(" ", 1)
    try:
        d = json.loads(j); print(n, d["value"], d["ms_per_step"], d["roofline"]["kernel_ms_per_step"])
    except Exception as e: print(n, "?", l[:200])
PY
