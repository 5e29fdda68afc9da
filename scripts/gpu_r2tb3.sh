#!/bin/bash
# one-barrier TB: K sweep on the cavity, and the size sweep (where the persistent path should stop)
set -u
mkdir -p gpurun_out
rm -f gpurun_out/r2tb3.txt
bash scripts/gpu_ab_libs.sh r2tb3 "tbk4 tbk6 tbk8" --workload cavity-d2q9 --steps 2000 --warmup 64
python - <<PY
import json
for l in open("gpurun_out/r2tb3.txt"):
    n, j = l.split(" ", 1); d = json.loads(j); print(n, d["value"], d["ms_per_step"])
PY
TSLB_LIB=ab/lib_tbk4.so python tools/micro/tb2d_sizes.py > gpurun_out/r2tb3_sizes.txt 2>&1
cat gpurun_out/r2tb3_sizes.txt
