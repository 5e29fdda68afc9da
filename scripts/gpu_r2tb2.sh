#!/bin/bash
# 2-D temporal blocking with one barrier per pass (gather fused with the next collide): tests + cavity A/B
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mstep.py tests/test_gpu_single.py -m gpu -x -q -k "temporal or persist or cavity or d2q9" > gpurun_out/r2tb2_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2tb2_tests.log
tail -3 gpurun_out/r2tb2_tests.log
rm -f gpurun_out/r2tb2.txt
bash scripts/gpu_ab_libs.sh r2tb2 "tbold tbnew" --workload cavity-d2q9 --steps 2000 --warmup 64
python - <<PY
import json
for l in open("gpurun_out/r2tb2.txt"):
    n, j = l.split(" ", 1); d = json.loads(j); print(n, d["value"], d["ms_per_step"])
PY
python tools/micro/tb2d_sizes.py 2>&1 | head -6
