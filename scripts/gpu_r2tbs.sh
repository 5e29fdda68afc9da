#!/bin/bash
# 2-D temporal blocking tile shapes (build variants), cavity 256^2, same box
set -u
mkdir -p gpurun_out
bash scripts/gpu_ab_libs.sh r2tbs "s3216 s16_16_256 s32_8_256 s64_16_512 s32_32_1024" --workload cavity-d2q9 --steps 2000 --warmup 64
python - <<PY
import json
for l in open("gpurun_out/r2tbs.txt"):
    n, j = l.split(" ", 1)
    try:
        d = json.loads(j); print(n, d["value"], d["ms_per_step"])
    except Exception as e: print(n, "?", l[:200])
PY
