#!/bin/bash
# D3Q27 channel after the wall-test hoist: march unroll 2 (build variant) and planes per CTA (TSLB_LZ)
set -u
mkdir -p gpurun_out
bash scripts/gpu_ab_libs.sh r2d27 "base u2" --workload channel-d3q27 --steps 10
for lz in 64 256; do
  TSLB_LZ=$lz TSLB_LIB=ab/lib_base.so timeout 300 python bench.py --workload channel-d3q27 --steps 10 --warmup 3 --no-e2e --no-cpu 2>>gpurun_out/r2d27.err | sed "s/^/lz$lz /" >> gpurun_out/r2d27.txt
done
python - <<PY
import json
for l in open("gpurun_out/r2d27.txt"):
    n, j = l.split(" ", 1)
    try:
        d = json.loads(j); print(n, d["value"], d["ms_per_step"])
    except Exception as e: print(n, "?", l[:200])
PY
