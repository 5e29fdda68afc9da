#!/bin/bash
# tile rows TY=10 (20 warps per SM at <= 96 registers) vs TY=8: same-box A/B, fp64 and fp32 node math,
# and the M tests on the variant library
set -u
mkdir -p gpurun_out
bash scripts/gpu_ab_libs.sh r2ty "base ty10"
bash scripts/gpu_ab_libs.sh r2ty_f32 "base ty10" --math f32
TSLB_LIB=ab/lib_ty10.so timeout 1200 python -m pytest tests/test_gpu_mstep.py -m gpu -x -q > gpurun_out/r2ty_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2ty_tests.log
tail -3 gpurun_out/r2ty_tests.log
python - <<PY
import json
for f in ("gpurun_out/r2ty.txt", "gpurun_out/r2ty_f32.txt"):
    for l in open(f):
        n, j = l.split(" ", 1)
        try:
            d = json.loads(j); print(f[11:], n, d["value"], d["ms_per_step"], d.get("clocks", {}).get("sm_mhz"))
        except Exception as e: print(n, "?", l[:200])
PY
