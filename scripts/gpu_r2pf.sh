#!/bin/bash
# next-plane moments prefetch beside the reduction (TSLB_MSTEP_PF=1) vs base: A/B + M tests on the variant
set -u
mkdir -p gpurun_out
bash scripts/gpu_ab_libs.sh r2pf "base pf"
bash scripts/gpu_ab_libs.sh r2pf_f32 "base pf" --math f32
TSLB_LIB=ab/lib_pf.so timeout 1200 python -m pytest tests/test_gpu_mstep.py tests/test_gpu_slabs.py -m gpu -x -q > gpurun_out/r2pf_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2pf_tests.log
tail -3 gpurun_out/r2pf_tests.log
python - <<PY
import json
for f in ("gpurun_out/r2pf.txt", "gpurun_out/r2pf_f32.txt"):
    for l in open(f):
        n, j = l.split(" ", 1)
        try:
            d = json.loads(j); print(f[11:], n, d["value"], d["ms_per_step"], d.get("clocks", {}).get("sm_mhz"))
        except Exception as e: print(n, "?", l[:200])
PY
