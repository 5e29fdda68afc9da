#!/bin/bash
# hoisted wall tests in k_mstep: D3Q27 channel A/B + mstep wall tests
set -u
mkdir -p gpurun_out
bash scripts/gpu_ab_libs.sh r2v_ch "base new" --workload channel-d3q27
timeout 1200 python -m pytest tests/test_gpu_mstep.py tests/test_gpu_configs.py -m gpu -x -q > gpurun_out/r2v_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2v_tests.log
tail -3 gpurun_out/r2v_tests.log
python - <<'PY'
import json
for l in open("gpurun_out/r2v_ch.txt"):
    n, j = l.split(" ", 1)
    try:
        d = json.loads(j); print(n, d["value"], d["ms_per_step"], d.get("clocks", {}).get("sm_mhz"))
    except Exception as e: print(n, "?", l[:200])
PY
