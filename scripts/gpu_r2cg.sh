#!/bin/bash
# two-fluid recolouring: one vs two nodes per thread (same box A/B) + the
# two-fluid GPU tests on the product library
set -u
mkdir -p gpurun_out
TAG=${1:-r2cg}
for i in 1 2; do
  for v in cgbase cg2 cg2npt1; do
    lib=ab/lib_$v.so; env=""
    [ $v = cg2npt1 ] && lib=ab/lib_cg2.so && env="TSLB_CG_NPT=1"
    env $env TSLB_LIB=$lib timeout 300 python bench.py --workload droplet-d3q19 --steps 10 --warmup 3 --no-e2e --no-cpu \
      2>>gpurun_out/${TAG}.err | sed "s/^/$v /" >> gpurun_out/${TAG}.txt
  done
done
timeout 1500 python -m pytest tests/test_gpu_two.py tests/test_gpu_slabs.py tests/test_gpu_configs.py tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
tail -3 gpurun_out/${TAG}_tests.log
python - <<PY
import json
for l in open("gpurun_out/${TAG}.txt"):
    n, j = l.split(" ", 1)
    try:
        d = json.loads(j); print(n, d["value"], d["ms_per_step"], d.get("clocks", {}).get("sm_mhz"))
    except Exception as e: print(n, "?", l[:200])
PY
