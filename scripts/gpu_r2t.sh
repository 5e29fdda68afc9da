#!/bin/bash
# totals/stability reduction change: tests that read the reductions + default bench e2e
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_single.py tests/test_gpu_mstep.py tests/test_gpu_slabs.py -m gpu -x -q \
  -k "totals or stability or conserv or diagnos or refresh or init_state" > gpurun_out/r2t_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2t_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2t_bench.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu >> gpurun_out/r2t_bench.log 2>&1
tail -3 gpurun_out/r2t_tests.log; grep -o '"e2e".*' gpurun_out/r2t_bench.log | cut -c1-400
