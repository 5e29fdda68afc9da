#!/bin/bash
# 2-D temporal blocking: parity tests, then the cavity bench (TB vs per-pass persistent)
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_mstep.py -m gpu -x -q -k "temporal_blocking or persist" > gpurun_out/r2tb_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2tb_tests.log
timeout 600 python -m pytest tests/test_gpu_single.py -m gpu -x -q -k "cavity_c1" >> gpurun_out/r2tb_tests.log 2>&1
echo "c1 rc=$?" >> gpurun_out/r2tb_tests.log
for i in 1 2; do
  timeout 300 python bench.py --workload cavity-d2q9 --steps 2000 --warmup 64 --no-cpu > gpurun_out/r2tb_cav_tb$i.json 2>>gpurun_out/r2tb.err
  TSLB_TB2D=0 timeout 300 python bench.py --workload cavity-d2q9 --steps 2000 --warmup 64 --no-cpu > gpurun_out/r2tb_cav_pp$i.json 2>>gpurun_out/r2tb.err
done
tail -6 gpurun_out/r2tb_tests.log
for f in gpurun_out/r2tb_cav_*.json; do echo $f; cut -c1-160 $f; done
