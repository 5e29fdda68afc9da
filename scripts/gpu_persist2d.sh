#!/bin/bash
# persistent 2-D M kernel: GPU tests of the M schedule, then the cavity and
# the 4096^2 TGV bench lines with and without it
TAG=${1:-p2d}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mstep.py -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for i in 1 2; do
  for p in 1 0; do
    TSLB_PERSIST=$p timeout 300 python bench.py --workload cavity-d2q9 --steps 2000 --warmup 64 --no-e2e --no-cpu 2>>gpurun_out/${TAG}.err | sed "s/^/cavity P$p /" >> gpurun_out/${TAG}.txt
  done
done
TSLB_PERSIST=1 timeout 300 python bench.py --workload tgv-d2q9 --steps 20 --warmup 3 --no-e2e --no-cpu 2>>gpurun_out/${TAG}.err | sed "s/^/tgv2d P1 /" >> gpurun_out/${TAG}.txt
timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
