#!/bin/bash
# M-schedule and slab GPU tests + the default bench line (after an M change)
TAG=${1:-mc}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_mstep.py tests/test_gpu_slabs.py tests/test_gpu_golden.py -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_bench_$i.json 2>> gpurun_out/${TAG}.err
done
timeout 600 python bench.py --nccl-self --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_selfx.json 2>> gpurun_out/${TAG}.err
