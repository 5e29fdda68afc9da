#!/bin/bash
# two-fluid slab step with the population exchange overlapped (lib_new) vs
# the serial order (lib_old): NCCL self-exchange probe of the droplet, then
# the slab / two-fluid GPU tests on the new library
TAG=${1:-tso}
mkdir -p gpurun_out
L=paper_2304_06437_b200/libtslb_cuda.so
for i in 1 2; do
  for v in old new; do
    cp ab/lib_$v.so $L
    timeout 300 python bench.py --workload droplet-d3q19 --nccl-self --steps 20 --warmup 3 --no-e2e --no-cpu 2>>gpurun_out/${TAG}.err | sed "s/^/$v /" >> gpurun_out/${TAG}.txt
  done
done
cp ab/lib_new.so $L
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_two.py -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
