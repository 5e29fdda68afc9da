#!/bin/bash
# same-box A/B of two-fluid recolouring-kernel register caps (ab/lib_mb*.so,
# built with -DTSLB_CG_MINB=N); droplet 512^3 device-only bench lines, then
# the two-fluid GPU tests on each capped variant
TAG=${1:-abtwo}
VARS=${2:-"mb1 mb5 mb6 mb8"}
TESTS=${3:-"mb5 mb6 mb8"}
mkdir -p gpurun_out
L=paper_2304_06437_b200/libtslb_cuda.so
cp $L ab/lib_orig.so
for i in 1 2; do
  for v in $VARS; do
    cp ab/lib_$v.so $L
    timeout 300 python bench.py --workload droplet-d3q19 --steps 20 --warmup 3 --no-e2e --no-cpu 2>>gpurun_out/${TAG}.err | sed "s/^/$v /" >> gpurun_out/${TAG}.txt
  done
done
for v in $TESTS; do
  cp ab/lib_$v.so $L
  timeout 600 python -m pytest tests/test_gpu_two.py -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_${v}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_${v}_pytest.log
done
cp ab/lib_orig.so $L
