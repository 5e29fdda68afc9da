#!/bin/bash
# Same-box A/B of prebuilt library variants ab/lib_<name>.so (built with
# `python paper_2304_06437_b200/build.py ab/lib_<name>.so -DFLAG ...`), loaded
# through TSLB_LIB -- the product libtslb_cuda.so is never replaced.
# usage: gpu_ab_libs.sh TAG "name1 name2 ..." [bench args] ; bench lines device-only
TAG=${1:-ab}
NAMES=${2:-"base new"}
shift 2
mkdir -p gpurun_out
for i in 1 2; do
  for n in $NAMES; do
    TSLB_LIB=ab/lib_$n.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu "$@" \
      2>>gpurun_out/${TAG}.err | sed "s/^/$n /" >> gpurun_out/${TAG}.txt
  done
done
