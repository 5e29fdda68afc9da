#!/bin/bash
# same-box A/B of prebuilt library variants in ab/: lib_base.so, lib_new.so,
# lib_c.so (variant C runs with TSLB_MSTEP_RD=0); bench lines device-only
TAG=${1:-ab}
mkdir -p gpurun_out
L=paper_2304_06437_b200/libtslb_cuda.so
run() {  # variant env-prefix extra-args
  cp ab/lib_$1.so $L
  env $2 timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu $3 2>>gpurun_out/${TAG}.err | sed "s/^/$1 /" >> gpurun_out/${TAG}.txt
}
for i in 1 2; do
  run base "X=1" ""
  run new "X=1" ""
  run c "TSLB_MSTEP_RD=0" ""
done
run base "X=1" "--workload channel-d3q27"
run new "X=1" "--workload channel-d3q27"
run base "X=1" "--workload tgv-d2q9"
run new "X=1" "--workload tgv-d2q9"
cp ab/lib_c.so $L
TSLB_MSTEP_RD=0 timeout 900 python -m pytest tests/test_gpu_mstep.py -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_c_pytest.log
cp ab/lib_new.so $L
