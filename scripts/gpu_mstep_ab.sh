#!/bin/bash
# ring-variant A/B: parity (default + forced RD=1), bench f64 RD1 vs RD0, f32
TAG=${1:-s9}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mstep.py tests/test_gpu_slabs.py -m gpu -x -q -p no:cacheprovider -k "mstep" > gpurun_out/${TAG}_pytest_mstep.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_mstep.log
TSLB_MSTEP_RD=1 timeout 900 python -m pytest tests/test_gpu_mstep.py -m gpu -x -q -p no:cacheprovider -k "float32 or f32" > gpurun_out/${TAG}_pytest_mstep_rd1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_mstep_rd1.log
for R in 1 0; do
TSLB_MSTEP_RD=$R timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_bench_f64_rd$R.json 2>&1
done
TSLB_MSTEP_RD=1 timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --math f32 > gpurun_out/${TAG}_bench_f32_rd1.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mstep -s 3 -c 1 -o gpurun_out/${TAG}_prof_mstep_f64 python bench.py --steps 2 --warmup 3 --n 512 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_m64.log 2>&1
