#!/bin/bash
# quick M-kernel iteration: parity + bench f64/f32 + ncu f32
TAG=${1:-s5}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mstep.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_mstep.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_mstep.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_bench_m_f64.json 2> gpurun_out/${TAG}_bench_m_f64.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --math f32 > gpurun_out/${TAG}_bench_m_f32.json 2> gpurun_out/${TAG}_bench_m_f32.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mstep -s 3 -c 1 -o gpurun_out/${TAG}_prof_mstep_f32 python bench.py --steps 2 --warmup 3 --n 512 --no-e2e --no-cpu --math f32 > gpurun_out/${TAG}_ncu_m32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mstep -s 3 -c 1 -o gpurun_out/${TAG}_prof_mstep_f64 python bench.py --steps 2 --warmup 3 --n 512 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_m64.log 2>&1
