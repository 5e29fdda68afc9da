#!/bin/bash
# Session-2 validation: smoke, full GPU parity suite, bench lines (default,
# f32 math, TMA variants), ncu launch list + full captures of both kernels.
TAG=${1:-s2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,clocks.sm --format=csv > gpurun_out/${TAG}_env.txt 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
for M in f64 f32; do
  for V in vec tma; do
    TSLB_STREAMCOLL=$V timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --math $M > gpurun_out/${TAG}_${M}_${V}.json 2>&1
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --n 512 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_streamcoll -s 3 -c 1 -o gpurun_out/${TAG}_prof_streamcoll python bench.py --steps 2 --warmup 3 --n 512 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_sc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_moments -s 3 -c 1 -o gpurun_out/${TAG}_prof_moments python bench.py --steps 2 --warmup 3 --n 512 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_mo.log 2>&1
