#!/bin/bash
# full GPU suite + default bench (e2e + cpu) + ncu evidence of the M kernel
TAG=${1:-s8}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,clocks.sm --format=csv > gpurun_out/${TAG}_env.txt 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --math f32 > gpurun_out/${TAG}_bench_m_f32.json 2> gpurun_out/${TAG}_bench_m_f32.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --schedule f1 > gpurun_out/${TAG}_bench_f1_f64.json 2> gpurun_out/${TAG}_bench_f1_f64.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --n 512 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mstep -s 3 -c 1 -o gpurun_out/${TAG}_prof_mstep_f64 python bench.py --steps 2 --warmup 3 --n 512 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu_m64.log 2>&1
