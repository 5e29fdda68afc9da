#!/bin/bash
# bench + ncu evidence (run after gpu_check.sh in the same gpurun call)
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --n 512 --no-e2e --no-cpu > gpurun_out/bench512.json 2> gpurun_out/bench512.err
timeout 900 python bench.py --steps 20 --warmup 3 --no-e2e > gpurun_out/bench1024.json 2> gpurun_out/bench1024.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --math f32 > gpurun_out/bench1024_f32math.json 2> gpurun_out/bench1024_f32math.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --n 256 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_streamcoll -s 2 -c 1 -o gpurun_out/prof_streamcoll python bench.py --steps 2 --warmup 1 --n 256 --no-e2e --no-cpu > gpurun_out/ncu_sc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_moments -s 2 -c 1 -o gpurun_out/prof_moments python bench.py --steps 2 --warmup 1 --n 256 --no-e2e --no-cpu > gpurun_out/ncu_mo.log 2>&1
