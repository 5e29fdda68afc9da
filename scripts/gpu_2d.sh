#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s23_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s23_pytest.log
timeout 600 python bench.py --workload tgv-d2q9 --steps 50 --warmup 5 > gpurun_out/s23_d2q9_4096.json 2>&1
timeout 600 python bench.py --workload tgv-d2q9 --steps 50 --warmup 5 --math f32 > gpurun_out/s23_d2q9_4096_f32.json 2>&1
timeout 600 python bench.py --workload cavity-d2q9 --steps 2000 --warmup 64 > gpurun_out/s23_cavity.json 2>&1
timeout 600 python bench.py --workload cavity-d2q9 --steps 2000 --warmup 64 --schedule f1 > gpurun_out/s23_cavity_f1.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mstep2d -s 3 -c 1 -o gpurun_out/s23_prof_m2d python bench.py --workload tgv-d2q9 --steps 2 --warmup 3 > gpurun_out/s23_ncu.log 2>&1
