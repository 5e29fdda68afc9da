#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/v4_pytest.log 2>&1; echo rc=$? >> gpurun_out/v4_pytest.log
bash scripts/gpu_sweep.sh v4
TSLB_VX=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_streamcoll -s 2 -c 1 -o gpurun_out/v4_prof_sc_f64_vx2 python bench.py --steps 2 --warmup 1 --n 256 --no-e2e --no-cpu > gpurun_out/v4_ncu.log 2>&1
