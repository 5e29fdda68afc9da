#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/v5_pytest.log 2>&1; echo rc=$? >> gpurun_out/v5_pytest.log
TSLB_STREAMCOLL=lean timeout 900 python -m pytest tests/test_gpu_single.py tests/test_gpu_golden.py tests/test_gpu_slabs.py -m gpu -x -q -p no:cacheprovider > gpurun_out/v5_pytest_lean.log 2>&1; echo rc=$? >> gpurun_out/v5_pytest_lean.log
bash scripts/gpu_sweep.sh v5
TSLB_STREAMCOLL=lean timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_streamcoll -s 2 -c 1 -o gpurun_out/v5_prof_lean_f64 python bench.py --steps 2 --warmup 1 --n 256 --no-e2e --no-cpu > gpurun_out/v5_ncu.log 2>&1
