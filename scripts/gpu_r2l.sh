#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_mstep.py tests/test_gpu_single.py tests/test_gpu_slabs.py tests/test_gpu_golden.py -m gpu -q -p no:cacheprovider > gpurun_out/r2l_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_pytest.log
bash scripts/gpu_ab_libs.sh r2l_ab "u2 f32f"
bash scripts/gpu_ab_libs.sh r2l_ab32 "u2 f32f" --math f32
