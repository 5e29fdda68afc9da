#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_mstep.py tests/test_gpu_single.py -m gpu -q -p no:cacheprovider > gpurun_out/r2q_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_pytest.log
bash scripts/gpu_ab_libs.sh r2q_tg "cur7 lvl"
bash scripts/gpu_ab_libs.sh r2q_ch "cur7 lvl" --workload channel-d3q27
