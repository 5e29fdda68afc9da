#!/bin/bash
mkdir -p gpurun_out
bash scripts/gpu_ab_libs.sh r2f_ab "msum cur2"
timeout 600 python bench.py --nccl-self --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2f_selfx.json 2> gpurun_out/r2f_selfx.err
timeout 1500 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_two.py -m gpu -q -p no:cacheprovider > gpurun_out/r2f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_pytest.log
