#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_single.py tests/test_gpu_mstep.py -m gpu -q -p no:cacheprovider -k "init_state or init or lazy" > gpurun_out/r2g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2g_default.json 2> gpurun_out/r2g_default.err
