#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_two.py tests/test_gpu_slabs.py tests/test_gpu_golden.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2j_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_pytest.log
bash scripts/gpu_ab_libs.sh r2j_ab "cur3 two" --workload droplet-d3q19
