#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_two.py tests/test_gpu_slabs.py tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -k "two or droplet or c4 or nci" > gpurun_out/r2p_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_pytest.log
bash scripts/gpu_ab_libs.sh r2p_dr "cur6 two2" --workload droplet-d3q19
bash scripts/gpu_ab_libs.sh r2p_ch "two2 ref" --workload channel-d3q27
