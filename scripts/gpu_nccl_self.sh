#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_mstep.py -m gpu -q -p no:cacheprovider -k "nccl or full_size" > gpurun_out/s18_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s18_pytest.log
