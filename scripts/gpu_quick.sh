#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_single.py -m gpu -q -p no:cacheprovider -k "${1:-slice}" > gpurun_out/slice_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/slice_pytest.log
