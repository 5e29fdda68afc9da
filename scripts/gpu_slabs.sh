#!/bin/bash
# z-slab decomposition (local transport + NCCL self-exchange), all species
TAG=${1:-slabs}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_two.py -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
