#!/bin/bash
# round-2 iteration: M-kernel tests + same-box A/B of library variants
# usage: gpu_r2_iter.sh TAG "variants" [pytest -k expr]
TAG=${1:-r2}
NAMES=${2:-"base new"}
K=${3:-""}
mkdir -p gpurun_out
(free -g; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv) > gpurun_out/${TAG}_env.txt 2>&1
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
bash scripts/gpu_ab_libs.sh ${TAG}_ab "$NAMES"
