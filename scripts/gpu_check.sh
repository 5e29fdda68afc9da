#!/bin/bash
# One gpurun session: environment facts, smoke, GPU parity tests, bench, ncu.
# Usage (from the repo root): bash scripts/gpu_check.sh [quick]
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,clocks.sm --format=csv > gpurun_out/env.txt 2>&1
free -g >> gpurun_out/env.txt; nproc >> gpurun_out/env.txt; lscpu | head -20 >> gpurun_out/env.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
