#!/bin/bash
# peer-memory (CUDA IPC) slab transport: tests (one process, 2-3 processes on this GPU)
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ipc.py -m gpu -x -q > gpurun_out/r2ipc_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2ipc_tests.log
tail -40 gpurun_out/r2ipc_tests.log
