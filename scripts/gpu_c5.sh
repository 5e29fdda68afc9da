#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --dims 2048,1024,1024 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/c5_one_gpu.json 2> gpurun_out/c5_one_gpu.err
timeout 900 python bench.py --dims 2048,1024,512 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/c5_half.json 2> gpurun_out/c5_half.err
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/c5_one_gpu.err
