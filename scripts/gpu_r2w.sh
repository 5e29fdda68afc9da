#!/bin/bash
# HBM read:write mix probe + D3Q27 channel fp32 math line
set -u
mkdir -p gpurun_out
timeout 300 tools/micro/rw_mix > gpurun_out/r2w_rwmix.txt 2>&1
timeout 600 python bench.py --workload channel-d3q27 --steps 10 --warmup 3 --math f32 --no-cpu --no-e2e > gpurun_out/r2w_channel_f32.json 2> gpurun_out/r2w.err
cat gpurun_out/r2w_rwmix.txt; cut -c1-200 gpurun_out/r2w_channel_f32.json
