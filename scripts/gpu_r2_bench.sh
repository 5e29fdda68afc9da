#!/bin/bash
# round-2 bench pass: default line, slab probe, C5 on one GPU, reference arm (whole workload)
TAG=${1:-r2bench}
mkdir -p gpurun_out
B="--no-e2e --no-cpu"
timeout 600 python bench.py --nccl-self --steps 20 --warmup 3 $B > gpurun_out/${TAG}_selfx.json 2> gpurun_out/${TAG}_selfx.err
TSLB_LZB=32 timeout 600 python bench.py --nccl-self --steps 20 --warmup 3 $B > gpurun_out/${TAG}_selfx_lzb32.json 2>> gpurun_out/${TAG}_selfx.err
timeout 900 python bench.py --workload tgv-c5 --steps 10 --warmup 3 $B > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_default.json 2> gpurun_out/${TAG}_default.err
