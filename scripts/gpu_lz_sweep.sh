#!/bin/bash
# planes marched per CTA (TSLB_LZ) for the 3-D M kernel, headline workload
TAG=${1:-lz}
mkdir -p gpurun_out
for i in 1 2; do
  for Z in 32 64 128 256 512; do
    TSLB_LZ=$Z timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>>gpurun_out/${TAG}.err | sed "s/^/LZ$Z /" >> gpurun_out/${TAG}.txt
  done
done
for Z in 64 128 256; do
  TSLB_LZ=$Z timeout 300 python bench.py --workload channel-d3q27 --steps 10 --warmup 3 --no-e2e --no-cpu 2>>gpurun_out/${TAG}.err | sed "s/^/q27LZ$Z /" >> gpurun_out/${TAG}.txt
done
