#!/bin/bash
# planes per CTA for the fp32-math M kernel (opt-in path)
TAG=${1:-lzf}
mkdir -p gpurun_out
for i in 1 2 3; do
  for Z in 64 128; do
    TSLB_LZ=$Z timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --math f32 2>>gpurun_out/${TAG}.err | sed "s/^/LZ$Z /" >> gpurun_out/${TAG}.txt
  done
done
