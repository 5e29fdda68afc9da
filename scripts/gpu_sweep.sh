#!/bin/bash
# stream-collide variant sweep at 1024^3 (device-timed bench lines)
TAG=${1:-sweep}
mkdir -p gpurun_out
for M in f64 f32; do
  for VX in 2 4; do
    TSLB_STREAMCOLL=vec TSLB_VX=$VX timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --math $M > gpurun_out/${TAG}_${M}_vec$VX.json 2>&1
  done
  TSLB_STREAMCOLL=lean timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --math $M > gpurun_out/${TAG}_${M}_lean.json 2>&1
  TSLB_STREAMCOLL=scalar timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --math $M > gpurun_out/${TAG}_${M}_scalar.json 2>&1
done
