#!/bin/bash
# streamcoll variant sweep at 1024^3 (device-timed bench lines)
TAG=${1:-sweep}
mkdir -p gpurun_out
for VX in 1 2 4; do
  TSLB_VX=$VX timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_f64_vx$VX.json 2>&1
  TSLB_VX=$VX timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --math f32 > gpurun_out/${TAG}_f32_vx$VX.json 2>&1
done
TSLB_STREAMCOLL=scalar timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_f64_scalar.json 2>&1
