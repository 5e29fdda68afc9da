#!/bin/bash
mkdir -p gpurun_out
for R in 8 12 16 24; do
TSLB_ROWS2D=$R timeout 300 python bench.py --workload tgv-d2q9 --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/rows_$R.json 2>&1
done
