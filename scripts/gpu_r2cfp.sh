#!/bin/bash
# ncu --set full of the one-pass two-fluid kernel (droplet 512^3), summarised on the box
set -u
TAG=r2cfp
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_fused -s 2 -c 1 -o gpurun_out/${TAG}_droplet_fused \
  python bench.py --workload droplet-d3q19 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}_droplet_fused.ncu-rep --page source --csv --print-source=sass > gpurun_out/${TAG}_droplet_fused_sass.csv 2>/dev/null
python tools/collect_r2.py ${TAG} r02 gpurun_out/${TAG}_profiles > gpurun_out/${TAG}_collect.log 2>&1
rm -f gpurun_out/${TAG}_*.ncu-rep gpurun_out/${TAG}_*_sass.csv
head -60 gpurun_out/${TAG}_profiles/r02_droplet_fused_ncu_full.txt
