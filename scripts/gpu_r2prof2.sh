#!/bin/bash
# ncu --set full: the 2-D temporally blocked cavity launch (200 passes) and the colour-moments kernel
set -u
TAG=r2p2
mkdir -p gpurun_out
N="--set full --clock-control none --import-source on"
timeout 900 ncu $N -k regex:k_mstep2d_tb -c 1 -o gpurun_out/${TAG}_cavity_tb \
  python bench.py --workload cavity-d2q9 --steps 200 --warmup 64 --no-e2e --no-cpu > gpurun_out/${TAG}_cav.log 2>&1
timeout 900 ncu $N -k regex:k_cg_moments -s 2 -c 1 -o gpurun_out/${TAG}_droplet_cgm \
  python bench.py --workload droplet-d3q19 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_cgm.log 2>&1
for n in cavity_tb droplet_cgm; do
  ncu -i gpurun_out/${TAG}_$n.ncu-rep --page source --csv --print-source=sass > gpurun_out/${TAG}_${n}_sass.csv 2>/dev/null
done
python tools/collect_r2.py ${TAG} r02 gpurun_out/${TAG}_profiles > gpurun_out/${TAG}_collect.log 2>&1
rm -f gpurun_out/${TAG}_*.ncu-rep gpurun_out/${TAG}_*_sass.csv
for n in cavity_tb droplet_cgm; do head -24 gpurun_out/${TAG}_profiles/r02_${n}_ncu_full.txt; done
