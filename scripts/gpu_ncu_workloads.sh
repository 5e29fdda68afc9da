#!/bin/bash
# one ncu --set full capture of the dominant kernel of each non-headline
# bench workload (feeds profiles/traffic.json: DRAM bytes per node per launch)
TAG=${1:-nw}
mkdir -p gpurun_out
N="--clock-control none --import-source on --set full"
B="--steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 900 ncu $N -k regex:k_mstep -s 3 -c 1 -o gpurun_out/${TAG}_d3q27_mstep python bench.py --workload channel-d3q27 --dims 512,512,512 $B > gpurun_out/${TAG}_ncu.log 2>&1
timeout 900 ncu $N -k regex:k_cg_streamcoll_box -s 3 -c 1 -o gpurun_out/${TAG}_droplet_scr python bench.py --workload droplet-d3q19 $B >> gpurun_out/${TAG}_ncu.log 2>&1
timeout 900 ncu $N -k regex:k_cg_moments -s 3 -c 1 -o gpurun_out/${TAG}_droplet_cgm python bench.py --workload droplet-d3q19 $B >> gpurun_out/${TAG}_ncu.log 2>&1
timeout 900 ncu $N -k regex:k_mstep2d -s 3 -c 1 -o gpurun_out/${TAG}_d2q9_mstep python bench.py --workload tgv-d2q9 $B >> gpurun_out/${TAG}_ncu.log 2>&1
timeout 900 ncu $N -k regex:k_mstep -s 3 -c 1 -o gpurun_out/${TAG}_porous_mstep python bench.py --workload porous-d3q19 $B >> gpurun_out/${TAG}_ncu.log 2>&1
# summarise on the box and drop the reports (gpurun copies back <= 64 MiB)
declare -A NODES=([d3q27_mstep]=134217728 [droplet_scr]=134217728 [droplet_cgm]=134217728 [d2q9_mstep]=16777216 [porous_mstep]=134217728)
for r in d3q27_mstep droplet_scr droplet_cgm d2q9_mstep porous_mstep; do
  f=gpurun_out/${TAG}_$r.ncu-rep
  [ -f $f ] || continue
  python tools/ncu_summary.py $f > gpurun_out/${TAG}_${r}_summary.txt 2>&1
  ncu -i $f --page source --csv --print-source=sass > /tmp/${TAG}_${r}_sass.csv 2>/dev/null
  python tools/sass_mix.py /tmp/${TAG}_${r}_sass.csv ${NODES[$r]} > gpurun_out/${TAG}_${r}_sass_mix.txt 2>&1
  rm -f $f
done
