#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_streamcoll_box -s 2 -c 1 -o gpurun_out/tw_prof python bench.py --workload droplet-d3q19 --n 256 --steps 2 --warmup 2 > gpurun_out/tw_ncu.log 2>&1
