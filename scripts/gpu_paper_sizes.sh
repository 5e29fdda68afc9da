#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --workload tgv-d2q9 --steps 50 --warmup 5 > gpurun_out/paper_d2q9_4096.json 2> gpurun_out/paper_d2q9_4096.err
timeout 600 python bench.py --workload tgv-d2q9 --steps 50 --warmup 5 --math f32 > gpurun_out/paper_d2q9_4096_f32.json 2>&1
timeout 600 python bench.py --n 256 --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/paper_d3q19_256.json 2>&1
timeout 600 python bench.py --workload droplet-d3q19 --n 256 --steps 50 --warmup 5 > gpurun_out/paper_droplet_256.json 2>&1
