#!/bin/bash
# BASELINE.json configs besides the headline, one bench line each
TAG=${1:-wl}
mkdir -p gpurun_out
timeout 600 python bench.py --workload droplet-d3q19 --steps 10 --warmup 3 > gpurun_out/${TAG}_droplet.json 2> gpurun_out/${TAG}_droplet.err
timeout 900 python bench.py --workload channel-d3q27 --steps 10 --warmup 3 > gpurun_out/${TAG}_channel1024.json 2> gpurun_out/${TAG}_channel1024.err
timeout 900 python bench.py --workload channel-d3q27 --steps 10 --warmup 3 --math f32 > gpurun_out/${TAG}_channel1024_f32.json 2> gpurun_out/${TAG}_channel1024_f32.err
timeout 600 python bench.py --workload cavity-d2q9 --steps 2000 --warmup 64 > gpurun_out/${TAG}_cavity.json 2> gpurun_out/${TAG}_cavity.err
timeout 600 python bench.py --n 512 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_tgv512.json 2> gpurun_out/${TAG}_tgv512.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --math f32 > gpurun_out/${TAG}_tgv1024_f32.json 2> gpurun_out/${TAG}_tgv1024_f32.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --schedule f1 > gpurun_out/${TAG}_tgv1024_f1.json 2> gpurun_out/${TAG}_tgv1024_f1.err
timeout 600 python bench.py --workload tgv-d2q9 --steps 20 --warmup 3 > gpurun_out/${TAG}_tgv2d.json 2> gpurun_out/${TAG}_tgv2d.err
timeout 600 python bench.py --workload porous-d3q19 --steps 20 --warmup 3 > gpurun_out/${TAG}_porous.json 2> gpurun_out/${TAG}_porous.err
