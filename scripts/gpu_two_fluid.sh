#!/bin/bash
# two-fluid box kernels: parity + droplet bench + ncu of the recolouring kernel
TAG=${1:-s12}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_two.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_two.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_two.log
timeout 600 python bench.py --workload droplet-d3q19 --steps 10 --warmup 3 > gpurun_out/${TAG}_droplet.json 2> gpurun_out/${TAG}_droplet.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg -s 6 -c 3 -o gpurun_out/${TAG}_prof_two python bench.py --workload droplet-d3q19 --n 256 --steps 2 --warmup 2 > gpurun_out/${TAG}_ncu_two.log 2>&1
