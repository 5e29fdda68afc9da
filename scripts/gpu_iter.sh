#!/bin/bash
# Iteration loop on the GPU: parity tests, bench variants, ncu of the top kernel.
# usage: bash scripts/gpu_iter.sh <tag> [pytest-args...]
TAG=${1:-iter}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_env.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider "$@" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for M in f64 f32; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --math $M > gpurun_out/${TAG}_bench_${M}.json 2> gpurun_out/${TAG}_bench_${M}.err
done
TSLB_STREAMCOLL=scalar timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_bench_scalar.json 2> gpurun_out/${TAG}_bench_scalar.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 1 --n 512 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_streamcoll -s 2 -c 1 -o gpurun_out/${TAG}_prof_streamcoll python bench.py --steps 2 --warmup 1 --n 256 --no-e2e --no-cpu > gpurun_out/${TAG}_ncu.log 2>&1
