#!/bin/bash
# seed-free moment sums: full GPU parity suite + device-only A/B bench lines
TAG=${1:-s27}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu >> gpurun_out/${TAG}_ab.jsonl 2>>gpurun_out/${TAG}_ab.err
done
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --math f32 >> gpurun_out/${TAG}_ab.jsonl 2>>gpurun_out/${TAG}_ab.err
timeout 300 python bench.py --workload tgv-d2q9 --steps 20 --warmup 3 --no-e2e --no-cpu >> gpurun_out/${TAG}_ab.jsonl 2>>gpurun_out/${TAG}_ab.err
timeout 600 python bench.py --workload channel-d3q27 --steps 10 --warmup 3 --no-e2e --no-cpu >> gpurun_out/${TAG}_ab.jsonl 2>>gpurun_out/${TAG}_ab.err
timeout 300 python bench.py --workload porous-d3q19 --steps 20 --warmup 3 --no-e2e --no-cpu >> gpurun_out/${TAG}_ab.jsonl 2>>gpurun_out/${TAG}_ab.err
