#!/bin/bash
# lazy-f M init: parity + full suite + default bench + D3Q27 1024^3 (M now fits)
TAG=${1:-s16}
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err
timeout 900 python bench.py --workload channel-d3q27 --steps 10 --warmup 3 > gpurun_out/${TAG}_channel1024.json 2> gpurun_out/${TAG}_channel1024.err
timeout 900 python bench.py --workload channel-d3q27 --steps 10 --warmup 3 --math f32 > gpurun_out/${TAG}_channel1024_f32.json 2> gpurun_out/${TAG}_channel1024_f32.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --math f32 > gpurun_out/${TAG}_bench_m_f32.json 2> gpurun_out/${TAG}_bench_m_f32.err
