#!/bin/bash
# body-force extension: parity + Poiseuille + channel bench; C++ drop-in tests
TAG=${1:-s17}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mstep.py tests/test_cpp_dropin.py -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --workload channel-d3q27 --steps 10 --warmup 3 > gpurun_out/${TAG}_channel1024.json 2> gpurun_out/${TAG}_channel1024.err
