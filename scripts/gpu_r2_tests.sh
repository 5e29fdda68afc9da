#!/bin/bash
# round-2 test pass: selected -m gpu files (default: all) with durations
TAG=${1:-r2t}
shift
mkdir -p gpurun_out
(free -g; nproc) > gpurun_out/${TAG}_env.txt 2>&1
timeout 3000 python -m pytest ${@:-tests} -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
