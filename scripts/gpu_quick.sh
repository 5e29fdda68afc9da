#!/bin/bash
# quick GPU iteration: the -m gpu tests selected by -k "$1"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "${1:-slice}" > gpurun_out/quick_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/quick_pytest.log
