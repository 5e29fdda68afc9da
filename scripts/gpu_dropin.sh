#!/bin/bash
# the reference's unit suites + acceptance gate on the B200 through the C++ drop-in
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_cpp_dropin.py -m gpu -q -p no:cacheprovider -s > gpurun_out/dropin_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/dropin_pytest.log
