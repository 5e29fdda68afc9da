#!/bin/bash
# the reference's acceptance gate and unit suites on the B200 through the C++ drop-in
mkdir -p gpurun_out
timeout 1500 ./oracle/_ref/dropin_acceptance > gpurun_out/acceptance.log 2>&1; echo "rc=$?" >> gpurun_out/acceptance.log
