#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mstep.py -m gpu -q -p no:cacheprovider -k "f16" -s > gpurun_out/r2n_f16.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_f16.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2n_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_pytest.log
for st in native f16; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --storage $st --math f32 > gpurun_out/r2n_bench_$st.json 2>> gpurun_out/r2n_bench.err
done
