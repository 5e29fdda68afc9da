#!/bin/bash
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/r2o_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2o_smoke.log
bash scripts/gpu_ab_libs.sh r2o_ch "cur6 u1" --workload channel-d3q27
bash scripts/gpu_ab_libs.sh r2o_po "cur6 u1" --workload porous-d3q19
bash scripts/gpu_ab_libs.sh r2o_tg "cur6 u1"
