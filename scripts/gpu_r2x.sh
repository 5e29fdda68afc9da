#!/bin/bash
# two NCCL ranks on one GPU? + the HBM read:write mix probe (vector variants)
set -u
mkdir -p gpurun_out
NCCL_DEBUG=WARN timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 tools/micro/nccl_share_probe.py > gpurun_out/r2x_share.log 2>&1
echo "share rc=$?" >> gpurun_out/r2x_share.log
timeout 300 tools/micro/rw_mix > gpurun_out/r2x_rwmix.txt 2>&1
tail -15 gpurun_out/r2x_share.log; cat gpurun_out/r2x_rwmix.txt
