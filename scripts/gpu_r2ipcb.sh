#!/bin/bash
# peer-memory transport in bench: self-exchange probes (NCCL vs IPC) at 1024^3,
# and the 2-rank bench path on this one GPU (functional; timings meaningless)
set -u
mkdir -p gpurun_out
B="--steps 20 --warmup 3 --no-e2e --no-cpu"
for i in 1 2; do
  timeout 600 python bench.py --nccl-self $B > gpurun_out/r2ipcb_nccl$i.json 2>>gpurun_out/r2ipcb.err
  timeout 600 python bench.py --ipc-self $B > gpurun_out/r2ipcb_ipc$i.json 2>>gpurun_out/r2ipcb.err
done
TSLB_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --transport ipc --n 256 --steps 10 --warmup 3 > gpurun_out/r2ipcb_two.json 2>>gpurun_out/r2ipcb.err
echo "two rc=$?" >> gpurun_out/r2ipcb.err
TSLB_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 3 --transport ipc --workload tgv-c5 --dims 256,256,384 --steps 10 --warmup 3 > gpurun_out/r2ipcb_c5x3.json 2>>gpurun_out/r2ipcb.err
echo "c5x3 rc=$?" >> gpurun_out/r2ipcb.err
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/r2ipcb_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        r=d.get("roofline",{})
        print(f, d["value"], d["ms_per_step"], r.get("kernel_ms_per_step"), d["config"].get("parallelism"))
    except Exception as e: print(f, "ERR", e, open(f).read()[-300:])
PY
tail -5 gpurun_out/r2ipcb.err
