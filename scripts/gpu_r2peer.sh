#!/bin/bash
# fused peer epilogue: default path unchanged? IPC tests, IPC self probe
set -u
mkdir -p gpurun_out
rm -f gpurun_out/r2peer2*.txt
bash scripts/gpu_ab_libs.sh r2peer2 "base peer"
timeout 900 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_slabs.py -m gpu -x -q > gpurun_out/r2peer_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2peer_tests.log
tail -3 gpurun_out/r2peer_tests.log
for i in 1 2; do
  timeout 300 python bench.py --ipc-self --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2peer_ipcself$i.json 2>>gpurun_out/r2peer.err
done
python - <<PY
import json, glob
for l in open("gpurun_out/r2peer2.txt"):
    n, j = l.split(" ", 1); d = json.loads(j); print(n, d["value"])
for f in sorted(glob.glob("gpurun_out/r2peer_ipcself*.json")):
    d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
    print(f, d["value"], r["kernel_ms_per_step"], r["launches_per_step"])
PY
