#!/bin/bash
# streaming (evict-first) loads/stores: colour moments kernel (droplet) and M kernel moment stores (TGV 1024^3)
set -u
mkdir -p gpurun_out
rm -f gpurun_out/r2str_*.txt
bash scripts/gpu_ab_libs.sh r2str_cg "base cgms" --workload droplet-d3q19 --steps 10
bash scripts/gpu_ab_libs.sh r2str_m "base mstcs"
bash scripts/gpu_ab_libs.sh r2str_m32 "base mstcs" --math f32
python - <<PY
import json
for f in ("gpurun_out/r2str_cg.txt", "gpurun_out/r2str_m.txt", "gpurun_out/r2str_m32.txt"):
    for l in open(f):
        n, j = l.split(" ", 1); d = json.loads(j); print(f[11:], n, d["value"], d["roofline"]["kernel_ms_per_step"])
PY
