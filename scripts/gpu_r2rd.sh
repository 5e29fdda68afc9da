#!/bin/bash
# fp32 node math: slot-ring depth rd=1 (2 CTAs/SM, default) vs rd=0 (3 CTAs/SM)
set -u
mkdir -p gpurun_out
for i in 1 2; do
  for rd in 1 0; do
    TSLB_MSTEP_RD=$rd timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --math f32 2>>gpurun_out/r2rd.err | sed "s/^/rd$rd /" >> gpurun_out/r2rd.txt
  done
done
python - <<PY
import json
for l in open("gpurun_out/r2rd.txt"):
    n, j = l.split(" ", 1)
    d = json.loads(j); print(n, d["value"], d["ms_per_step"], d.get("clocks", {}).get("sm_mhz"))
PY
