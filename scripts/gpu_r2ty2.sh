#!/bin/bash
# TY=10 with the shallow slot rings (rd=0: ~91 KB shared memory, surely 2 CTAs/SM) vs base
set -u
mkdir -p gpurun_out
for i in 1 2; do
  TSLB_LIB=ab/lib_base.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>>gpurun_out/r2ty2.err | sed "s/^/base /" >> gpurun_out/r2ty2.txt
  TSLB_MSTEP_RD=0 TSLB_LIB=ab/lib_ty10.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>>gpurun_out/r2ty2.err | sed "s/^/ty10rd0 /" >> gpurun_out/r2ty2.txt
  TSLB_MSTEP_RD=0 TSLB_LIB=ab/lib_base.so timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>>gpurun_out/r2ty2.err | sed "s/^/baserd0 /" >> gpurun_out/r2ty2.txt
done
python - <<PY
import json
for l in open("gpurun_out/r2ty2.txt"):
    n, j = l.split(" ", 1)
    d = json.loads(j); print(n, d["value"], d["ms_per_step"], d.get("clocks", {}).get("sm_mhz"))
PY
