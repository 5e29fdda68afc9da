#!/bin/bash
# two-fluid one-pass step: parity tests, then droplet 512^3 one-pass vs two-kernel
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_two.py -m gpu -x -q -k "one_pass" > gpurun_out/r2cf_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2cf_tests.log
tail -30 gpurun_out/r2cf_tests.log
for i in 1 2; do
  timeout 300 python bench.py --workload droplet-d3q19 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2cf_fused$i.json 2>>gpurun_out/r2cf.err
  TSLB_CG_FUSED=0 timeout 300 python bench.py --workload droplet-d3q19 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2cf_two$i.json 2>>gpurun_out/r2cf.err
done
for f in gpurun_out/r2cf_*.json; do echo $f; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['ms_per_step'], r['frac'], r['kernel_ms_per_step'], d['schedule'][:40])"; done
tail -3 gpurun_out/r2cf.err
