#!/bin/bash
mkdir -p gpurun_out
TSLB_STREAMCOLL=row TSLB_KZ=3 timeout 900 python -m pytest tests/test_gpu_single.py tests/test_gpu_golden.py tests/test_gpu_slabs.py -m gpu -x -q -p no:cacheprovider > gpurun_out/v7_pytest_row.log 2>&1; echo rc=$? >> gpurun_out/v7_pytest_row.log
for M in f64 f32; do
  for KZ in 4 8 16; do
    TSLB_STREAMCOLL=row TSLB_VX=2 TSLB_KZ=$KZ timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --math $M > gpurun_out/v7_${M}_row_kz${KZ}.json 2>&1
  done
  TSLB_STREAMCOLL=vec TSLB_VX=2 TSLB_KZ=8 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --math $M > gpurun_out/v7_${M}_pipe2_kz8.json 2>&1
done
TSLB_STREAMCOLL=row TSLB_VX=2 TSLB_KZ=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_streamcoll -s 2 -c 1 -o gpurun_out/v7_prof_row_f64 python bench.py --steps 2 --warmup 1 --n 256 --no-e2e --no-cpu > gpurun_out/v7_ncu.log 2>&1
