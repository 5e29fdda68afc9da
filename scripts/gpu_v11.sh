#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/tma_repro.py 256 4 4 > gpurun_out/v11_repro.log 2>&1
timeout 900 python -m pytest tests/test_gpu_single.py -m gpu -x -q -p no:cacheprovider -k "wide_rows or graph" > gpurun_out/v11_pytest_tma.log 2>&1; echo rc=$? >> gpurun_out/v11_pytest_tma.log
TSLB_VX=2 timeout 900 python -m pytest tests/test_gpu_single.py -m gpu -x -q -p no:cacheprovider -k "wide_rows and tma" > gpurun_out/v11_pytest_tma_vx2.log 2>&1; echo rc=$? >> gpurun_out/v11_pytest_tma_vx2.log
for M in f64 f32; do
  for VX in 1 2; do
    for KZ in 4 16; do
      TSLB_STREAMCOLL=tma TSLB_VX=$VX TSLB_KZ=$KZ timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --math $M > gpurun_out/v11_${M}_tma_vx${VX}_kz${KZ}.json 2>&1
    done
  done
done
TSLB_STREAMCOLL=tma TSLB_VX=1 TSLB_KZ=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_streamcoll -s 2 -c 1 -o gpurun_out/v11_prof_tma_f64 python bench.py --steps 2 --warmup 1 --n 256 --no-e2e --no-cpu > gpurun_out/v11_ncu.log 2>&1
