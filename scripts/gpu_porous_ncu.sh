# ncu of the masked M kernel (porous workload, 256^3) + its bench lines
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mstep -s 3 -c 1 -o gpurun_out/porous_mstep_f64 python bench.py --workload porous-d3q19 --dims 256,256,256 --steps 2 --warmup 3 > gpurun_out/porous_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mstep -s 3 -c 1 -o gpurun_out/tgv256_mstep_f64 python bench.py --workload tgv-d3q19 --dims 256,256,256 --steps 2 --warmup 3 --no-e2e --no-cpu >> gpurun_out/porous_ncu.log 2>&1
