bash scripts/gpu_ab_libs.sh r2e_ab "msum cur"
( time timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r2e_ref.json 2> gpurun_out/r2e_ref.err
