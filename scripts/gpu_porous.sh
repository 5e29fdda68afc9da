mkdir -p gpurun_out
for s in m f1; do timeout 300 python bench.py --workload porous-d3q19 --schedule $s --steps 20 --warmup 3 >> gpurun_out/porous.jsonl 2>> gpurun_out/porous.err; done
timeout 300 python bench.py --workload porous-d3q19 --schedule m --math f32 --steps 20 --warmup 3 >> gpurun_out/porous.jsonl 2>> gpurun_out/porous.err
