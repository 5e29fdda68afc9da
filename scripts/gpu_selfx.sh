# multi-GPU step probe on one GPU: slab + 1-rank NCCL self exchange vs the plain box
mkdir -p gpurun_out
for s in m f1; do
timeout 400 python bench.py --nccl-self --schedule $s --steps 20 --warmup 3 >> gpurun_out/selfx.jsonl 2>>gpurun_out/selfx.err
timeout 400 python bench.py --schedule $s --steps 20 --warmup 3 --no-e2e --no-cpu >> gpurun_out/selfx.jsonl 2>>gpurun_out/selfx.err
done
timeout 900 python bench.py > gpurun_out/default_check.json 2> gpurun_out/default_check.err
