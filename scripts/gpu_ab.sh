# A/B bench lines of the default workload (device only)
mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --workload porous-d3q19 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
done
