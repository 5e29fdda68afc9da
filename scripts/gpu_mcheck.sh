# M parity tests + default-workload bench lines (device only)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "mstep or slab or smoke" > gpurun_out/mcheck_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/mcheck_pytest.log
for i in 1 2 3; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu >> gpurun_out/mcheck.jsonl 2>>gpurun_out/mcheck.err
done
