# TMA-stored output tile A/B (TSLB_MSTEP_TST) + M parity tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "mstep or slab" > gpurun_out/tst_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/tst_pytest.log
for i in 1 2; do for t in 0 1; do
TSLB_MSTEP_TST=$t timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu | sed "s/^/tst=$t /" >> gpurun_out/tst.txt 2>>gpurun_out/tst.err
TSLB_MSTEP_TST=$t timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --math f32 | sed "s/^/tst=$t,f32 /" >> gpurun_out/tst.txt 2>>gpurun_out/tst.err
done; done
