# memcheck over the whole GPU suite; racecheck over the shared-memory M kernel variants
mkdir -p gpurun_out
timeout 3000 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "not full_size and not dropin and not acceptance" > gpurun_out/san_all_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_all_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 99 --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "test_mstep_bitwise and (box-corners or periodic-wide)" > gpurun_out/san_all_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_all_racecheck.log
