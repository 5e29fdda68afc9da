# compute-sanitizer over a selection of GPU tests (memcheck, then racecheck
# and synccheck on the shared-memory kernels)
mkdir -p gpurun_out
SEL=${1:-"masked or solid_bitwise"}
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$SEL" > gpurun_out/san_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 99 --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "${2:-mstep_solid_bitwise and periodic and d3q19 and float32}" > gpurun_out/san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.log
timeout 1500 compute-sanitizer --tool synccheck --error-exitcode 99 --print-limit 20 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "${2:-mstep_solid_bitwise and periodic and d3q19 and float32}" > gpurun_out/san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck.log
