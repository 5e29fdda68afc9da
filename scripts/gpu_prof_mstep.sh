#!/bin/bash
# ncu --set full of k_mstep (512^3, fp64 node math) for library variants
# ab/lib_<name>.so; keeps the report, its summary, the SASS source page
# (per-instruction stall samples) and the raw page
# usage: gpu_prof_mstep.sh TAG "names" [bench args]
TAG=${1:-prof}
NAMES=${2:-"new"}
shift 2
mkdir -p gpurun_out
for n in $NAMES; do
  R=gpurun_out/${TAG}_${n}
  TSLB_LIB=ab/lib_$n.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mstep -s 3 -c 1 \
    -o $R python bench.py --steps 2 --warmup 3 --n 512 --no-e2e --no-cpu "$@" > ${R}_ncu.log 2>&1
  python tools/ncu_summary.py $R.ncu-rep 10737418240 > ${R}_summary.txt 2>&1
  ncu -i $R.ncu-rep --page source --csv --print-source=sass > ${R}_sass.csv 2>/dev/null
  ncu -i $R.ncu-rep --page raw --csv > ${R}_raw.csv 2>/dev/null
  python tools/sass_mix.py ${R}_sass.csv 134217728 > ${R}_sass_mix.txt 2>&1
done
