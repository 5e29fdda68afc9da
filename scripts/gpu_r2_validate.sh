#!/bin/bash
# round-2 validation: smoke, every -m gpu test, the default bench line (the
# driver's command), every workload line, the slab probe, C5 on one GPU, the
# reference arm, the ncu launch list and one --set full capture per
# dominant kernel (summaries + SASS stall pages kept under gpurun_out/)
TAG=${1:-r2v}
mkdir -p gpurun_out
(nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,clocks.sm --format=csv; free -g; nproc) > gpurun_out/${TAG}_env.txt 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_default.json 2> gpurun_out/${TAG}_default.err
B="--no-e2e --no-cpu"
timeout 600 python bench.py --steps 20 --warmup 3 $B --math f32 > gpurun_out/${TAG}_tgv1024_f32.json 2>> gpurun_out/${TAG}_wl.err
timeout 600 python bench.py --steps 20 --warmup 3 $B --storage f16 > gpurun_out/${TAG}_tgv1024_f16.json 2>> gpurun_out/${TAG}_wl.err
timeout 600 python bench.py --steps 20 --warmup 3 $B --schedule f1 > gpurun_out/${TAG}_tgv1024_f1.json 2>> gpurun_out/${TAG}_wl.err
timeout 600 python bench.py --n 512 --steps 20 --warmup 3 $B > gpurun_out/${TAG}_tgv512.json 2>> gpurun_out/${TAG}_wl.err
timeout 600 python bench.py --dims 1000,1000,1000 --steps 20 --warmup 3 $B > gpurun_out/${TAG}_tgv1000.json 2>> gpurun_out/${TAG}_wl.err
timeout 600 python bench.py --nccl-self --steps 20 --warmup 3 $B > gpurun_out/${TAG}_selfx.json 2>> gpurun_out/${TAG}_wl.err
timeout 900 python bench.py --workload tgv-c5 --steps 10 --warmup 3 $B > gpurun_out/${TAG}_c5.json 2>> gpurun_out/${TAG}_wl.err
timeout 600 python bench.py --workload droplet-d3q19 --steps 10 --warmup 3 > gpurun_out/${TAG}_droplet.json 2>> gpurun_out/${TAG}_wl.err
timeout 900 python bench.py --workload channel-d3q27 --steps 10 --warmup 3 > gpurun_out/${TAG}_channel.json 2>> gpurun_out/${TAG}_wl.err
timeout 900 python bench.py --workload channel-d3q27 --steps 10 --warmup 3 --math f32 --no-cpu > gpurun_out/${TAG}_channel_f32.json 2>> gpurun_out/${TAG}_wl.err
timeout 600 python bench.py --workload cavity-d2q9 --steps 2000 --warmup 64 > gpurun_out/${TAG}_cavity.json 2>> gpurun_out/${TAG}_wl.err
timeout 600 python bench.py --workload tgv-d2q9 --steps 20 --warmup 3 > gpurun_out/${TAG}_tgv2d.json 2>> gpurun_out/${TAG}_wl.err
timeout 600 python bench.py --workload porous-d3q19 --steps 20 --warmup 3 > gpurun_out/${TAG}_porous.json 2>> gpurun_out/${TAG}_wl.err
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err
# ncu: launch list of the default command (512^3), then one full capture per dominant kernel
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --n 512 $B > /dev/null 2>&1
N="--set full --clock-control none --import-source on"
cap() {  # name kernel-regex bench-args...
  local name=$1 kre=$2; shift 2
  timeout 900 ncu $N -k regex:$kre -s 3 -c 1 -o gpurun_out/${TAG}_$name python bench.py --steps 2 --warmup 3 $B "$@" > gpurun_out/${TAG}_${name}_ncu.log 2>&1
  ncu -i gpurun_out/${TAG}_$name.ncu-rep --page source --csv --print-source=sass > gpurun_out/${TAG}_${name}_sass.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_$name.ncu-rep --page raw --csv > gpurun_out/${TAG}_${name}_raw.csv 2>/dev/null
}
cap mstep_f64 k_mstep --n 512
cap mstep_f32 k_mstep --n 512 --math f32
cap mstep_f16 k_mstep --n 512 --storage f16
cap droplet_scr k_cg_streamcoll_box --workload droplet-d3q19
cap d3q27_mstep k_mstep --workload channel-d3q27 --dims 512,512,512
# summarise on the box (gpurun copies back <= 64 MiB): text summaries into
# gpurun_out/${TAG}_profiles/, then drop the reports and SASS pages
python tools/collect_r2.py ${TAG} r02 gpurun_out/${TAG}_profiles > gpurun_out/${TAG}_collect.log 2>&1
rm -f gpurun_out/${TAG}_*.ncu-rep gpurun_out/${TAG}_*_sass.csv gpurun_out/${TAG}_*_raw.csv
