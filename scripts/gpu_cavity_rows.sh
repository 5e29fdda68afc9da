mkdir -p gpurun_out
for R in 0 1 2 3 4 8; do
  if [ $R = 0 ]; then E=""; else E="TSLB_ROWS2D=$R"; fi
  env $E timeout 300 python bench.py --workload cavity-d2q9 --steps 2000 --warmup 64 --no-e2e --no-cpu 2>/dev/null | sed "s/^/R$R /" >> gpurun_out/cav_rows.txt
done
