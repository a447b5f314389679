# ncu full capture of the C5 and C4 update kernels (3 CTAs/SM build)
for cfg in c5 c4; do
  CMD="python bench.py --config $cfg --steps 4 --warmup 3 --no-e2e --no-cpu --no-ref-code"
  $CMD > gpurun_out/pl_${cfg}_plain.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"k_update_w" -s 4 -c 1 -o gpurun_out/pl_$cfg $CMD > gpurun_out/pl_${cfg}_ncu.log 2>&1
  ncu -i gpurun_out/pl_$cfg.ncu-rep --page raw --csv > gpurun_out/pl_${cfg}_raw.csv 2>/dev/null
  ncu -i gpurun_out/pl_$cfg.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pl_${cfg}_src.csv 2>/dev/null
  rm -f gpurun_out/pl_$cfg.ncu-rep
done
echo done
