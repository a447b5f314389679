# ncu full capture of the C5 fp32 update kernel (issue-bound?)
CMD="python bench.py --config c5 --precision f32 --steps 3 --warmup 3 --no-e2e --no-cpu --no-ref-code"
$CMD > gpurun_out/f32_plain.log 2>&1; echo plain_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_update_w" -s 4 -c 1 -o gpurun_out/f32_prof $CMD > gpurun_out/f32_ncu.log 2>&1; echo ncu_rc=$?
ncu -i gpurun_out/f32_prof.ncu-rep --page raw --csv > gpurun_out/f32_raw.csv 2>/dev/null
ncu -i gpurun_out/f32_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/f32_src.csv 2>/dev/null
rm -f gpurun_out/f32_prof.ncu-rep
