CMD="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_p5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_update_w" -s 4 -c 1 -o gpurun_out/prof_p5 $CMD > gpurun_out/ncu_p5.log 2>&1
echo ncu_rc=$?
ncu -i gpurun_out/prof_p5.ncu-rep --page raw --csv > gpurun_out/raw_p5.csv 2>/dev/null
ncu -i gpurun_out/prof_p5.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_p5.csv 2>/dev/null
ncu -i gpurun_out/prof_p5.ncu-rep --page details --csv > gpurun_out/det_p5.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
