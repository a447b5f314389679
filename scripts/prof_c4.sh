CMD="python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/c4p_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_update_w" -s 4 -c 1 -o gpurun_out/c4p $CMD > gpurun_out/c4p_ncu.log 2>&1
echo ncu_rc=$?
ncu -i gpurun_out/c4p.ncu-rep --page raw --csv > gpurun_out/c4p_raw.csv 2>/dev/null
ncu -i gpurun_out/c4p.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c4p_src.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
