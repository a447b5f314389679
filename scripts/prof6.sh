# full ncu capture of one k_update_w launch for ${CFG:-c3}, with source
CMD="python bench.py --config ${CFG:-c3} --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_p6.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"${KRN:-k_update_w}" -s 3 -c 1 -o gpurun_out/prof_p6 $CMD > gpurun_out/ncu_p6.log 2>&1
echo ncu_rc=$?
ncu -i gpurun_out/prof_p6.ncu-rep --page raw --csv > gpurun_out/raw_p6.csv 2>/dev/null
ncu -i gpurun_out/prof_p6.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_p6.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
