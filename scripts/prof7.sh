# full ncu capture of one k_update_w launch, C5 recipe at 4096^2 in fp32
CMD="python bench.py --config c5 --size 4096 --precision f32 --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_p7.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_update_w" -s 3 -c 1 -o gpurun_out/prof_p7 $CMD > gpurun_out/ncu_p7.log 2>&1
echo ncu_rc=$?
ncu -i gpurun_out/prof_p7.ncu-rep --page raw --csv > gpurun_out/raw_p7.csv 2>/dev/null
ncu -i gpurun_out/prof_p7.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_p7.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
