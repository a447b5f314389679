# C4 / C5 executed-instruction profile per SASS address (joined locally with nvdisasm line info)
for c in c4 c5; do
CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu --no-ref-code"
ncu --set full --clock-control none --import-source on -k regex:"k_update_w" -s 4 -c 1 -o gpurun_out/s6p_$c $CMD > gpurun_out/s6p_${c}_ncu.log 2>&1
echo ncu_rc=$?
ncu -i gpurun_out/s6p_$c.ncu-rep --page raw --csv > gpurun_out/s6p_${c}_raw.csv 2>/dev/null
ncu -i gpurun_out/s6p_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/s6p_${c}_sass.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
done
ls -la gpurun_out/s6p_*
