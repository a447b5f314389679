# round-2 final evidence (v5), part A: ncu launch list of the default command and full captures
# of the update kernel per config / precision (refresh profiles/ncu_traffic.json from the raw exports)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-ref-code > gpurun_out/v5_plain.log 2>&1; echo plain_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v5_launches_c5.csv python bench.py --steps 20 --warmup 5 > gpurun_out/v5_ncu_launch.log 2>&1; echo launch_rc=$?
prof() {  # name, bench args...
  local n=$1; shift
  ncu --set full --clock-control none --import-source on -k regex:"k_update_w|k_speeds_t" -s 6 -c 2 -o gpurun_out/v5_$n python bench.py "$@" --steps 4 --warmup 3 --no-e2e --no-cpu --no-ref-code > gpurun_out/v5_${n}_ncu.log 2>&1; echo "$n ncu rc=$?"
  ncu -i gpurun_out/v5_$n.ncu-rep --page raw --csv > gpurun_out/v5_raw_$n.csv 2>/dev/null
  if [ "$n" = c5 ] || [ "$n" = c4 ]; then ncu -i gpurun_out/v5_$n.ncu-rep --page source --csv --print-source sass > gpurun_out/v5_sass_$n.csv 2>/dev/null; fi
  rm -f gpurun_out/v5_$n.ncu-rep
}
prof c5 --config c5
prof c4 --config c4
prof c3 --config c3
prof c2 --config c2
prof c5f32 --config c5 --precision f32
prof c5fast --config c5 --precision f32fast
prof c4f32 --config c4 --precision f32
ls -la gpurun_out/v5_*
