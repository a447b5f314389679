# ncu full captures of the round-2 kernels: C3 fp64 (2 CTAs/SM), C5 f32fast
# and f32 (4 CTAs/SM), C1 multi-step kernel (k_run_small)
prof() {  # name cmd...
  local n=$1; shift
  "$@" > gpurun_out/p2_${n}_plain.log 2>&1; echo "$n plain rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:"k_update_w|k_run_small" -s 4 -c 1 -o gpurun_out/p2_$n "$@" > gpurun_out/p2_${n}_ncu.log 2>&1; echo "$n ncu rc=$?"
  ncu -i gpurun_out/p2_$n.ncu-rep --page raw --csv > gpurun_out/p2_${n}_raw.csv 2>/dev/null
  ncu -i gpurun_out/p2_$n.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/p2_${n}_src.csv 2>/dev/null
  rm -f gpurun_out/p2_$n.ncu-rep
}
prof c3 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-ref-code
prof c5fast python bench.py --config c5 --precision f32fast --steps 3 --warmup 3 --no-e2e --no-cpu --no-ref-code
prof c5f32 python bench.py --config c5 --precision f32 --steps 3 --warmup 3 --no-e2e --no-cpu --no-ref-code
