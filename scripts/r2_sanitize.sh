# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) on the GPU parity subset,
# including the device-side reduction / halo shards that spin-wait on peer counters
mkdir -p gpurun_out/san
SUB="tests/test_gpu_parity.py -k first_order_bitwise or second_order_bitwise or tiny_grids or t_final or inadmissible"
MS="tests/test_gpu_multishard.py"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 99 --print-limit 50 \
     --log-file gpurun_out/san/${tool}_parity.log \
     python -m pytest tests/test_gpu_parity.py -q -x -k "first_order_bitwise and extrapolate or second_order_bitwise and mc or tiny_grids or back_to_back or inadmissible" > gpurun_out/san/${tool}_parity.out 2>&1
  echo "$tool parity rc=$?"; tail -2 gpurun_out/san/${tool}_parity.out
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 99 --print-limit 50 \
     --log-file gpurun_out/san/${tool}_shards.log \
     python -m pytest $MS -q -x -k "device_side or fake_shards_bitwise and 2-extrapolate" > gpurun_out/san/${tool}_shards.out 2>&1
  echo "$tool shards rc=$?"; tail -2 gpurun_out/san/${tool}_shards.out
  grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|Hazard\|Error" gpurun_out/san/${tool}_*.log | sort | uniq -c | head -8
done
