set -x
CMD="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launch_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_update -s 4 -c 1 -o gpurun_out/prof_update $CMD > gpurun_out/ncu_full_update.log 2>&1
echo full_update_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_speeds -s 4 -c 1 -o gpurun_out/prof_speeds $CMD > gpurun_out/ncu_full_speeds.log 2>&1
echo full_speeds_rc=$?
tail -1 gpurun_out/plain.log
