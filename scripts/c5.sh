# C5 (16384^2 shallow water, 20 steps) at N=1, fp64 and fp32; no CPU leg (one
# oracle step of 268M cells needs tens of GB of host temporaries)
for p in f64 f32; do
timeout 1200 python bench.py --config c5 --precision $p --steps 5 --warmup 3 --no-cpu > gpurun_out/c5_$p.log 2>&1
echo "$p rc=$?"; tail -1 gpurun_out/c5_$p.log | cut -c1-400
done
