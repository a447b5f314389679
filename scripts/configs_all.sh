# bench lines for C3, C4 and C5 (fp64, fp32) on one GPU (no CPU leg for C5)
for c in c3 c4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; echo "$c rc=$?"
done
for p in f64 f32; do
  timeout 1200 python bench.py --config c5 --precision $p --steps 5 --warmup 3 --no-cpu > gpurun_out/cfg_c5_$p.json 2> gpurun_out/cfg_c5_$p.err; echo "c5 $p rc=$?"
done
python tools/cta_trace.py --flush > gpurun_out/cta_c2.txt 2>&1
python tools/cta_trace.py --config c3 --size 2048 --flush > gpurun_out/cta_c3.txt 2>&1
