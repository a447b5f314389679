# final evidence pass: headline both arms, every config line (fp64, fp32,
# f32fast), the bench matrix, the ncu launch list of the default command and a
# full capture of its step kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke_rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; echo ref_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/fin_c5.json 2> gpurun_out/fin_c5.err; echo c5_rc=$?
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/fin_$c.json 2> gpurun_out/fin_$c.err; echo "$c rc=$?"
done
for c in c5 c4 c3; do for p in f32 f32fast; do
  timeout 900 python bench.py --config $c --precision $p --steps 10 --warmup 3 --no-cpu > gpurun_out/fin_${c}_$p.json 2> gpurun_out/fin_${c}_$p.err; echo "$c $p rc=$?"
done; done
bash scripts/matrix.sh
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c5.csv python bench.py --steps 20 --warmup 5 > gpurun_out/fin_ncu_launch.log 2>&1; echo launch_rc=$?
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-ref-code"
ncu --set full --clock-control none --import-source on -k regex:"k_update_w|k_speeds" -s 6 -c 2 -o gpurun_out/fin_prof_c5 $CMD > gpurun_out/fin_ncu_full.log 2>&1; echo full_rc=$?
ncu -i gpurun_out/fin_prof_c5.ncu-rep --page raw --csv > gpurun_out/fin_raw_c5.csv 2>/dev/null
ncu -i gpurun_out/fin_prof_c5.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/fin_src_c5.csv 2>/dev/null
rm -f gpurun_out/fin_prof_c5.ncu-rep
for f in gpurun_out/fin_*.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d.get('roofline',{})
    e=d.get('e2e') or {}
    print(sys.argv[1], round(d['value']/1e9,4), 'G/s  ms/step', round(d['ms_per_step'],4), 'e2e', round((e.get('value') or 0)/1e9,3), 'sim', round((d.get('simulation') or {}).get('cell_updates_per_s',0)/1e9,3), 'fp64', (r.get('fp64') or {}).get('frac'), 'issue', (r.get('issue') or {}).get('frac'))
except Exception as ex: print(sys.argv[1], 'FAILED', ex)
PY
done
