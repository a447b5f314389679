# A/B of the update kernels on C3 / C4 (session-start build in _ab vs HEAD), same box
for round in 1 2; do
for side in head ab; do
  d=.; [ $side = ab ] && d=_ab
  for c in c3 c4; do
    (cd $d && timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu) > gpurun_out/ab_${side}_${c}_$round.json 2>&1
  done
done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["value"]/1e9,3), d["roofline"].get("kernel_ms"), d["roofline"].get("speeds_kernel_ms"))
    except Exception as e: print(f, "ERR", open(f).read()[-300:])
PY
