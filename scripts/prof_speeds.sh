# launch list (filtered vs exact pre-pass) and one full capture of k_speeds_b on C2
CMD="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/ps_plain.log 2>&1; echo plain_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ps_launch_filter.csv $CMD > /dev/null 2>&1; echo rc=$?
WS_SPEEDS=exact ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ps_launch_exact.csv $CMD > /dev/null 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_speeds" -s 6 -c 1 -o gpurun_out/ps_prof $CMD > gpurun_out/ps_ncu.log 2>&1; echo full_rc=$?
ncu -i gpurun_out/ps_prof.ncu-rep --page raw --csv > gpurun_out/ps_raw.csv 2>/dev/null
ncu -i gpurun_out/ps_prof.ncu-rep --page details --csv > gpurun_out/ps_details.csv 2>/dev/null
ncu -i gpurun_out/ps_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ps_src.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
python - <<'PY'
import csv, re, collections
for f in ["ps_launch_filter", "ps_launch_exact"]:
    rows=[r for r in csv.reader(open(f"gpurun_out/{f}.csv")) if len(r)>10]
    h=rows[0]; agg=collections.defaultdict(list)
    for r in rows[1:]:
        d=dict(zip(h,r))
        if d.get("Metric Name")!="gpu__time_duration.sum": continue
        v=float(d["Metric Value"].replace(",",""))* (1e3 if d["Metric Unit"]=="us" else (1e6 if d["Metric Unit"]=="ms" else 1))
        agg[re.sub(r"\(.*$","",d["Kernel Name"]).strip()[:60]].append(v/1e3)
    print(f)
    for k,v in agg.items(): print("  ", k, len(v), "mean us %.2f min %.2f"%(sum(v)/len(v), min(v)))
PY
