"""Summarise an ncu launch list + raw --set full export into markdown tables.

    python tools/ncu_summary.py LAUNCHES.csv RAW.csv [--json OUT.json --config c2]

LAUNCHES.csv: `ncu --metrics gpu__time_duration.sum --csv --log-file`;
RAW.csv: `ncu -i rep --page raw --csv`.  Prints the launch-share table and
one column of full-set metrics per captured kernel; --json refreshes the
per-config entry bench.py reads for roofline.traffic / roofline.fp64.
"""
import argparse
import collections
import csv
import json
import re


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    agg = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Unit"] == "us":
            v *= 1e3
        elif d["Metric Unit"] == "ms":
            v *= 1e6
        name = re.sub(r"\(.*$", "", d["Kernel Name"]).strip()
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + v)
    total = sum(t for _, t in agg.values())
    out = ["| kernel | launches | mean us | share of GPU time |", "|---|---|---|---|"]
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{name}` | {n} | {t / n / 1e3:.2f} | {100 * t / total:.1f}% |")
    return "\n".join(out), agg


METRICS = [
    ("duration us", "gpu__time_duration.sum", 1e-3),
    ("DRAM read bytes", "dram__bytes_read.sum", None),
    ("DRAM write bytes", "dram__bytes_write.sum", None),
    ("FP64 pipe active % of peak", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("warps active % of peak", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("SM active cycles / elapsed", None, None),
    ("warp instructions", "smsp__inst_executed.sum", 1),
    ("registers / thread", "launch__registers_per_thread", 1),
    ("grid", "launch__grid_size", 1),
    ("block", "launch__block_size", 1),
]


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    kernels = []
    for r in data:
        d = dict(zip(hdr, r))
        kernels.append(d)
    return hdr, units, kernels


def num(d, k):
    try:
        return float(str(d.get(k, "")).replace(",", ""))
    except ValueError:
        return None


def dram_bytes(d, units, hdr, k):
    v = num(d, k)
    if v is None:
        return None
    u = dict(zip(hdr, units)).get(k, "byte").lower()
    scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
    return v * scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("launches")
    ap.add_argument("raw")
    ap.add_argument("--json", default=None)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--key", default=None,
                    help="entry name in the --json file (default: --config; e.g. c5_f32)")
    ap.add_argument("--cells", type=float, default=None,
                    help="cells per launch (default: the --config's grid)")
    a = ap.parse_args()
    if a.cells is None:
        a.cells = float({"c1": 256, "c2": 1024, "c3": 4096, "c4": 8192, "c5": 16384}[a.config] ** 2)
    table, _ = launches(a.launches)
    print("## Launch list (cold-cache, serialised; shares)\n")
    print(table)
    hdr, units, ks = raw(a.raw)
    names = [re.sub(r"<.*", "", d.get("Kernel Name", "?")).replace("void ", "") for d in ks]
    print("\n## Full-set metrics, one launch each\n")
    print("| metric | " + " | ".join(f"`{n}`" for n in names) + " |")
    print("|---|" + "---|" * len(ks))
    for label, key, scale in METRICS:
        vals = []
        for d in ks:
            if key is None:
                a_ = num(d, "sm__cycles_active.avg")
                e_ = num(d, "gpc__cycles_elapsed.max")
                vals.append(f"{a_ / e_:.3f}" if a_ and e_ else "—")
            elif "dram" in key:
                v = dram_bytes(d, units, hdr, key)
                vals.append(f"{v / 1e6:.3f} MB" if v is not None else "—")
            else:
                v = num(d, key)
                if v is None:
                    vals.append(str(d.get(key, "—")))
                else:
                    if key == "gpu__time_duration.sum":
                        u = dict(zip(hdr, units)).get(key, "ns")
                        v = v * (1e-3 if u == "ns" else (1 if u == "us" else 1e3))
                        vals.append(f"{v:.2f}")
                    else:
                        vals.append(f"{v:g}")
        print(f"| {label} | " + " | ".join(vals) + " |")
    stall = {}
    for d, n in zip(ks, names):
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(d, k) for k in d
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        top = sorted(((v, k) for k, v in st.items() if v), reverse=True)[:6]
        stall[n] = ", ".join(f"{k} {int(v)}" for v, k in top)
    print("| top stall samples | " + " | ".join(stall[n] for n in names) + " |")
    if a.json:
        upd = next(d for d, n in zip(ks, names) if "k_update" in n)
        b = dram_bytes(upd, units, hdr, "dram__bytes_read.sum") + \
            dram_bytes(upd, units, hdr, "dram__bytes_write.sum")
        fp = num(upd, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")
        dur = num(upd, "gpu__time_duration.sum")
        u = dict(zip(hdr, units)).get("gpu__time_duration.sum", "ns")
        dur_us = dur * {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(u, 1.0)
        # FP64 warp-instr = pct x 0.5 warp-instr/clk/SMSP x 4 SMSP x 148 SM x active cycles
        cyc = num(upd, "sm__cycles_active.avg")
        per_cell = fp / 100 * 0.5 * 4 * 148 * cyc * 32 / a.cells if cyc else None
        try:
            js = json.load(open(a.json))
        except Exception:
            js = {}
        js[a.key or a.config] = {
            "bytes_per_launch": int(b), "kernel": names[ks.index(upd)],
            "source": f"{a.raw} (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum)",
            "note": ("1024^2 state (25 MB) is L2-resident: q_new stays in the 126 MB L2 "
                     "during the launch; ncu flushes caches before the replay, so the reads "
                     "come from DRAM") if a.cells <= (1 << 21) else
                    "state larger than L2: DRAM bytes vs the algorithmic 48 B/cell show the "
                    "re-read overhead",
            "fp64_pipe_active_pct": fp,
            "issue_active_pct": num(upd, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "ncu_duration_us": dur_us,
            "fp64_instr_per_cell_approx": round(per_cell) if per_cell and fp > 1.0 else None,
            "instr_per_cell": round(num(upd, "smsp__inst_executed.sum") * 32 / a.cells),
            "issue_peak_instr_per_s": 148 * 4 * 32 * 1.965e9,
            "fp64_peak_instr_per_s": 18.05e12,
            "fp64_peak_source": "profiles/r1_fp64_peak.json"}
        with open(a.json, "w") as f:
            json.dump(js, f, indent=1)


if __name__ == "__main__":
    main()
