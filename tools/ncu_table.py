"""One markdown column per `ncu --page raw --csv` export: the update kernel's headline counters.

    python tools/ncu_table.py LABEL=RAW.csv:CELLS [LABEL=RAW.csv:CELLS ...]
"""
import csv
import re
import sys

ROWS = [("kernel", "kernel"), ("duration ms", "dur"), ("DRAM read + write GB", "gb"),
        ("DRAM GB/s (frac of 6547)", "gbs"), ("FP64 pipe % / FMA pipe %", "fp"),
        ("issue active %", "issue"), ("warps active %", "warps"),
        ("thread instructions / cell", "ipc"), ("registers", "regs"),
        ("grid × block, smem KB", "grid"), ("top stalls", "stalls")]


def num(d, k):
    try:
        return float(d[k].replace(",", ""))
    except Exception:
        return None


def column(label, path, cells):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    u = dict(zip(hdr, units))
    ks = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    d = next(k for k in ks if "k_update_w" in k["Kernel Name"])
    dur_ms = num(d, "gpu__time_duration.sum") * {"ns": 1e-6, "us": 1e-3, "ms": 1, "s": 1e3}[u["gpu__time_duration.sum"]]

    def byt(k):
        return num(d, k) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[k]]

    b = byt("dram__bytes_read.sum") + byt("dram__bytes_write.sum")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(d, k) for k in d
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(v for v in st.values() if v)
    top = sorted(((v, k) for k, v in st.items() if v), reverse=True)[:6]
    smem = num(d, "launch__shared_mem_per_block_dynamic")
    smem = smem / 1e3 if u["launch__shared_mem_per_block_dynamic"] == "byte" else smem
    kern = re.sub(r"\(const.*$", "", d["Kernel Name"])
    for junk in ("ws::", "(int)", "(bool)"):
        kern = kern.replace(junk, "")
    return dict(
        label=label, kernel="`" + kern + "`", dur=f"{dur_ms:.3f}", gb=f"{b / 1e9:.3f}",
        gbs=f"{b / 1e9 / (dur_ms * 1e-3):.0f} ({b / 1e9 / (dur_ms * 1e-3) / 6547:.3f})",
        fp=f"{num(d, 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):.1f} / "
           f"{num(d, 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active') or 0:.1f}",
        issue=f"{num(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f}",
        warps=f"{num(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}",
        ipc=f"{num(d, 'smsp__inst_executed.sum') * 32 / cells:.0f}", regs=d["launch__registers_per_thread"],
        grid=f"{d['launch__grid_size']} × {d['launch__block_size']}, {smem:.1f}",
        stalls=", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in top))


def main():
    cols = []
    for a in sys.argv[1:]:
        label, rest = a.split("=", 1)
        path, cells = rest.rsplit(":", 1)
        cols.append(column(label, path, float(cells)))
    print("| | " + " | ".join(c["label"] for c in cols) + " |")
    print("|---|" + "---|" * len(cols))
    for lab, key in ROWS:
        print(f"| {lab} | " + " | ".join(c[key] for c in cols) + " |")


if __name__ == "__main__":
    main()
