"""Executed warp instructions of one kernel per source region and opcode.

Joins an ncu `--page source --csv --print-source sass` export (per SASS
address: Instructions Executed, stall samples) with the line info of the
same binary (`nvdisasm --print-line-info-inline -c X.cubin > X.lsass`): each
instruction is attributed to the OUTERMOST ws_kernels.cuh line of its inline
chain, regions are line ranges of the kernel body.

    python tools/ncu_regions.py SASS.csv X.lsass KERNEL_MANGLED_SUBSTR CELLS name:a-b [name:a-b ...]
"""
import collections
import csv
import re
import sys


def lsass_lines(path, kern):
    """[(offset, outer_line, opcode)] of the kernel, in address order."""
    out, cur, line = [], None, None
    for ln in open(path):
        m = re.match(r"\.text\.(\S+):", ln)
        if m:
            cur = m.group(1)
            continue
        if cur is None or kern not in cur:
            continue
        if ln.lstrip().startswith("//## File"):
            o = re.findall(r'ws_kernels\.cuh", line (\d+)', ln)
            line = int(o[-1]) if o else line
            continue
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
        if m:
            out.append((int(m.group(1), 16), line, m.group(2)))
    return out


def main():
    csvp, lsass, kern, cells = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    regions = []
    for a in sys.argv[5:]:
        n, r = a.split(":")
        lo, hi = r.split("-")
        regions.append((n, int(lo), int(hi)))
    ins = lsass_lines(lsass, kern)
    rows = list(csv.reader(open(csvp)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    iex, ist = hdr.index("Instructions Executed"), hdr.index("# Samples")
    data = [r for r in rows if r and r[0].startswith("0x") and len(r) >= len(hdr) - 1]
    base = int(data[0][0], 16)
    assert len(data) == len(ins), (len(data), len(ins))
    per = collections.defaultdict(collections.Counter)
    stall = collections.Counter()
    tot = 0
    for r, (off, line, op) in zip(data, ins):
        assert int(r[0], 16) - base == off - ins[0][0], (r[0], off)
        ex = int(r[iex] or 0) * 32   # lane-instructions (warp-level count x 32)
        name = next((n for n, lo, hi in regions if line is not None and lo <= line <= hi), "other")
        per[name][op] += ex
        stall[name] += int(r[ist] or 0)
        tot += ex
    ts = sum(stall.values())
    print(f"total {tot / cells:.1f} lane-instructions per cell")
    for name in [n for n, _, _ in regions] + ["other"]:
        c = per[name]
        t = sum(c.values())
        fp = sum(v for k, v in c.items() if k in ("DMUL", "DADD", "DFMA", "DSETP"))
        print(f"{name:10s} {t / cells:7.1f}/cell  fp64 {fp / cells:6.1f}  stall samples {100 * stall[name] / max(ts, 1):4.1f}%  "
              + ", ".join(f"{k} {v / cells:.1f}" for k, v in c.most_common(14)))


if __name__ == "__main__":
    main()
