"""Executed warp instructions by SASS opcode (and per source line for one
opcode class) from an ncu `--page source --csv --print-source cuda,sass`
export.   python tools/ncu_sass_mix.py SRC.csv KERNEL [OPCODE_PREFIX]"""
import collections
import csv
import re
import sys


def main():
    path, kern = sys.argv[1], sys.argv[2]
    want = sys.argv[3] if len(sys.argv) > 3 else None
    rows = list(csv.reader(open(path)))
    fn = hdr = None
    src_line = None
    ops = collections.Counter()
    by_line = collections.Counter()
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if len(r) == 2 and r[0] == "Function Name":
            fn = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            iex = hdr.index("Instructions Executed")
            continue
        if not (hdr and fn and kern in fn) or len(r) != len(hdr):
            continue
        if r[0]:
            src_line = f"{cur_file}:{r[0]}"
            continue
        if r[2].startswith("0x"):
            m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", r[3])
            if not m:
                continue
            op = m.group(2)
            try:
                ex = int(r[iex] or 0)
            except ValueError:
                ex = 0
            ops[op] += ex
            if want and op.startswith(want):
                by_line[src_line] += ex
    tot = sum(ops.values())
    print("total warp instructions", tot)
    for op, v in ops.most_common(25):
        print(f"{op:12s} {v:11d} {100 * v / tot:5.1f}%")
    if want:
        t2 = sum(by_line.values())
        print(f"\n{want}* by source line ({t2} total)")
        for k, v in by_line.most_common(20):
            print(f"{v:11d} {100 * v / t2:5.1f}% {k}")


if __name__ == "__main__":
    main()
