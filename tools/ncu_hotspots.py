"""Top source lines by warp-stall samples for one kernel of an ncu
`--page source --csv` export.   python tools/ncu_hotspots.py SRC.csv KERNEL [N]"""
import collections
import csv
import sys


def main():
    path, kern = sys.argv[1], sys.argv[2]
    top_n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    rows = list(csv.reader(open(path)))
    cur_file = cur_fn = hdr = None
    agg = collections.Counter()
    stalls = collections.defaultdict(collections.Counter)
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file, hdr = r[1].split("/")[-1], None
            continue
        if len(r) == 2 and r[0] == "Function Name":
            cur_fn = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and cur_fn and kern in cur_fn and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            try:
                n, ln = int(d["Warp Stall Sampling (All Samples)"] or 0), int(d["Line No"])
            except ValueError:
                continue
            agg[(cur_file, ln)] += n
            for k, v in d.items():
                if k.startswith("stall_") and "Not Issued" not in k:
                    try:
                        stalls[(cur_file, ln)][k[6:]] += int(v or 0)
                    except ValueError:
                        pass
    tot = sum(agg.values())
    print("total samples", tot)
    for k, v in agg.most_common(top_n):
        top = ", ".join(f"{a} {b}" for a, b in stalls[k].most_common(3))
        print(f"{v:6d} {100 * v / tot:5.1f}% {k[0]}:{k[1]:<5d} | {top}")
    tots = collections.Counter()
    for k in stalls:
        tots.update(stalls[k])
    print("by reason:", tots.most_common(10))


if __name__ == "__main__":
    main()
