"""Static SASS opcode counts per outermost source line range of one kernel.

    nvdisasm --print-line-info-inline -c X.cubin > X.lsass
    python tools/sass_regions.py X.lsass KERNEL_SUBSTR [a-b ...]

Each instruction is attributed to the OUTERMOST ws_kernels.cuh line of its
inline chain; ranges a-b select kernel-body lines (e.g. the x-pass loop).
"""
import collections
import re
import sys


def main():
    path, kern = sys.argv[1], sys.argv[2]
    ranges = [tuple(int(x) for x in r.split("-")) for r in sys.argv[3:]]
    cur_fn = None
    line = None
    per = collections.defaultdict(collections.Counter)
    for ln in open(path):
        m = re.match(r"\.text\.(\S+):", ln)
        if m:
            cur_fn = m.group(1)
            continue
        if cur_fn is None or kern not in cur_fn:
            continue
        if ln.lstrip().startswith("//## File"):
            outer = re.findall(r'ws_kernels\.cuh", line (\d+)', ln)
            line = int(outer[-1]) if outer else line
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", ln)
        if m and line is not None:
            for a, b in ranges or [(0, 10**9)]:
                if a <= line <= b:
                    per[(a, b)][m.group(1)] += 1
    for (a, b), c in per.items():
        tot = sum(c.values())
        print(f"lines {a}-{b}: {tot} instructions")
        print("  " + ", ".join(f"{k} {v}" for k, v in c.most_common(30)))


if __name__ == "__main__":
    main()
