"""Aggregate an ncu source-page CSV (--print-source sass) by CUDA source line,
using `nvdisasm -g` line annotations of the same cubin.

  python tools/sass_lines.py <ncu_sass.csv> <nvdisasm -g output> <kernel symbol prefix>
"""
import collections
import csv
import re
import sys


def main(csv_path, sass_path, kprefix, top=60):
    L = open(sass_path).read().splitlines()
    start = [i for i, l in enumerate(L) if l.startswith(kprefix)][0]
    lines, fn, cur = [], "kernel", None
    for l in L[start:]:
        m = re.search(r'\.type\s+\$\S+\$(\S+),@function', l)
        if m:
            fn = m.group(1)[-40:]
            continue
        if re.search(r'\.type\s+\S+,@object', l):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split('/')[-1], int(m.group(2)))
            continue
        if re.search(r'/\*[0-9a-f]{4,}\*/', l):
            lines.append((fn, cur))
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    data = []
    for r in rows[2:]:  # first kernel section only
        if len(r) < len(hdr):
            break
        data.append(r)
    ia = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    cols = ["stall_no_inst", "stall_long_sb", "stall_wait", "stall_short_sb", "stall_math",
            "stall_branch_resolving", "stall_mio", "stall_lg"]
    ic = [hdr.index(c) for c in cols]
    num = lambda v: int(v) if v.strip() else 0
    tot = sum(num(r[ia]) for r in data)
    agg = collections.defaultdict(lambda: [0, 0] + [0] * len(cols))
    for (fn, ln), r in zip(lines, data):
        a = agg[ln]
        a[0] += num(r[ia])
        a[1] += num(r[ie])
        for k, c in enumerate(ic):
            a[2 + k] += num(r[c])
    print(f"{'line':28s} {'samp%':>6s} {'exec':>12s} " + " ".join(c[6:12] for c in cols))
    for ln, a in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{str(ln):28s} {100 * a[0] / tot:6.2f} {a[1]:12d} " +
              " ".join(f"{x / max(a[0], 1):6.2f}" for x in a[2:]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], *(int(x) for x in sys.argv[4:]))
