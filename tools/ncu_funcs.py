"""Per-function sample / instruction breakdown of an ncu source-page CSV
(--print-source sass) for a kernel whose subroutines nvdisasm names.

  python tools/ncu_funcs.py <ncu_sass.csv> <nvdisasm -g output> <kernel symbol prefix>
"""
import collections
import csv
import re
import sys

KEYS = ['chain_coop', 'draw_start', 'eval_rigid', 'flex_phase', 'keep_phase', 'start_phase',
        'sweep_phase', 'finish_phase', 'diverse_from_kept', 'pose_coop', 'trig_reduction',
        'div_rn_f64', 'dsqrt', 'sqrt_rn_f32', 'div_rn_noftz', 'off_grid']


def main(csv_path, sass_path, kprefix):
    L = open(sass_path).read().splitlines()
    start = [i for i, l in enumerate(L) if l.startswith(kprefix)][0]
    ins, fn = [], 'kernel'
    for l in L[start:]:
        m = re.search(r'\.type\s+\$\S+\$(\S+),@function', l)
        if m:
            fn = next((k for k in KEYS if k in m.group(1)), m.group(1)[-30:])
            continue
        if re.search(r'\.type\s+\S+,@object', l):
            break
        if re.search(r'/\*[0-9a-f]{4,}\*/', l):
            ins.append(fn)
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    data = []
    for r in rows[2:]:  # first kernel section only
        if len(r) < len(hdr):
            break
        data.append(r)
    ia = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    ino = hdr.index("stall_no_inst")
    ilsb = hdr.index("stall_long_sb")
    agg = collections.defaultdict(lambda: [0, 0, 0, 0, 0])
    num = lambda v: int(v) if v.strip() else 0
    for f, r in zip(ins, data):
        a = agg[f]
        a[0] += 1
        a[1] += num(r[ia])
        a[2] += num(r[ie])
        a[3] += num(r[ino])
        a[4] += num(r[ilsb])
    tot = sum(a[1] for a in agg.values())
    te = sum(a[2] for a in agg.values())
    print(f"{'function':20s} {'instrs':>6s} {'samp%':>6s} {'exec%':>6s} {'no_inst':>7s} {'long_sb':>7s}")
    for f, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{f:20s} {a[0]:6d} {100 * a[1] / tot:6.1f} {100 * a[2] / te:6.1f} "
              f"{a[3] / max(a[1], 1):7.2f} {a[4] / max(a[1], 1):7.2f}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
