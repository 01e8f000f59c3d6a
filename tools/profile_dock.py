"""Small fixed workload for ncu captures of the dock kernel: the bench's C2
library (first N ligands), pocket and knobs; one warm-up dock then one
profiled dock (one persistent launch).

  ncu --set full --import-source on -k regex:vs_dock_kernel -s 1 -c 1 \
      -o gpurun_out/prof python tools/profile_dock.py --ligands 4000
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ligands", type=int, default=4000)
    ap.add_argument("--analytic", action="store_true")
    args = ap.parse_args()
    import bench
    import paper_2304_09953_b200 as V
    lib, _, _ = bench.build_workload(args.ligands, 0, 1, os.cpu_count() or 1)
    eng = V.Engine(0)
    eng.set_pocket(bench.make_pocket(), grid_spacing=0.0 if args.analytic else 0.4, grid_pad=2.0)
    eng.upload(lib)
    prm = bench.params()
    for _ in range(2):
        eng.dock(prm)
        ms = eng.last_dock_ms()
    ph = {k: round(v, 2) for k, v in eng.phase_ms_ex().items()}
    print(f"ligands={len(lib)} dock_ms={ms:.3f} lig/s={len(lib) / ms * 1e3:.1f} phases={ph}")
    eng.close()


if __name__ == "__main__":
    main()
