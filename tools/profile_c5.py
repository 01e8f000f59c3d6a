"""Small fixed C5 workload for ncu captures of the rescoring kernel: the
bench's C5 library (first N ligands), a C2-knob dock on 0.4 A maps, then
vs_rescore_survivors twice on the 0.2 A maps over the 30 A box.

  ncu --set full -k regex:vs_rescore_kernel -s 2 -c 2 -o gpurun_out/prof_c5 \\
      python tools/profile_c5.py --ligands 20000
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ligands", type=int, default=20000)
    args = ap.parse_args()
    import torch
    import bench
    import paper_2304_09953_b200 as V
    lib = bench.c5_library(args.ligands, 0, 1, os.cpu_count() or 1)
    pocket = bench.make_pocket()
    eng = V.Engine(0)
    eng.set_pocket(pocket, grid_spacing=0.4, grid_pad=2.0)
    prm = bench.params()
    eng.upload(lib, [(1, 41, 0, 11), (60, 81, 11, 21)])
    eng.dock(prm)
    eng.fetch()
    box = V.Pocket(pocket.sites, (-15.0, -15.0, -15.0), (15.0, 15.0, 15.0), pocket.clash_radius,
                   pocket.clash_penalty)
    eng.set_pocket(box, grid_spacing=0.2, grid_pad=2.0)
    g = torch.zeros(len(lib) * prm.keep_top, dtype=torch.float32, device="cuda")
    r = torch.zeros_like(g)
    for _ in range(2):
        eng.rescore_survivors(g.data_ptr(), r.data_ptr())
    torch.cuda.synchronize()
    print(f"ligands={len(lib)} rescored; mean geo {float(g[g != 0].mean()):.4f}")
    eng.close()


if __name__ == "__main__":
    main()
