"""Docking quality of sweep-v1 against the reference ascent on the same
ligands, conformers, seeds and pocket (C2 workload prefix, analytic pocket):
per ligand, the best survivor rescore of our GPU dock (each survivor pose
re-scored by the reference's FP64 rescore, so grid mode is judged by the
analytic score too) vs the reference's dock() + rescore + filter_poses.

  python tools/quality_vs_reference.py [n_ligands] [threads] [--grid] [--ref-only]

The reference arm's per-ligand results are cached in
tests/golden/quality_ref_<n>.json (the reference's own dock() output on
these inputs; --ref-only computes and writes it without a GPU).

Prints one JSON line: mean / median of (ours - reference) best rescore, the
fraction of ligands where ours >= reference, and both wall times."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def ref_lig(R, lib, i):
    import bench
    from paper_2304_09953_b200.chem import random_smiles
    ao, _, _ = lib.offsets()
    lg = R.RefLigand(random_smiles(bench.CORPUS_SEED, int(lib.ids[i][1:])), iterations=-1)
    lg.set_coords(lib.coords[ao[i]:ao[i + 1]])
    return lg


def ref_arm(lib, pocket, prm, threads, cache):
    """The reference's dock() + rescore + filter_poses + best on these
    ligands (same conformer bytes and seeds), written to `cache`."""
    import paper_2304_09953_b200 as V
    from oracle import ref as R
    rp = R.RefPocket(V.pocket_to_json(pocket))
    ligs = [ref_lig(R, lib, i) for i in range(len(lib))]
    t0 = time.perf_counter()
    kept, best = R.dock_best_many(ligs, rp, prm.restarts, prm.diversity_delta,
                                  [int(s) for s in lib.seeds], 500, prm.keep_top, prm.min_score,
                                  threads)
    t_ref = time.perf_counter() - t0
    with open(cache, "w") as f:
        json.dump({"ids": list(lib.ids), "best": [float(b) if k > 0 else None
                                                 for k, b in zip(kept, best)],
                   "ref_s": round(t_ref, 2), "threads": threads,
                   "knobs": "bench.params(): R=30, delta 1.0, keep_top 4, min_score -5, "
                            "ls_max_steps 500; bench.make_pocket() analytic"}, f)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n = int(args[0]) if args else 64
    threads = int(args[1]) if len(args) > 1 else (os.cpu_count() or 1)
    grid = "--grid" in sys.argv
    import bench
    import paper_2304_09953_b200 as V
    from oracle import ref as R
    from paper_2304_09953_b200.chem import random_smiles
    lib_all, _, _ = bench.build_workload(max(4 * n, 64), 0, 1, threads)
    sel = list(range(0, len(lib_all), len(lib_all) // n))[:n]
    lib = lib_all.subset(sel)
    lib.seeds = lib_all.seeds[sel]
    pocket = bench.make_pocket()
    prm = bench.params()
    cache = os.path.join(ROOT, "tests", "golden", f"quality_ref_{n}.json")
    if "--ref-only" in sys.argv or not os.path.exists(cache):
        ref_arm(lib, pocket, prm, threads, cache)
        if "--ref-only" in sys.argv:
            return
    with open(cache) as f:
        c = json.load(f)
    assert c["ids"] == list(lib.ids), "reference cache is for other ligands"
    ref = np.array([np.nan if v is None else v for v in c["best"]], np.float64)
    eng = V.Engine(0)
    eng.set_pocket(pocket, grid_spacing=0.4 if grid else 0.0, grid_pad=2.0)
    t0 = time.perf_counter()
    res = eng.dock_host(lib, prm)
    t_gpu = time.perf_counter() - t0
    ours = np.where(res.n_surv > 0, res.best.astype(np.float64), np.nan)
    ours_ref_scored = np.full(len(lib), np.nan)  # our poses re-scored by the reference
    # the reference arm: same conformer bytes, same dock seeds, its own ascent
    rp = R.RefPocket(V.pocket_to_json(pocket))
    ao, _, _ = lib.offsets()
    ligs = [ref_lig(R, lib, i) for i in range(len(lib))]
    surv = {i: [(np.array(p.translation, np.float64), np.array(p.rotation, np.float64),
                 np.array(p.torsions, np.float64)) for p in res.poses(i, int(lib.n_tors[i]), "surv")]
            for i in range(len(lib))}
    t_ref_gpu = 0.0
    if "--refine" in sys.argv:
        # the reference ascent on the GPU from every survivor (refine.py)
        from paper_2304_09953_b200.refine import ascend_poses_device as ascend_poses
        pl = [i for i in range(len(lib)) for _ in surv[i]]
        T3 = [p[0] for i in range(len(lib)) for p in surv[i]]
        Q4 = [p[1] for i in range(len(lib)) for p in surv[i]]
        TH = np.concatenate([p[2] for i in range(len(lib)) for p in surv[i]] or [np.zeros(0)])
        t1 = time.perf_counter()
        rt, rq, rtor, _, _ = ascend_poses(eng, lib, pl, T3, Q4, TH, max_steps=500)
        t_ref_gpu = time.perf_counter() - t1
        k, off = 0, 0
        for i in range(len(lib)):
            new = []
            for p in surv[i]:
                T = len(p[2])
                new.append((rt[k], rq[k], rtor[off:off + T]))
                k += 1
                off += T
            surv[i] = new
    for i in range(len(lib)):
        vals = [ligs[i].rescore(rp, t, q, th) for (t, q, th) in surv[i]]
        if vals:
            ours_ref_scored[i] = max(vals)
    t_ref = c["ref_s"]
    both = ~np.isnan(ours_ref_scored) & ~np.isnan(ref)
    d = ours_ref_scored[both] - ref[both]  # both sides scored by the reference's FP64 rescore
    out = {"ligands": len(lib), "compared": int(both.sum()), "grid": grid,
           "ours_only": int((~np.isnan(ours) & np.isnan(ref)).sum()),
           "ref_only": int((np.isnan(ours) & ~np.isnan(ref)).sum()),
           "mean_delta": float(d.mean()) if d.size else None,
           "median_delta": float(np.median(d)) if d.size else None,
           "frac_ours_ge_ref": float((d >= -1e-9).mean()) if d.size else None,
           "mean_ours": float(np.nanmean(ours_ref_scored)), "mean_ours_own_score": float(np.nanmean(ours)),
           "mean_ref": float(np.nanmean(ref)), "polish": int(prm.polish),
           "refined_by_gpu_ascent": "--refine" in sys.argv, "refine_s": round(t_ref_gpu, 3),
           "gpu_s": round(t_gpu, 3), "ref_s": round(t_ref, 2), "ref_threads": threads}
    print(json.dumps(out))
    eng.close()


if __name__ == "__main__":
    main()
