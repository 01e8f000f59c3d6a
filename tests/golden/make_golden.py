"""Regenerate the golden fixtures from the UNMODIFIED reference library
(oracle/_ref/libvsref.so, compiled from /root/reference by oracle/Makefile).

    python tests/golden/make_golden.py

Writes (small, committed):
  scores.npz   reference conformers (embed_3d) + seeded random poses with
               dock::geometric_score / dock::rescore on data/pocket.json
  rng.npz      Rng u64 streams and uniform/normal draws (rng.hpp)
  buckets.json BatchQueue replay of the run_campaign dock stage
  rank.json    rank_ligands / filter_poses outputs
pocket.json is the reference's proj/data/pocket.json, copied verbatim.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref as R  # noqa: E402


def main():
    pj = open(os.path.join(HERE, "pocket.json")).read()
    rp = R.RefPocket(pj)
    rng = np.random.default_rng(20241018)
    smis, seeds, coords, n_atoms, n_tors, classes, axes = [], [], [], [], [], [], []
    pose_lig, T, Q, TH, geo, resc = [], [], [], [], [], []
    i = 0
    while len(smis) < 40:
        s = R.random_smiles(99, i)
        i += 1
        lig = R.RefLigand(s, 1000 + i)
        if lig.n_atoms > 40 or lig.n_tors > 8:
            continue
        k = len(smis)
        smis.append(s)
        seeds.append(1000 + i)
        coords.append(lig.coords())
        n_atoms.append(lig.n_atoms)
        n_tors.append(lig.n_tors)
        classes.append(lig.classes())
        axes.append(lig.axes())
        for _ in range(10):
            t = rng.uniform(-5, 5, 3).astype(np.float32).astype(np.float64)
            q = rng.normal(size=4)
            q = (q / np.linalg.norm(q)).astype(np.float32).astype(np.float64)
            th = rng.uniform(-np.pi, np.pi, lig.n_tors).astype(np.float32).astype(np.float64)
            pose_lig.append(k)
            T.append(t)
            Q.append(q)
            TH.extend(th)
            geo.append(lig.geometric_score(rp, t, q, th))
            resc.append(lig.rescore(rp, t, q, th))
    np.savez_compressed(
        os.path.join(HERE, "scores.npz"), smiles=np.array(smis), embed_seeds=np.array(seeds),
        coords=np.concatenate(coords), n_atoms=np.array(n_atoms), n_tors=np.array(n_tors),
        classes=np.concatenate(classes),
        axis_a=np.array([a for ax in axes for (a, b, m) in ax], np.int32),
        axis_b=np.array([b for ax in axes for (a, b, m) in ax], np.int32),
        moving_count=np.array([len(m) for ax in axes for (a, b, m) in ax], np.int32),
        moving=np.array([v for ax in axes for (a, b, m) in ax for v in m], np.int32),
        pose_lig=np.array(pose_lig), t=np.array(T), q=np.array(Q), tors=np.array(TH),
        geo=np.array(geo), resc=np.array(resc))

    streams = {}
    for seed, path in ((0, []), (2024, [2, 7]), (99, [5]), (2**63 + 11, [1, 2, 3])):
        streams[f"u64_{seed}_{'_'.join(map(str, path))}"] = R.rng_u64(seed, path, 32)
    kinds = [0, 1, 2] * 20
    lo = [0.0, -6.0, 0.0] * 20
    hi = [1.0, 6.0, 1.0] * 20
    streams["draws_kinds"] = np.array(kinds)
    streams["draws_lo"] = np.array(lo)
    streams["draws_hi"] = np.array(hi)
    streams["draws_2024_2_7"] = R.rng_draws(2024, [2, 7], kinds, lo, hi)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **streams)

    classes = [(1, 24, 0, 6), (1, 24, 6, 32), (24, 48, 0, 6), (24, 48, 6, 32), (48, 96, 0, 6),
               (48, 96, 6, 32)]
    r2 = np.random.default_rng(5)
    atoms = r2.integers(1, 110, 2500).tolist()
    rot = r2.integers(0, 40, 2500).tolist()
    ir, batches = R.bucket_replay(atoms, rot, classes, 4096.0, 256.0, 2.0, 8.0)
    json.dump({"classes": classes, "atoms": atoms, "rot": rot, "cap": 4096.0, "fixed": 256.0,
               "per_atom": 2.0, "per_rot": 8.0, "in_range": [bool(v) for v in ir],
               "batches": batches}, open(os.path.join(HERE, "buckets.json"), "w"))

    cases = []
    for _ in range(50):
        n = int(r2.integers(0, 20))
        sc = np.round(r2.normal(size=n), 1).tolist()
        kt = int(r2.integers(0, 6))
        ms = float(np.round(r2.normal(), 2))
        ids = {f"MOL{int(v)}": s for v, s in zip(r2.integers(0, 200, n), sc)}
        cases.append({"scores": sc, "keep_top": kt, "min_score": ms,
                      "filter": R.filter_poses(sc, kt, ms), "ids": ids,
                      "rank": R.rank_ligands(ids)})
    json.dump(cases, open(os.path.join(HERE, "rank.json"), "w"))
    print("golden fixtures written")


if __name__ == "__main__":
    main()
