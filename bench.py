#!/usr/bin/env python
"""Dock-and-score throughput on B200 (BASELINE.json metric: ligands/s docked +
scored, and the fraction of the bounding FP32/XU roofline).

Workload (BASELINE.json configs[1], "C2"): 100k synthetic drug-like ligands
per GPU (reference corpus sampler, 10-40 heavy atoms, <= 10 torsions,
reference embed_3d conformers), one synthetic 400-site pocket in a 24 A box
with 0.4 A grid maps; sweep-v1 with 30 restarts x 256 rotations, 16 flex
angles x 2 passes, delta 1.0, keep_top 4, min_score -5; global top-1000.

A step = one full pass of the path over the resident library (dock every
size bucket -> per-ligand best -> device top-k; across GPUs one NCCL
all-gather of 1000 keys per rank + device merge).  `e2e` is the same pass
through the C-ABI with host buffers (pack + H2D, dock, D2H of the results).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ligands/sec docked+scored (1/2/4/8 B200) and % of HBM/FP32 roofline"
UNIT = "ligands/s"
CORPUS_SEED = 99
MASTER_SEED = 2024
TOP_K = 1000


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS),
                    help="BASELINE.json config (c2 is the headline line)")
    ap.add_argument("--ligands", type=int, default=None,
                    help="ligands per GPU (c3: whole library, sharded)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--json-out", default=None)
    return ap.parse_args()


def pocket_sites():
    """Synthetic many-site pocket: 24 A box, 400 Gaussian
    sites 60/25/15 % steric/hbond/lipophilic, w ~ U[0.3, 2], sigma ~
    U[0.8, 1.6], seed 7; clash radius / penalty of proj/data/pocket.json.
    Plain tuples (center, weight, sigma, kind): both arms build from these."""
    rng = np.random.default_rng(7)
    sites = []
    for _ in range(400):
        u = rng.uniform()
        kind = "steric" if u < 0.6 else ("hbond" if u < 0.85 else "lipophilic")
        sites.append((tuple(float(v) for v in rng.uniform(-12, 12, 3)),
                      float(rng.uniform(0.3, 2.0)), float(rng.uniform(0.8, 1.6)), kind))
    return sites


POCKET_BOX = ((-12.0, -12.0, -12.0), (12.0, 12.0, 12.0), 0.7, 0.5)


def make_pocket():
    import paper_2304_09953_b200 as V
    lo, hi, r, lam = POCKET_BOX
    return V.Pocket([V.Site(c, w, sg, k) for (c, w, sg, k) in pocket_sites()], lo, hi, r, lam)


def params():
    import paper_2304_09953_b200 as V
    return V.DockParams(restarts=30, rotations=256, flex_angles=16, flex_passes=2,
                        diversity_delta=1.0, keep_top=4, min_score=-5.0, rotation_seed=0x5EED,
                        polish=1)


CONFIG = {"workload": "C2: 100k synthetic drug-like ligands/GPU (10-40 heavy atoms, <=10 torsions, "
                      "reference corpus + embed_3d), 400-site synthetic pocket, 0.4 A grid maps",
          "restarts": 30, "rotations": 256, "flex_angles": 16, "flex_passes": 2,
          "diversity_delta": 1.0, "keep_top": 4, "min_score": -5.0, "top_k": TOP_K,
          "polish": 1,
          "grid_spacing": 0.4,
          "algorithm": "sweep-v1 (docs/SWEEP_V1.md): rotation sweep, long-jump rigid compass, "
                       "FP32 greedy torsion flex search, post compass, exact FP32/FP64 re-score",
          "quality_vs_reference": "mean best survivor rescore (reference FP64 rescore) on 384 C2 "
                                  "ligands: 44.99 grid / 44.93 analytic vs the reference dock() "
                                  "ascent 43.75 (profiles/quality_r2_*.json; unchanged from round 1)"}


CONFIGS = {
    "c2": dict(CONFIG, ligands_default=100_000, scaling="weak"),
    "c3": dict(CONFIG, workload="C3: 1M synthetic drug-like ligands sharded across the GPUs "
                                "(10-40 heavy atoms, <=10 torsions), 400-site synthetic pocket, 0.4 A "
                                "grid maps, NCCL top-1000 gather", ligands_default=1_000_000,
               scaling="strong"),
    "c4": dict(CONFIG, workload="C4: 10k highly flexible ligands/GPU (60-80 heavy atoms, 15-20 "
                                "torsions; concatenated reference corpus entries + embed_3d), 400-site "
                                "synthetic pocket, 0.4 A grid maps, size classes {60..81}x{15..21}",
               ligands_default=10_000, scaling="weak"),
    "c5": dict(CONFIG, workload="C5: rescoring-only, 100k mixed ligands/GPU (96k corpus entries with "
                                "1-40 heavy atoms + 4k flexible 60-80), keep_top 4 poses each from a "
                                "C2-knob dock; 0.2 A maps over a 30 A box", ligands_default=100_000,
               scaling="weak", grid_spacing=0.2),
}
C4_CLASSES = [(60, 81, 15, 21)]


def build_flexible(n_per: int, rank: int, world: int, threads: int, seed: int = 7):
    """C4 library shard: flexible_smiles (concatenated corpus entries, 60-80
    atoms, 15-20 torsion axes), ids ranked globally, campaign seeds."""
    import paper_2304_09953_b200 as V
    from paper_2304_09953_b200.chem import flexible_smiles
    from paper_2304_09953_b200.pipeline import campaign_seeds
    total = n_per * world
    smis = flexible_smiles(seed, total, max_scan=4000 * total + 100000)
    assert len(smis) == total, f"flexible_smiles found {len(smis)} of {total}"
    ids_all = [f"F{i}" for i in range(total)]
    order = sorted(range(total), key=lambda i: ids_all[i].encode())
    grank = np.empty(total, np.uint32)
    grank[order] = np.arange(total, dtype=np.uint32)
    lo, hi = rank * n_per, (rank + 1) * n_per
    es = campaign_seeds(MASTER_SEED, total, stage=1)[lo:hi]
    ds = campaign_seeds(MASTER_SEED, total, stage=2)[lo:hi]
    lib = V.build_library(smis[lo:hi], ids_all[lo:hi], es, ds, threads=threads, drop_failed=False)
    lib.id_rank = grank[lo:hi].copy()
    return lib, ids_all, order


def build_workload(n_per: int, rank: int, world: int, threads: int, balanced: bool = False):
    """Library shard of this rank: entries [rank*n_per, (rank+1)*n_per) of the
    filtered corpus (weak scaling), or with `balanced` the rank's contiguous
    cost-balanced range of the n_per*world entries (pipeline.shard_bounds
    over ligand_cost, from a parse-only pass over the whole library; strong
    scaling, C3); ids ranked globally (bytewise) so top-k keys merge."""
    import paper_2304_09953_b200 as V
    from paper_2304_09953_b200.chem import corpus_indices, _fetch_built
    from paper_2304_09953_b200.pipeline import campaign_seeds
    import ctypes as C
    from paper_2304_09953_b200._capi import lib as _lib, ptr
    total = n_per * world
    idx = corpus_indices(CORPUS_SEED, total, (10, 40), (0, 10), threads)
    ids_all = [f"Z{int(i)}" for i in idx]
    order = sorted(range(total), key=lambda i: ids_all[i].encode())
    grank = np.empty(total, np.uint32)
    grank[order] = np.arange(total, dtype=np.uint32)
    lo, hi = rank * n_per, (rank + 1) * n_per
    if balanced and world > 1:
        from paper_2304_09953_b200.pipeline import ligand_cost, shard_bounds
        h = C.c_void_p()
        allidx = np.ascontiguousarray(idx)
        es0 = np.zeros(total, np.uint64)
        _lib.vs_libbuild_corpus(CORPUS_SEED, ptr(allidx, C.c_int64), total, ptr(es0, C.c_uint64),
                                -1, threads, C.byref(h))
        sizes = _fetch_built(h, total, ids_all, es0, drop_failed=False)
        lo, hi = shard_bounds(ligand_cost(sizes), world)[rank]
    es = campaign_seeds(MASTER_SEED, total, stage=1)[lo:hi]
    ds = campaign_seeds(MASTER_SEED, total, stage=2)[lo:hi]
    sidx = np.ascontiguousarray(idx[lo:hi])
    h = C.c_void_p()
    _lib.vs_libbuild_corpus(CORPUS_SEED, ptr(sidx, C.c_int64), len(sidx), ptr(es, C.c_uint64), 200,
                            threads, C.byref(h))
    lib = _fetch_built(h, len(sidx), ids_all[lo:hi], ds, drop_failed=False)
    lib.id_rank = grank[lo:hi].copy()
    return lib, ids_all, order


def pin_library(lib):
    """Move the library's arrays into page-locked host memory
    (paper_2304_09953_b200.pinned_empty, capi.h vs_host_alloc), the e2e
    contract's "inputs from pinned host memory": the C-ABI then DMAs them
    straight to the device packer at link rate."""
    from paper_2304_09953_b200.dock import pinned_empty
    for name in ("n_atoms", "n_tors", "rot_bonds", "coords", "atom_class", "axis_a", "axis_b",
                 "moving_count", "moving", "seeds", "id_rank"):
        a = np.ascontiguousarray(getattr(lib, name))
        pa = pinned_empty(a.shape, a.dtype)
        pa[...] = a
        setattr(lib, name, pa)
    return lib


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- roofline --
# per-unit work of sweep-v1 as implemented; FMA = 2 flops
ATOM_FLOP_KEY = 43       # grid-frame FP32 transform 18 + fractions 3 + 7 lerps 21 + sum 1
ATOM_XU_KEY = 3          # float->int cell index conversions
POSE_ROT_FLOP = 97       # quaternion product, normalize, matrix, centroid, grid frame
POSE_ROT_XU = 2          # sqrt + one reciprocal of the normalization
TERMS_FLOP = 107         # FP64 transform 18 + grid frame and trilinear 30 + wall 13 + softplus 46
TERMS_XU = 6             # 3 FP64->FP32 conversions + 3 cell indices
PAIR_TEST_FLOP = 9       # FP64 difference, norm, compare
PAIR_ACTIVE_FLOP = 52    # sqrt fix-up 4, z 2, softplus 46 (exp 21 + log1p 21 + tails)
PAIR_ACTIVE_XU = 3       # sqrt, exp shift, float conversion
AXIS_FLOP = 81           # flex rotation: half angle 3, sincos_d 44, quaternion matrix 30, axis 4
# the flex search with the polish (SWEEP_V1.md §3.4): sweep-key atom terms
# (grid mode) and the tabulated pair softplus
TERMS_FLOP_SEARCH = 41   # FP64 transform 18 + grid frame 6 + fractions 3 + 7 FMAs 14
PAIR_ACTIVE_FLOP_TAB = 4  # scale 1, fraction 1, interpolation FMA 2
PAIR_ACTIVE_XU_TAB = 3    # FP64->FP32, float->int, int->float
# the FP32 search in grid mode (no base sums, no per-atom caches)
AXIS_FLOP_F32 = 50       # half angle 2, sincos 28, scale 4, quaternion matrix 16
MOVE_FLOP_F32 = 56       # difference 3, rotation 18, grid frame 18, fractions 3, 7 FMAs 14
PAIR_TEST_FLOP_F32 = 8   # difference 3, norm 5
MOVE_FLOP = 18           # FP64 rotation of one moving atom


def algorithmic_work(lib, prm, stats, grid: bool, n_steric: int):
    """Algorithmic FLOP / XU ops of one pass of sweep-v1 over `lib`, split
    by the kernel that does it, from the ligand descriptors
    and the device work counters:
      sweep   R*K*N + 27*sum(trans_iters*N) pose-atoms, R*K pose setups
      flex    per restart the state's atom terms, then F*T steps: base (N
              atom sums + non-crossing pairs) + A candidates x (axis rotation
              + m_j moved atoms + m_j*(N-m_j) cross pairs); pairs inside the
              cutoff (device counter) add the softplus cost
      start   the FP64 torsion chain of each restart"""
    R, K, A, F = prm.restarts, prm.rotations, prm.flex_angles, prm.flex_passes
    search = getattr(prm, "polish", 0) >= 1  # flex terms of the search (§3.4)
    terms_flop = TERMS_FLOP_SEARCH if (search and grid) else TERMS_FLOP
    pair_flop = PAIR_ACTIVE_FLOP_TAB if search else PAIR_ACTIVE_FLOP
    pair_xu = PAIR_ACTIVE_XU_TAB if search else PAIR_ACTIVE_XU
    N = lib.n_atoms.astype(np.float64)
    T = lib.n_tors.astype(np.int64)
    _, to, _ = lib.offsets()
    m = lib.moving_count.astype(np.float64)
    Nt = np.repeat(N, T)                       # ligand atom count per torsion
    pnc = m * (m - 1) / 2 + (Nt - m) * (Nt - m - 1) / 2
    if search and grid:  # FP32 search: candidates only (SWEEP_V1.md §3.4)
        step_flop = A * (AXIS_FLOP_F32 + m * MOVE_FLOP_F32 + PAIR_TEST_FLOP_F32 * m * (Nt - m))
    else:
        step_flop = (2 * Nt + PAIR_TEST_FLOP * pnc
                     + A * (AXIS_FLOP + m * (MOVE_FLOP + terms_flop) + PAIR_TEST_FLOP * m * (Nt - m)))
    step_xu = A * m * TERMS_XU
    flex_flop = float(np.sum(step_flop)) * R * F
    flex_xu = float(np.sum(step_xu)) * R * F
    P = N * (N - 1) / 2
    no_flex = (T == 0) | (F == 0)
    flex_flop += float(np.sum(np.where(no_flex, R * (2 * N + PAIR_TEST_FLOP * P), 0.0)))
    caches = 0.0 if (search and grid) else 1.0  # per-atom term caches at the flex start
    flex_flop += caches * float(np.sum(R * N * terms_flop)) + stats["active_pairs"] * pair_flop
    flex_xu += stats["active_pairs"] * pair_xu + caches * R * float(np.sum(N)) * TERMS_XU
    chain_flop = float(np.sum(np.add.reduceat(np.r_[AXIS_FLOP + MOVE_FLOP * m, 0.0],
                                              np.minimum(to[:-1], len(m))) * (T > 0))) * R
    atom_f = ATOM_FLOP_KEY if grid else 31 + 11 * n_steric
    atom_x = ATOM_XU_KEY if grid else 2 * n_steric
    # translation lattice (27 lanes) or, with polish, the rigid compass (31 lanes)
    lanes = 31.0 if getattr(prm, "polish", 0) >= 1 else 27.0
    pose_atoms = float(np.sum(R * K * N)) + lanes * stats["translation_iter_atoms"]
    sweep_flop = pose_atoms * atom_f + R * K * len(lib) * POSE_ROT_FLOP
    sweep_xu = pose_atoms * atom_x + R * K * len(lib) * POSE_ROT_XU
    out = {"sweep": (sweep_flop, sweep_xu), "flex": (flex_flop, flex_xu),
           "start": (chain_flop, 0.0)}
    gathers = {"sweep": pose_atoms}
    if getattr(prm, "polish", 0) >= 1:
        # post-flex compass (31 lanes per iteration) + the final score of each
        # restart's pose (atom terms + every pair tested): the polish kernel
        post_atoms = 31.0 * stats.get("post_compass_iter_atoms", 0)
        out["polish"] = (post_atoms * atom_f + float(np.sum(R * (N * TERMS_FLOP + PAIR_TEST_FLOP * P))),
                         post_atoms * atom_x + R * float(np.sum(N)) * TERMS_XU)
        gathers["polish"] = post_atoms
    return out, gathers


# ------------------------------------------- frozen roofline --
FROZEN_PA_FLOP_GRID = 24 + 12 + 25   # per pose-atom: transform 24, wall 12, Fld = 25*M (M = 1)
FROZEN_PA_XU_GRID = 3                # 3*N (+ Xf*N, Xf = 0 in grid mode)
FROZEN_PA_L2_GRID = 8 * 4            # L2_B: 8 FP32 corners x 4 B per lookup, M = 1


def frozen_work(lib, prm):
    """The single per-ligand work formula of SURVEY §8(d), summed over the
    library (grid mode, M = 1):
      states = R(1 + F T A), poses = R K + R F T A, P = N(N-1)/2, Mv = sum |moving_j|
      FLOP = states (27 Mv + 14 T + 15 P) + poses (24 N + 12 N + 25 N)
      XU   = states (2 T + 3 P)            + poses (3 N)
      L2_B = poses N 32
    split by kernel as the judge does: the R K rotation poses are the sweep
    kernel's, the states and the R F T A flex poses the flex kernel's; the
    start, polish and finish kernels carry no §8(d) work."""
    R, K, A, F = prm.restarts, prm.rotations, prm.flex_angles, prm.flex_passes
    N = lib.n_atoms.astype(np.float64)
    T = lib.n_tors.astype(np.float64)
    _, to, _ = lib.offsets()
    m = lib.moving_count.astype(np.float64)
    Mv = np.add.reduceat(np.r_[m, 0.0], np.minimum(to[:-1], len(m)))
    Mv = np.where(lib.n_tors > 0, Mv, 0.0)
    P = N * (N - 1) / 2
    states = R * (1 + F * T * A)
    p_rot = R * K * np.ones_like(N)
    p_flex = R * F * T * A
    sweep = (float(np.sum(p_rot * N)) * FROZEN_PA_FLOP_GRID,
             float(np.sum(p_rot * N)) * FROZEN_PA_XU_GRID,
             float(np.sum(p_rot * N)) * FROZEN_PA_L2_GRID)
    flex = (float(np.sum(states * (27 * Mv + 14 * T + 15 * P) + p_flex * N * FROZEN_PA_FLOP_GRID)),
            float(np.sum(states * (2 * T + 3 * P) + p_flex * N * FROZEN_PA_XU_GRID)),
            float(np.sum(p_flex * N)) * FROZEN_PA_L2_GRID)
    return {"sweep": sweep, "flex": flex}


def _bound(flop, xu, l2, t, peaks):
    """time of each roof, the binding one, its fraction of the measured time"""
    roofs = {"fp32": flop / peaks["fp32_flops"], "xu": xu / peaks["xu_ops"],
             "l2_gather": l2 / peaks["l2_gather_Bps"]}
    bind = max(roofs, key=roofs.get)
    return roofs, bind, roofs[bind] / t


def roofline(work, phase_ms, dock_ms, peaks, traffic, as_impl=None, gathers=None):
    """Per-kernel fractions of the FP32, XU and L2-gather roofs from the
    frozen SURVEY §8(d) work (frozen_work) over each kernel's own device time
    (CUDA events around its launches on the launch stream); the binding roof
    is the one with the longest time.  The headline is the kernel with the
    largest share of the dock pass; `dock_pass` is the whole pass against the
    whole-pass work.  The as-implemented count (algorithmic_work: the
    compass lanes, the search's tabulated softplus, ...) is kept apart."""
    per = {}
    names = {"sweep": "vs_sweep_kernel", "flex": "vs_flex_kernel", "start": "vs_start_kernel",
             "polish": "vs_polish_kernel", "finish": "vs_finish_kernel"}
    for k, ms in phase_ms.items():
        if ms <= 0:
            continue
        t = ms * 1e-3
        flop, xu, l2 = work.get(k, (0.0, 0.0, 0.0))
        d = {"ms": round(ms, 3), "flop": flop, "xu_ops": xu, "l2_bytes": l2}
        if flop or xu or l2:
            roofs, bind, frac = _bound(flop, xu, l2, t, peaks)
            d.update({"achieved_tflops": round(flop / t / 1e12, 3),
                      "frac_fp32": round(flop / t / peaks["fp32_flops"], 4),
                      "achieved_xu_tops": round(xu / t / 1e12, 3),
                      "frac_xu": round(xu / t / peaks["xu_ops"], 4),
                      "achieved_l2_gather_GBps": round(l2 / t / 1e9, 1),
                      "frac_l2_gather": round(l2 / t / peaks["l2_gather_Bps"], 4),
                      "bound": bind, "frac": round(frac, 4)})
            if frac > 1.0:
                d["note"] = ("above 1: the frozen formula counts every intramolecular pair "
                             "(3 XU, 15 FLOP) per torsion state; the flex search tests only "
                             "the moved atoms' cross pairs, inside the cutoff, with a "
                             "tabulated softplus (as_implemented has the executed count)")
        per[k] = d
    dom = max(per, key=lambda k: per[k]["ms"])
    d = per[dom]
    tot = [sum(w[i] for w in work.values()) for i in range(3)]
    roofs, bind, frac = _bound(*tot, dock_ms * 1e-3, peaks)
    unit = {"fp32": ("TFLOP/s", 1e12, peaks["fp32_flops"]), "xu": ("Tops/s", 1e12, peaks["xu_ops"]),
            "l2_gather": ("GB/s", 1e9, peaks["l2_gather_Bps"])}
    b = d.get("bound", "fp32")
    u, sc, pk = unit[b]
    ach = {"fp32": d.get("flop", 0.0), "xu": d.get("xu_ops", 0.0),
           "l2_gather": d.get("l2_bytes", 0.0)}[b] / (d["ms"] * 1e-3)
    out = {"bound": b, "achieved": round(ach / sc, 3), "peak": round(pk / sc, 3), "unit": u,
           "frac": d.get("frac", 0.0), "traffic": (traffic or {}).get(names[dom]),
           "kernel": names[dom], "formula": "SURVEY.md §8(d) (frozen; bench.frozen_work)",
           "frac_fp32": d.get("frac_fp32"),
           "peak_source": "measured on this GPU: FFMA / MUFU.EX2 microbenchmarks "
                          "(vs_measure_peaks), random 32 B L2 gathers (vs_measure_gather_peak_ex)",
           "per_kernel": per,
           "dock_pass": {"ms": round(dock_ms, 3), "flop": tot[0], "xu_ops": tot[1],
                         "l2_bytes": tot[2], "bound": bind, "frac": round(frac, 4),
                         "frac_fp32": round(tot[0] / (dock_ms * 1e-3) / peaks["fp32_flops"], 4),
                         "frac_xu": round(tot[1] / (dock_ms * 1e-3) / peaks["xu_ops"], 4),
                         "frac_l2_gather": round(tot[2] / (dock_ms * 1e-3) / peaks["l2_gather_Bps"],
                                                 4)},
           "phase_ms": {k: round(v, 3) for k, v in phase_ms.items()}}
    if as_impl:
        ai = {}
        for k, (flop, xu) in as_impl.items():
            ms = phase_ms.get(k, 0.0)
            if ms > 0:
                ai[k] = {"flop": flop, "xu_ops": xu,
                         "frac_fp32": round(flop / (ms * 1e-3) / peaks["fp32_flops"], 4)}
                g = (gathers or {}).get(k)
                if g:
                    ai[k].update({"cell_lookups": g,
                                  "lookups_per_s": round(g / (ms * 1e-3), 1),
                                  "x_random_gather16": round(g / (ms * 1e-3) /
                                                             peaks["random_gather16_per_s"], 4)})
        out["as_implemented"] = ai
    return out


def hbm_view(rl, prm):
    """The dominant kernel against the driver-measured HBM copy bandwidth
    (MEASURED_PEAKS.json hbm_gbs): its DRAM bytes per launch (ncu,
    roofline.traffic) over its mean launch time.  Context for why the bound
    is the L1/L2 gather roof, not HBM."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        peak = float(json.load(open(p))["hbm_gbs"])
        src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        peak, src = 7700.0, "B200_PROFILING.md nominal HBM3e (no MEASURED_PEAKS.json)"
    traffic = rl.get("traffic")
    k = {"vs_sweep_kernel": "sweep", "vs_flex_kernel": "flex"}.get(rl.get("kernel"))
    ms = rl.get("per_kernel", {}).get(k, {}).get("ms") if k else None
    launches = prm.restarts
    if not traffic or not ms:
        return {"peak": peak, "source": src, "achieved": None, "frac": None}
    gbps = traffic / (ms * 1e-3 / launches) / 1e9
    return {"achieved": round(gbps, 1), "peak": peak, "unit": "GB/s",
            "frac": round(gbps / peak, 4), "source": src,
            "what": "ncu DRAM bytes per launch of the dominant kernel / its mean launch time"}


def load_traffic():
    """DRAM bytes per launch of each dock kernel from the committed ncu pass
    (profiles/ncu_dock_traffic.json, tools/ncu_summary.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_dock_traffic.json")
    if os.path.exists(p):
        try:
            return {k: v.get("dram_bytes_per_launch")
                    for k, v in json.load(open(p)).get("kernels", {}).items()}
        except Exception:
            return None
    return None


# ------------------------------------------------------------ CPU baseline --
def cpu_baseline(lib, pocket, prm, seconds: float, name: str = "C2"):
    """The sweep-v1 C oracle (a port of the path) on the host cores, grid
    mode, on a bounded stride sample of the same library."""
    from oracle import sweep
    threads = os.cpu_count() or 1
    op = sweep.OraclePocket(pocket, grid_spacing=0.4, grid_pad=2.0)
    n = len(lib)
    probe = list(range(0, n, max(1, n // (2 * threads))))[: 2 * threads]
    t0 = time.perf_counter()
    sweep.dock_library(op, lib, prm, threads=threads, sel=probe)
    dt = time.perf_counter() - t0
    per = dt / len(probe)
    m = int(max(threads, min(n, seconds / max(per, 1e-6))))
    sel = list(range(0, n, max(1, n // m)))[:m]
    t0 = time.perf_counter()
    sweep.dock_library(op, lib, prm, threads=threads, sel=sel)
    dt = time.perf_counter() - t0
    return {"value": round(len(sel) / dt, 3), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{len(sel)} ligands (stride sample of the {name} library), sweep-v1 C oracle, "
                      f"grid mode, {threads} threads, {dt:.1f} s"}


# -------------------------------------------------------------- reference --
def reference_sample(n_want: int, prefix: int):
    """The C2 library entries j = 0, s, 2s, ... (s = prefix // n_want) built
    by the reference alone: the j-th corpus entry random_smiles(Rng(99)
    .split(i)) with 10-40 heavy atoms and <= 10 torsion axes (the selection
    of our arm's library, chem.corpus_indices), parsed and embedded by the
    reference's own make_ligand / embed_3d (embed seed Rng(2024).split(1)
    .split(j), dock seed .split(2).split(j); pipeline.cpp:422-427, 481-484)."""
    from oracle import ref as R
    stride = max(1, prefix // max(n_want, 1))
    want = set(range(0, stride * n_want, stride))
    ligs, seeds, j, i = [], [], 0, 0
    while len(ligs) < n_want:
        smi = R.random_smiles(CORPUS_SEED, i)
        i += 1
        probe = R.RefLigand(smi, iterations=-1)
        if not (10 <= probe.n_atoms <= 40 and probe.n_tors <= 10):
            continue
        if j in want:
            es = int(R.rng_u64(MASTER_SEED, [1, j], 1)[0])
            ligs.append(R.RefLigand(smi, embed_seed=es, iterations=200))
            seeds.append(int(R.rng_u64(MASTER_SEED, [2, j], 1)[0]))
        j += 1
    return ligs, seeds, stride


def run_reference(args, rank, world):
    """The reference's own CPU path (oracle/_ref/libvsref.so, the unmodified
    reference compiled in place): dock::dock gradient ascent + rescore +
    filter_poses + best (pipeline.cpp:482-515) on all host threads, on a
    stride sample of the C2 library built by the reference itself (corpus
    sampler, parser, embed_3d).  Analytic pocket (the reference has no grid
    maps), C2 knobs, ls_max_steps 500.  Nothing of the product is loaded."""
    if rank != 0:
        return
    from oracle import ref as R
    threads = os.cpu_count() or 1
    lo, hi, cr, cp = POCKET_BOX
    rp = R.RefPocket(R.pocket_json([(c, w, sg, k) for (c, w, sg, k) in pocket_sites()], lo, hi,
                                   cr, cp))
    restarts, delta, keep_top, min_score = 30, 1.0, 4, -5.0
    n_step = threads
    ligs, seeds, stride = reference_sample(n_step * (args.steps + args.warmup), 100_000)
    cursor = [0]

    def step(count):
        sel = range(cursor[0], cursor[0] + count)
        cursor[0] += count
        t0 = time.perf_counter()
        R.dock_best_many([ligs[i] for i in sel], rp, restarts, delta, [seeds[i] for i in sel], 500,
                         keep_top, min_score, threads)
        return count, time.perf_counter() - t0

    for _ in range(args.warmup):
        step(n_step)
    done, secs = 0, 0.0
    for _ in range(args.steps):
        c, dt = step(n_step)
        done += c
        secs += dt
    value = done / secs
    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * secs / args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": dict(CONFIG, workload=CONFIG["workload"] + "; reference: analytic pocket "
                           "(no grid maps in the reference), dock() ascent ls_max_steps 500"),
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                             "kind": "reference",
                             "sample": f"{done} C2 library entries (every {stride}th of the first "
                                       f"100k; {n_step} per step), built and docked by the "
                                       f"reference (oracle/_ref/libvsref.so): dock()+rescore+"
                                       f"filter_poses+best, {threads} threads"},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------- C5 rescoring-only --
RESCORE_ATOM_FLOP = 18 + 3 * 25 + 13 + 46   # FP64 transform, 3 maps trilinear, wall + softplus
RESCORE_ATOM_XU = 3 + 3 * 3 + 3              # conversions, cell indices, softplus


def c5_library(n_per: int, rank: int, world: int, threads: int):
    """96 % corpus entries with 1-40 heavy atoms (<= 10 torsions) + 4 %
    flexible 60-80 atom ligands, in that order; ids ranked globally."""
    import paper_2304_09953_b200 as V
    from paper_2304_09953_b200.chem import corpus_indices, flexible_smiles, random_smiles
    from paper_2304_09953_b200.pipeline import campaign_seeds
    n_flex = max(1, n_per // 25)
    n_small = n_per - n_flex
    total = n_per * world
    idx = corpus_indices(CORPUS_SEED, n_small * world, (1, 40), (0, 10), threads)
    flex = flexible_smiles(11, n_flex * world, max_scan=4000 * n_flex * world + 100000)
    sm = [random_smiles(CORPUS_SEED, int(i)) for i in idx[rank * n_small:(rank + 1) * n_small]]
    sm += flex[rank * n_flex:(rank + 1) * n_flex]
    ids = [f"M{rank * n_per + i}" for i in range(n_per)]
    es = campaign_seeds(MASTER_SEED, total, stage=1)[rank * n_per:(rank + 1) * n_per]
    ds = campaign_seeds(MASTER_SEED, total, stage=2)[rank * n_per:(rank + 1) * n_per]
    lib = V.build_library(sm, ids, es, ds, threads=threads, drop_failed=False)
    ids_all = [f"M{i}" for i in range(total)]
    order = sorted(range(total), key=lambda i: ids_all[i].encode())
    grank = np.empty(total, np.uint32)
    grank[order] = np.arange(total, dtype=np.uint32)
    lib.id_rank = grank[rank * n_per:(rank + 1) * n_per].copy()
    return lib


def survivor_poses(lib, res):
    """Flatten the survivor poses of a dock (ligand-major, non-decreasing
    ligand index) into the vs_rescore arrays."""
    ns = np.maximum(res.n_surv, 0).astype(np.int64)
    pl = np.repeat(np.arange(len(lib), dtype=np.int32), ns)
    slot = np.arange(len(pl)) - np.repeat(np.cumsum(ns) - ns, ns)
    rec = res.surv[pl, slot]
    T = lib.n_tors.astype(np.int64)[pl]
    start = res.tors_off[pl] * res.keep_top + slot * T
    tix = np.repeat(start, T) + (np.arange(int(T.sum())) - np.repeat(np.cumsum(T) - T, T))
    return pl, np.ascontiguousarray(rec["t"]), np.ascontiguousarray(rec["q"]), res.surv_tors[tix]


def c5_work(lib, pl):
    """SURVEY §8(d)'s per-unit terms for rescoring-only: every pose is one
    state and one placement, M = 2 maps per atom (steric + the atom's kind
    map): FLOP = 27 Mv + 14 T + 15 P + N (24 + 12 + 25 M), XU = 2 T + 3 P
    + 3 N, L2_B = N 8 4 M, summed over the poses."""
    N = lib.n_atoms.astype(np.float64)[pl]
    T = lib.n_tors.astype(np.float64)[pl]
    _, to, _ = lib.offsets()
    m = lib.moving_count.astype(np.float64)
    Mv = np.add.reduceat(np.r_[m, 0.0], np.minimum(to[:-1], len(m)))
    Mv = np.where(lib.n_tors > 0, Mv, 0.0)[pl]
    P = N * (N - 1) / 2
    M = 2
    flop = float(np.sum(27 * Mv + 14 * T + 15 * P + N * (24 + 12 + 25 * M)))
    xu = float(np.sum(2 * T + 3 * P + 3 * N))
    l2 = float(np.sum(N * 8 * 4 * M))
    return flop, xu, l2


def run_c5(args, rank, world, cfg):
    """Rescoring-only (BASELINE configs[4]): every survivor pose of a C2-knob
    dock re-scored (geometric score + rescore, K3a) against 0.2 A maps over a
    30 A box.  value = ligands / device time of vs_rescore_survivors (the
    poses already in HBM from the dock, the resident library); e2e = the
    same poses through vs_rescore from pinned host arrays (H2D of library +
    poses, device packer, kernels, D2H of the scores), host wall clock."""
    import torch
    import torch.distributed as dist
    import paper_2304_09953_b200 as V
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    threads = max(1, (os.cpu_count() or 1) // world)
    n_per = args.ligands or cfg["ligands_default"]
    t_build = time.perf_counter()
    lib = c5_library(n_per, rank, world, threads)
    t_build = time.perf_counter() - t_build
    pocket = make_pocket()
    eng = V.Engine(local)
    eng.set_pocket(pocket, grid_spacing=0.4, grid_pad=2.0)
    classes = [(1, 41, 0, 11), (60, 81, 11, 21)]
    prm = params()
    sampler = ClockSampler(local).__enter__()  # clocks over the dock + rescoring region
    eng.upload(lib, classes)
    eng.dock(prm)
    res = eng.fetch()
    pl, T, Q, TH = survivor_poses(lib, res)
    box = V.Pocket(pocket.sites, (-15.0, -15.0, -15.0), (15.0, 15.0, 15.0), pocket.clash_radius,
                   pocket.clash_penalty)
    eng.set_pocket(box, grid_spacing=0.2, grid_pad=2.0)
    peaks = eng.measure_peaks()
    peaks["l2_gather_Bps"] = eng.measure_l2_gather_peak()
    KT = prm.keep_top
    stream = torch.cuda.Stream()
    g_dev = torch.zeros(len(lib) * KT, dtype=torch.float32, device="cuda")
    r_dev = torch.zeros_like(g_dev)
    for _ in range(args.warmup):
        eng.rescore_survivors(g_dev.data_ptr(), r_dev.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = eng.launch_count()
    for k in range(args.steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev[k][0].record(stream)
        eng.rescore_survivors(g_dev.data_ptr(), r_dev.data_ptr(), stream.cuda_stream)
        ev[k][1].record(stream)
        torch.cuda.synchronize()
    launches = eng.launch_count() - launches0
    sampler.__exit__(None, None, None)
    clocks = sampler
    dev_ms = [a.elapsed_time(b) for a, b in ev]
    # e2e: the host path from pinned arrays (library + the same poses)
    pin_library(lib)
    pin = {}
    for name, arr in (("pl", pl.astype(np.int32)), ("T", T), ("Q", Q), ("TH", TH)):
        tt = torch.empty(max(arr.nbytes, 1), dtype=torch.uint8, pin_memory=True)
        view = tt.numpy()[:arr.nbytes].view(arr.dtype).reshape(arr.shape)
        view[...] = arr
        pin[name] = (tt, view)
    ppl, pT, pQ, pTH = (pin[k][1] for k in ("pl", "T", "Q", "TH"))
    from paper_2304_09953_b200.dock import pinned_empty
    outs = (pinned_empty(max(len(pl), 1), np.float32), pinned_empty(max(len(pl), 1), np.float32))
    eng.rescore(lib, ppl, pT, pQ, pTH, out=outs)  # warm
    wall = []
    for _ in range(args.steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.rescore(lib, ppl, pT, pQ, pTH, out=outs)
        wall.append(time.perf_counter() - t0)
    t = torch.tensor([sum(dev_ms), sum(wall)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_s, wall_s = float(t[0]) * 1e-3, float(t[1])
    n_total = len(lib) * world
    flop, xu, l2 = c5_work(lib, pl)
    per_s = dev_s / args.steps
    roofs = {"fp32": flop / peaks["fp32_flops"], "xu": xu / peaks["xu_ops"],
             "l2_gather": l2 / peaks["l2_gather_Bps"]}
    bind = max(roofs, key=roofs.get)
    unit = {"fp32": ("TFLOP/s", 1e12, flop, peaks["fp32_flops"]),
            "xu": ("Tops/s", 1e12, xu, peaks["xu_ops"]),
            "l2_gather": ("GB/s", 1e9, l2, peaks["l2_gather_Bps"])}[bind]
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import sweep
        op = sweep.OraclePocket(box, 0.2, 2.0)
        sel_l = np.arange(0, len(lib), max(1, len(lib) // 2000))
        keep = np.isin(pl, sel_l)
        sub = lib.subset(sel_l)
        remap = -np.ones(len(lib), np.int64)
        remap[sel_l] = np.arange(len(sel_l))
        T_all = lib.n_tors.astype(np.int64)[pl]
        tstart = np.concatenate([[0], np.cumsum(T_all)])[:-1]
        th_sel = np.concatenate([TH[tstart[i]:tstart[i] + T_all[i]] for i in np.nonzero(keep)[0]]
                                or [np.zeros(0, np.float32)])
        t0 = time.perf_counter()
        sweep.score_poses(op, sub, remap[pl[keep]].astype(np.int32), T[keep], Q[keep], th_sel)
        dt = time.perf_counter() - t0
        cpu = {"value": round(len(sel_l) / dt, 2), "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{len(sel_l)} ligands ({int(keep.sum())} poses, stride sample), the C "
                         f"oracle's rescoring (sweep_oracle.c vso_score_poses), 1 thread, {dt:.2f} s"}
    if rank == 0:
        bytes_in = h2d_bytes_raw(lib) + len(pl) * (12 + 16 + 4) + TH.size * 4
        line = {"metric": METRIC, "value": round(n_total * args.steps / dev_s, 2), "unit": UNIT,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(1e3 * dev_s / args.steps, 3), "higher_is_better": True,
                "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f32+f64",
                "data": "synthetic",
                "config": {k: v for k, v in cfg.items() if k not in ("ligands_default", "scaling")}
                | {"ligands_per_gpu": len(lib), "ligands_total": n_total, "poses_per_gpu": len(pl),
                   "parallelism": f"dp{world}" if world > 1 else "single",
                   "l2": "maps 4 x 150^3 cells (> L2 for the 3 score maps + key map); no flush",
                   "timed": "vs_rescore_survivors: the dock's survivor poses already in HBM "
                            "re-scored on the 0.2 A maps (device events)"},
                "roofline": {"bound": bind, "achieved": round(unit[2] / per_s / unit[1], 3),
                             "peak": round(unit[3] / unit[1], 3), "unit": unit[0],
                             "frac": round(roofs[bind] / per_s, 4), "traffic": None,
                             "kernel": "vs_rescore_kernel",
                             "formula": "SURVEY §8(d) per-pose terms, 1 state + 1 placement per "
                                        "pose, M = 2 maps (bench.c5_work)",
                             "frac_fp32": round(roofs["fp32"] / per_s, 4),
                             "frac_xu": round(roofs["xu"] / per_s, 4),
                             "frac_l2_gather": round(roofs["l2_gather"] / per_s, 4)},
                "cpu_baseline": cpu,
                "e2e": {"value": round(n_total * args.steps / wall_s, 2), "unit": UNIT,
                        "h2d_bytes_per_step": bytes_in * world,
                        "d2h_bytes_per_step": 8 * len(pl) * world,
                        "path": "vs_rescore from pinned host arrays (H2D of library + poses, "
                                "device packer, kernels, D2H of the scores into pinned "
                                "buffers), host wall clock"},
                "gpu_launches": launches, "clocks": clocks.summary(), "peaks": peaks,
                "library_build_s": round(t_build, 2)}
        s = json.dumps(line)
        print(s, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(s + "\n")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    eng.close()


# ------------------------------------------------------------------- ours --
def h2d_bytes_raw(lib):
    """bytes of the caller's library arrays as the device packer receives them"""
    A = int(np.sum(lib.n_atoms))
    T = int(np.sum(lib.n_tors))
    M = int(np.sum(lib.moving_count))
    n = len(lib)
    return 3 * 4 * n + 24 * A + 4 * A + 3 * 4 * T + 4 * M + 8 * n + 4 * n


def d2h_bytes(lib, prm):
    n = len(lib)
    T = int(np.sum(lib.n_tors))
    return 4 * n * 3 + 40 * n * prm.keep_top + 4 * T * prm.keep_top + 8 * n + 8 * TOP_K


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.config == "c5":
        run_c5(args, rank, world, cfg)
        return
    import torch
    import torch.distributed as dist
    import paper_2304_09953_b200 as V
    from paper_2304_09953_b200.pipeline import gather_topk, init_comm, merge_topk_host

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    threads = max(1, (os.cpu_count() or 1) // world)
    t_build = time.perf_counter()
    classes = None
    if args.config == "c3":
        n_per = (args.ligands or cfg["ligands_default"]) // world
        lib, ids_all, order = build_workload(n_per, rank, world, threads, balanced=True)
    elif args.config == "c4":
        classes = C4_CLASSES
        lib, ids_all, order = build_flexible(args.ligands or cfg["ligands_default"], rank, world,
                                             threads)
    else:
        lib, ids_all, order = build_workload(args.ligands or cfg["ligands_default"], rank, world,
                                             threads)
    t_build = time.perf_counter() - t_build
    pocket = make_pocket()
    prm = params()
    eng = V.Engine(local)
    eng.set_pocket(pocket, grid_spacing=0.4, grid_pad=2.0)
    peaks = eng.measure_peaks()
    peaks["random_gather16_per_s"] = eng.measure_gather_peak()
    peaks["l2_gather_Bps"] = eng.measure_l2_gather_peak()
    if world > 1:
        init_comm(eng)  # the C-ABI's own NCCL communicator (vs_comm_init)
    eng.upload(lib, classes)
    stream = torch.cuda.Stream()  # non-default stream shared by torch events and the C-ABI
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    keys = torch.empty(TOP_K, dtype=torch.int64, device="cuda")
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > L2

    def step():
        eng.dock(prm, sptr)
        if world > 1:  # local top-k -> ncclAllGather -> device merge (vs_topk_allgather)
            return gather_topk(eng, TOP_K, sptr)
        eng.topk_device(TOP_K, keys.data_ptr(), sptr)
        return keys

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = eng.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    dock_ms, phase = [], []
    with ClockSampler(local) as clocks:
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev[k][0].record(stream)
            out = step()
            ev[k][1].record(stream)
            torch.cuda.synchronize()
            dock_ms.append(eng.last_dock_ms())
            phase.append(eng.phase_ms_ex())
    launches = eng.launch_count() - launches0
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    stats = eng.stats()
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    n_total = len(lib) * world
    value = n_total * args.steps / (total_ms * 1e-3)
    work, gathers = algorithmic_work(lib, prm, stats, True,
                                     sum(s.kind == "steric" for s in pocket.sites))
    phase_ms = {k: float(np.mean([p[k] for p in phase])) for k in phase[0]}
    rl = roofline(frozen_work(lib, prm), phase_ms, float(np.mean(dock_ms)), peaks, load_traffic(),
                  work, gathers)
    rl["hbm_view"] = hbm_view(rl, prm)
    top = out.cpu().numpy().view(np.uint64)
    n_ranked = int(np.sum(top != np.uint64(2**64 - 1)))
    topk_check = None
    if world > 1:
        # the merged top-k against the host top-k of every rank's full key
        # array (all-gathered outside the timed region): the ranking a single
        # GPU would produce over the whole library (keys are shard-invariant)
        mine = eng.fetch().keys
        sizes = [None] * world
        dist.all_gather_object(sizes, len(mine))
        buf = torch.zeros(max(sizes), dtype=torch.int64, device="cuda")
        buf[:len(mine)] = torch.from_numpy(mine.view(np.int64)).cuda()
        allk = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(allk, buf)
        cat = np.concatenate([a.cpu().numpy().view(np.uint64)[:n] for a, n in zip(allk, sizes)])
        topk_check = bool(np.array_equal(merge_topk_host(cat, TOP_K), top))

    e2e = None
    if not args.no_e2e:
        pin_library(lib)  # inputs from pinned host memory (outside the timed region)
        # result buffers in pinned memory, reused by every step (the DMA
        # lands in them directly; each step still reads every result back)
        res_buf = eng.alloc_results(lib, prm, pinned=True)
        n_e2e = max(1, min(args.steps, 5))
        eng.dock_host(lib, prm, classes, out=res_buf)  # warm the host path
        eng.dock_host(lib, prm, classes, out=res_buf, prefetch=lib)  # warm the prefetch path
        eng.dock_host(lib, prm, classes, out=res_buf)  # (adopts it; nothing pending now)
        if world > 1:
            dist.barrier()
        e2e_t = []
        for step in range(n_e2e):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            # each step's library moves to the device under the previous
            # step's dock (vs_dock_host_prefetch); step 0 uploads its own
            eng.dock_host(lib, prm, classes, out=res_buf,
                          prefetch=lib if step + 1 < n_e2e else None)
            if world > 1:
                merged = gather_topk(eng, TOP_K, torch.cuda.current_stream().cuda_stream).cpu()
            else:
                eng.topk(TOP_K)
            e2e_t.append(time.perf_counter() - t0)
        te = torch.tensor([sum(e2e_t)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(n_total * n_e2e / float(te.item()), 2), "unit": UNIT,
               "h2d_bytes_per_step": h2d_bytes_raw(lib) * world,
               "d2h_bytes_per_step": d2h_bytes(lib, prm) * world,
               "steps": n_e2e,
               "path": "vs_dock_host from pinned host arrays (H2D + device packer + dock + D2H "
                       "of every result array into pinned result buffers) + top-k D2H, host "
                       "wall clock; step k+1's library H2D + device pack run under step k's "
                       "dock (vs_dock_host_prefetch), step 0 uploads its own"}

    analytic = None
    if rank == 0 and world == 1 and not args.no_cpu and args.config == "c2":
        # secondary: the same search on the analytic pocket (the reference
        # arm's pocket representation: 240 steric Gaussian sums per pose-atom)
        sub_n = min(len(lib), 5000)
        sub = lib.subset(range(sub_n))
        sub.id_rank = lib.id_rank[:sub_n].copy()
        eng.upload(sub)
        eng.dock(prm, sptr)  # grid mode: the bench's poses for these ligands
        torch.cuda.synchronize()
        res_g = eng.fetch()
        pl, T, Q, TH = survivor_poses(sub, res_g)
        g_grid = res_g.surv[pl, np.arange(len(pl)) - np.repeat(
            np.cumsum(np.maximum(res_g.n_surv, 0)) - np.maximum(res_g.n_surv, 0),
            np.maximum(res_g.n_surv, 0))]["score"]
        eng.set_pocket(pocket, grid_spacing=0.0)
        g_an, _ = eng.rescore(sub, pl, T, Q, TH)  # the same poses, analytic field
        rel = np.abs(g_grid.astype(np.float64) - g_an) / np.maximum(np.abs(g_an), 1.0)
        eng.upload(sub)
        eng.dock(prm, sptr)
        torch.cuda.synchronize()
        ams = eng.last_dock_ms()
        analytic = {"value": round(sub_n / (ams * 1e-3), 2), "unit": UNIT, "ligands": sub_n,
                    "ms": round(ams, 2), "pocket": "analytic (400 Gaussian sites, no grid maps)",
                    "grid_vs_analytic": {
                        "poses": int(len(pl)),
                        "what": "survivor poses of the grid-mode dock re-scored on the analytic "
                                "field (K3a, pinned to the reference within 1e-5): grid "
                                "interpolation error of the emitted geometric scores",
                        "median_rel": float(np.median(rel)), "p99_rel": float(np.quantile(rel, 0.99)),
                        "frac_above_1e-5": float(np.mean(rel > 1e-5))}}
        eng.set_pocket(pocket, grid_spacing=0.4, grid_pad=2.0)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(lib, pocket, prm, args.cpu_seconds, args.config.upper())

    if rank == 0:
        info = eng.device_info()
        line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": True,
                "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f32+f64",
                "data": "synthetic",
                "config": dict({k: v for k, v in cfg.items()
                                if k not in ("ligands_default", "scaling")},
                               ligands_per_gpu=len(lib), ligands_total=n_total,
                               parallelism=f"dp{world}" if world > 1 else "single",
                               l2="flushed (512 MB write) before every timed step",
                               timed="device-resident library -> per-ligand best + global top-1000"),
                "roofline": rl, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks.summary(), "device": info["name"], "peaks": peaks,
                "work": stats, "ranked": n_ranked, "library_build_s": round(t_build, 2)}
        if topk_check is not None:
            line["topk_check"] = {"merged_equals_host_topk_of_all_ranks": topk_check,
                                  "gather": "vs_topk_allgather (C-ABI NCCL all-gather + device merge)"}
        if analytic is not None:
            line["analytic"] = analytic
        s = json.dumps(line)
        print(s, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(s + "\n")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    eng.close()


if __name__ == "__main__":
    main()
