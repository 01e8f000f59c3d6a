"""TEST INFRASTRUCTURE — ctypes bridge to the sweep-v1 C oracle
(oracle/_ref/libvsoracle.so built from oracle/sweep_oracle.c).

Accepts the product's Library / Pocket / DockParams objects (plain data) so
tests can run the GPU path and the oracle on identical inputs.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import ORACLE_SO, build

P = C.POINTER


class Site(C.Structure):
    _fields_ = [("center", C.c_double * 3), ("weight", C.c_double), ("sigma", C.c_double),
                ("kind", C.c_int32), ("reserved", C.c_int32)]


class PocketDesc(C.Structure):
    _fields_ = [("sites", P(Site)), ("n_sites", C.c_int32), ("reserved", C.c_int32),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("clash_radius", C.c_double),
                ("clash_penalty", C.c_double), ("grid_spacing", C.c_double), ("grid_pad", C.c_double)]


class Params(C.Structure):
    _fields_ = [("restarts", C.c_int32), ("rotations", C.c_int32), ("flex_angles", C.c_int32),
                ("flex_passes", C.c_int32), ("diversity_delta", C.c_double), ("keep_top", C.c_int32),
                ("write_all", C.c_int32), ("min_score", C.c_double), ("polish", C.c_int32),
                ("reserved", C.c_int32)]


class Lib(C.Structure):
    _fields_ = [("n_ligands", C.c_int32), ("reserved", C.c_int32),
                ("n_atoms", P(C.c_int32)), ("n_tors", P(C.c_int32)), ("coords", P(C.c_double)),
                ("atom_class", P(C.c_int32)), ("axis_a", P(C.c_int32)), ("axis_b", P(C.c_int32)),
                ("moving_count", P(C.c_int32)), ("moving", P(C.c_int32)), ("seeds", P(C.c_uint64)),
                ("id_rank", P(C.c_uint32))]


class Results(C.Structure):
    _fields_ = [("best", P(C.c_float)), ("n_kept", P(C.c_int32)), ("n_surv", P(C.c_int32)),
                ("surv", C.c_void_p), ("surv_tors", P(C.c_float)), ("all", C.c_void_p),
                ("all_tors", P(C.c_float)), ("keys", P(C.c_uint64))]


POSE_DTYPE = np.dtype([("t", np.float32, 3), ("q", np.float32, 4), ("score", np.float32),
                       ("rescore", np.float32), ("restart", np.int16), ("attempt", np.int16),
                       ("rot", np.int16), ("reserved", np.int16)])

_lib = None
KINDS = {"steric": 0, "hbond": 1, "lipophilic": 2}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = C.CDLL(ORACLE_SO)
        sig = {
            "vso_pocket_new": (C.c_int, [P(PocketDesc), P(C.c_void_p)]),
            "vso_pocket_free": (None, [C.c_void_p]),
            "vso_grid_info": (C.c_int, [C.c_void_p, P(C.c_int32), P(C.c_float), P(C.c_float)]),
            "vso_grid_fetch": (C.c_int, [C.c_void_p, P(C.c_float), P(C.c_float), P(C.c_float)]),
            "vso_rotation_set": (None, [C.c_int32, C.c_uint64, P(C.c_float)]),
            "vso_dock_library": (C.c_int, [C.c_void_p, P(Lib), P(C.c_int32), C.c_int32, P(Params),
                                           P(C.c_float), C.c_int32, P(Results)]),
            "vso_score_poses": (C.c_int, [C.c_void_p, P(Lib), C.c_int64, P(C.c_int32), P(C.c_float),
                                          P(C.c_float), P(C.c_float), P(C.c_float), P(C.c_float)]),
            "vso_exp_neg": (C.c_float, [C.c_float]),
            "vso_log1p01": (C.c_float, [C.c_float]),
            "vso_softplus": (C.c_float, [C.c_float]),
            "vso_sincos": (None, [C.c_float, P(C.c_float), P(C.c_float)]),
            "vso_topk": (C.c_int, [P(C.c_uint64), C.c_int64, C.c_int32, P(C.c_uint64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(P(t))


class OraclePocket:
    def __init__(self, pocket, grid_spacing: float = 0.0, grid_pad: float = 2.0):
        arr = (Site * max(1, len(pocket.sites)))()
        for i, s in enumerate(pocket.sites):
            arr[i].center[:] = list(s.center)
            arr[i].weight, arr[i].sigma, arr[i].kind = s.weight, s.sigma, KINDS[s.kind]
        d = PocketDesc()
        d.sites = C.cast(arr, P(Site))
        d.n_sites = len(pocket.sites)
        d.lo[:] = list(pocket.lo)
        d.hi[:] = list(pocket.hi)
        d.clash_radius, d.clash_penalty = pocket.clash_radius, pocket.clash_penalty
        d.grid_spacing, d.grid_pad = grid_spacing, grid_pad
        h = C.c_void_p()
        lib().vso_pocket_new(C.byref(d), C.byref(h))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().vso_pocket_free(self.h)

    def grid_maps(self):
        dims = (C.c_int32 * 3)()
        origin = (C.c_float * 3)()
        sp = C.c_float()
        lib().vso_grid_info(self.h, dims, origin, C.byref(sp))
        n = dims[0] * dims[1] * dims[2]
        maps = [np.zeros(n, np.float32) for _ in range(3)]
        lib().vso_grid_fetch(self.h, *(_p(m, C.c_float) for m in maps))
        shape = (dims[2], dims[1], dims[0])
        return [m.reshape(shape) for m in maps], tuple(origin), sp.value


def _lib_c(L):
    c = Lib()
    c.n_ligands = len(L.ids)
    keep = []
    for name, t in (("n_atoms", C.c_int32), ("n_tors", C.c_int32), ("coords", C.c_double),
                    ("atom_class", C.c_int32), ("axis_a", C.c_int32), ("axis_b", C.c_int32),
                    ("moving_count", C.c_int32), ("moving", C.c_int32), ("seeds", C.c_uint64),
                    ("id_rank", C.c_uint32)):
        dt = {C.c_int32: np.int32, C.c_double: np.float64, C.c_uint64: np.uint64,
              C.c_uint32: np.uint32}[t]
        a = np.ascontiguousarray(getattr(L, name), dt).reshape(-1)
        if a.size == 0:
            a = np.zeros(1, dt)
        keep.append(a)
        setattr(c, name, _p(a, t))
    c._keep = keep
    return c


def rotation_set(K: int, seed: int) -> np.ndarray:
    out = np.zeros(4 * K, np.float32)
    lib().vso_rotation_set(K, seed, _p(out, C.c_float))
    return out.reshape(K, 4)


def dock_library(pocket: OraclePocket, L, prm, threads: int = 1, sel=None):
    """Returns a dict with best, n_kept, n_surv, surv, surv_tors, keys (+all)."""
    n = len(L.ids)
    tt = int(np.sum(L.n_tors))
    kt, R = max(prm.keep_top, 1), prm.restarts
    out = {"best": np.full(max(n, 1), np.nan, np.float32), "n_kept": np.zeros(max(n, 1), np.int32),
           "n_surv": np.zeros(max(n, 1), np.int32), "surv": np.zeros((max(n, 1), kt), POSE_DTYPE),
           "surv_tors": np.zeros(max(tt * kt, 1), np.float32), "keys": np.zeros(max(n, 1), np.uint64)}
    r = Results()
    r.best, r.n_kept, r.n_surv = _p(out["best"], C.c_float), _p(out["n_kept"], C.c_int32), _p(out["n_surv"], C.c_int32)
    r.surv = out["surv"].ctypes.data_as(C.c_void_p)
    r.surv_tors = _p(out["surv_tors"], C.c_float)
    r.keys = _p(out["keys"], C.c_uint64)
    if prm.write_all_poses:
        out["all"] = np.zeros((max(n, 1), R), POSE_DTYPE)
        out["all_tors"] = np.zeros(max(tt * R, 1), np.float32)
        r.all = out["all"].ctypes.data_as(C.c_void_p)
        r.all_tors = _p(out["all_tors"], C.c_float)
    p = Params()
    p.restarts, p.rotations, p.flex_angles, p.flex_passes = prm.restarts, prm.rotations, prm.flex_angles, prm.flex_passes
    p.diversity_delta, p.keep_top, p.write_all, p.min_score = prm.diversity_delta, prm.keep_top, int(prm.write_all_poses), prm.min_score
    p.polish = int(getattr(prm, "polish", 0))
    rots = rotation_set(prm.rotations, prm.rotation_seed)
    lc = _lib_c(L)
    selc = None if sel is None else np.ascontiguousarray(sel, np.int32)
    rc = lib().vso_dock_library(pocket.h, C.byref(lc), None if selc is None else _p(selc, C.c_int32),
                                0 if selc is None else len(selc), C.byref(p), _p(rots.reshape(-1), C.c_float),
                                threads, C.byref(r))
    if rc != 0:
        raise RuntimeError(f"oracle dock failed: {rc}")
    for k in list(out):
        if k in ("surv_tors", "all_tors"):
            continue
        out[k] = out[k][:n]
    return out


def score_poses(pocket: OraclePocket, L, pose_lig, t, q, tors):
    n = len(pose_lig)
    pl = np.ascontiguousarray(pose_lig, np.int32)
    t = np.ascontiguousarray(t, np.float32).reshape(-1)
    q = np.ascontiguousarray(q, np.float32).reshape(-1)
    tors = np.ascontiguousarray(tors, np.float32).reshape(-1)
    if tors.size == 0:
        tors = np.zeros(1, np.float32)
    geo = np.zeros(max(n, 1), np.float32)
    resc = np.zeros(max(n, 1), np.float32)
    lc = _lib_c(L)
    lib().vso_score_poses(pocket.h, C.byref(lc), n, _p(pl, C.c_int32), _p(t, C.c_float), _p(q, C.c_float),
                          _p(tors, C.c_float), _p(geo, C.c_float), _p(resc, C.c_float))
    return geo[:n], resc[:n]


def topk(keys, k):
    keys = np.ascontiguousarray(keys, np.uint64)
    out = np.zeros(k, np.uint64)
    lib().vso_topk(_p(keys, C.c_uint64), len(keys), k, _p(out, C.c_uint64))
    return out
