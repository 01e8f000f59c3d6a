"""TEST INFRASTRUCTURE — ctypes bridge to the reference library
(oracle/_ref/libvsref.so, built by oracle/Makefile from /root/reference).
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from . import REF_SO

P = C.POINTER
_lib = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref`")
        L = C.CDLL(REF_SO)
        sig = {
            "vsref_last_error": (C.c_char_p, []),
            "vsref_ligand_new": (C.c_int, [C.c_char_p, C.c_char_p, C.c_uint64, C.c_int, P(C.c_void_p)]),
            "vsref_ligand_free": (None, [C.c_void_p]),
            "vsref_ligand_info": (C.c_int, [C.c_void_p] + [P(C.c_int)] * 4),
            "vsref_ligand_coords": (None, [C.c_void_p, P(C.c_double)]),
            "vsref_ligand_set_coords": (None, [C.c_void_p, P(C.c_double)]),
            "vsref_ligand_classes": (None, [C.c_void_p, P(C.c_int32)]),
            "vsref_ligand_bonds": (C.c_int, [C.c_void_p, P(C.c_int32), C.c_int]),
            "vsref_ligand_axes": (None, [C.c_void_p] + [P(C.c_int32)] * 4),
            "vsref_pocket_parse": (C.c_int, [C.c_char_p, P(C.c_void_p)]),
            "vsref_pocket_free": (None, [C.c_void_p]),
            "vsref_geometric_score": (C.c_int, [C.c_void_p, C.c_void_p, P(C.c_double), P(C.c_double),
                                                P(C.c_double), C.c_int, P(C.c_double)]),
            "vsref_score_gradient": (C.c_int, [C.c_void_p, C.c_void_p, P(C.c_double),
                                               P(C.c_double), P(C.c_double), C.c_int,
                                               P(C.c_double)]),
            "vsref_rescore": (C.c_int, [C.c_void_p, C.c_void_p, P(C.c_double), P(C.c_double),
                                        P(C.c_double), C.c_int, P(C.c_double)]),
            "vsref_apply_pose": (C.c_int, [C.c_void_p, P(C.c_double), P(C.c_double), P(C.c_double),
                                           C.c_int, P(C.c_double)]),
            "vsref_rmsd": (C.c_int, [P(C.c_double), C.c_int, P(C.c_double), C.c_int, P(C.c_double)]),
            "vsref_dock": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.c_int,
                                     C.c_int, P(C.c_double), C.c_int]),
            "vsref_dock_best": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_uint64,
                                          C.c_int, C.c_int, C.c_double, P(C.c_double)]),
            "vsref_dock_best_many": (C.c_int, [P(C.c_void_p), C.c_int, C.c_void_p, C.c_int, C.c_double,
                                               P(C.c_uint64), C.c_int, C.c_int, C.c_double, C.c_int,
                                               P(C.c_int32), P(C.c_double)]),
            "vsref_filter_poses": (C.c_int, [P(C.c_double), C.c_int, C.c_long, C.c_double, P(C.c_int32)]),
            "vsref_rank_ligands": (C.c_int, [C.c_char_p, P(C.c_double), C.c_int, P(C.c_int32)]),
            "vsref_size_class": (C.c_int, [C.c_int, C.c_int, P(C.c_int32), C.c_int]),
            "vsref_target_batch_size": (C.c_int, [C.c_double] * 4 + [C.c_int, C.c_int, P(C.c_long)]),
            "vsref_simulate_throughput": (C.c_double, [C.c_long, C.c_double, C.c_double]),
            "vsref_bucket_replay": (C.c_int, [P(C.c_int32), P(C.c_int32), C.c_int, P(C.c_int32), C.c_int]
                                    + [C.c_double] * 4 + [P(C.c_int32)] * 4),
            "vsref_rng_u64": (None, [C.c_uint64, P(C.c_uint64), C.c_int, C.c_int, P(C.c_uint64)]),
            "vsref_start_draws": (None, [P(C.c_uint64), P(C.c_int32), C.c_int, C.c_int, C.c_int,
                                         P(C.c_double), P(C.c_double), C.c_int, P(C.c_float)]),
            "vsref_parse_check": (C.c_int, [C.c_char_p, P(C.c_int), P(C.c_long), P(C.c_int),
                                         P(C.c_int)]),
            "vsref_pocket_json": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int]),
            "vsref_pose_json": (C.c_int, [C.c_char_p, P(C.c_double), P(C.c_double), P(C.c_double),
                                          C.c_int, C.c_double, C.c_int, C.c_double, C.c_char_p,
                                          C.c_int]),
            "vsref_report_bytes": (C.c_int, [C.c_char_p, C.c_int, C.c_char_p, C.c_int]),
            "vsref_smzc_compress": (C.c_int, [C.c_char_p, C.c_long, C.c_char_p, C.c_char_p, C.c_long]),
            "vsref_smzc_decompress": (C.c_int, [C.c_char_p, C.c_long, C.c_char_p, C.c_char_p,
                                                C.c_long]),
            "vsref_train_dictionary": (C.c_int, [C.c_char_p, C.c_long, C.c_int, C.c_char_p, C.c_long]),
            "vsref_run_campaign": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p]),
            "vsref_dictionary_entries": (C.c_int, [C.c_char_p, C.c_char_p, C.c_long]),
            "vsref_rng_draws": (None, [C.c_uint64, P(C.c_uint64), C.c_int, P(C.c_int32), P(C.c_double),
                                       P(C.c_double), C.c_int, P(C.c_double)]),
            "vsref_random_smiles": (C.c_int, [C.c_uint64, C.c_uint64, C.c_char_p, C.c_int]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(P(t))


class RefError(RuntimeError):
    def __init__(self, code: int):
        self.code = code
        super().__init__(f"reference error {code}: {lib().vsref_last_error().decode()}")


def _chk(rc: int) -> int:
    if rc < 0:
        raise RefError(rc)
    return rc


class RefPocket:
    def __init__(self, pocket_json: str):
        h = C.c_void_p()
        _chk(lib().vsref_pocket_parse(pocket_json.encode(), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().vsref_pocket_free(self.h)


class RefLigand:
    """make_ligand + embed_3d + torsion_topology of the reference."""

    def __init__(self, smiles: str, embed_seed: int = 0, iterations: int = 200, ligand_id: str = ""):
        h = C.c_void_p()
        _chk(lib().vsref_ligand_new(smiles.encode(), ligand_id.encode(), embed_seed & (2**64 - 1),
                                    iterations, C.byref(h)))
        self.h = h
        self.smiles = smiles
        n, t, r, m = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        lib().vsref_ligand_info(h, C.byref(n), C.byref(t), C.byref(r), C.byref(m))
        self.n_atoms, self.n_tors, self.rot_bonds, self.n_moving = n.value, t.value, r.value, m.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().vsref_ligand_free(self.h)

    def coords(self) -> np.ndarray:
        out = np.zeros(3 * max(self.n_atoms, 1))
        lib().vsref_ligand_coords(self.h, _p(out, C.c_double))
        return out[:3 * self.n_atoms].reshape(-1, 3)

    def set_coords(self, xyz: np.ndarray):
        a = np.ascontiguousarray(xyz, np.float64).reshape(-1)
        lib().vsref_ligand_set_coords(self.h, _p(a, C.c_double))

    def classes(self) -> np.ndarray:
        out = np.zeros(max(self.n_atoms, 1), np.int32)
        lib().vsref_ligand_classes(self.h, _p(out, C.c_int32))
        return out[:self.n_atoms]

    def bonds(self):
        out = np.zeros(4 * 512, np.int32)
        n = _chk(lib().vsref_ligand_bonds(self.h, _p(out, C.c_int32), 512))
        return out[:4 * n].reshape(-1, 4)

    def axes(self):
        T = max(self.n_tors, 1)
        a, b, c = (np.zeros(T, np.int32) for _ in range(3))
        m = np.zeros(max(self.n_moving, 1), np.int32)
        lib().vsref_ligand_axes(self.h, _p(a, C.c_int32), _p(b, C.c_int32), _p(c, C.c_int32),
                                _p(m, C.c_int32))
        out, k = [], 0
        for j in range(self.n_tors):
            out.append((int(a[j]), int(b[j]), [int(v) for v in m[k:k + c[j]]]))
            k += int(c[j])
        return out

    def _pose(self, t, q, tors):
        t = np.ascontiguousarray(t, np.float64)
        q = np.ascontiguousarray(q, np.float64)
        th = np.ascontiguousarray(tors if len(tors) else [0.0], np.float64)
        return t, q, th, len(tors)

    def geometric_score(self, pocket: RefPocket, t, q, tors) -> float:
        t, q, th, nt = self._pose(t, q, tors)
        out = C.c_double()
        _chk(lib().vsref_geometric_score(self.h, pocket.h, _p(t, C.c_double), _p(q, C.c_double),
                                         _p(th, C.c_double), nt, C.byref(out)))
        return out.value

    def score_gradient(self, pocket: RefPocket, t, q, tors):
        """(score, gt[3], gq[4], gtor[T]) of the reference score_gradient."""
        t, q, th, nt = self._pose(t, q, tors)
        out = np.zeros(8 + max(nt, 1), np.float64)
        _chk(lib().vsref_score_gradient(self.h, pocket.h, _p(t, C.c_double), _p(q, C.c_double),
                                        _p(th, C.c_double), nt, _p(out, C.c_double)))
        return out[0], out[1:4].copy(), out[4:8].copy(), out[8:8 + nt].copy()

    def rescore(self, pocket: RefPocket, t, q, tors) -> float:
        t, q, th, nt = self._pose(t, q, tors)
        out = C.c_double()
        _chk(lib().vsref_rescore(self.h, pocket.h, _p(t, C.c_double), _p(q, C.c_double),
                                 _p(th, C.c_double), nt, C.byref(out)))
        return out.value

    def apply_pose(self, t, q, tors) -> np.ndarray:
        t, q, th, nt = self._pose(t, q, tors)
        out = np.zeros(3 * self.n_atoms)
        _chk(lib().vsref_apply_pose(self.h, _p(t, C.c_double), _p(q, C.c_double), _p(th, C.c_double),
                                    nt, _p(out, C.c_double)))
        return out.reshape(-1, 3)

    def dock(self, pocket: RefPocket, restarts: int, delta: float, seed: int, max_steps: int = 500,
             with_rescore: bool = True):
        stride = 9 + self.n_tors
        out = np.zeros(stride * restarts)
        n = _chk(lib().vsref_dock(self.h, pocket.h, restarts, delta, seed & (2**64 - 1), max_steps,
                                  1 if with_rescore else 0, _p(out, C.c_double), restarts))
        return out[:n * stride].reshape(n, stride)


def dock_best_many(ligs, pocket: RefPocket, restarts, delta, seeds, max_steps, keep_top, min_score,
                   threads):
    n = len(ligs)
    hs = (C.c_void_p * n)(*[lg.h for lg in ligs])
    sd = np.ascontiguousarray(seeds, np.uint64)
    kept = np.zeros(n, np.int32)
    best = np.zeros(n)
    _chk(lib().vsref_dock_best_many(hs, n, pocket.h, restarts, delta, _p(sd, C.c_uint64), max_steps,
                                    keep_top, min_score, threads, _p(kept, C.c_int32),
                                    _p(best, C.c_double)))
    return kept, best


def rng_u64(seed: int, path, n: int) -> np.ndarray:
    pa = np.ascontiguousarray(path if len(path) else [0], np.uint64)
    out = np.zeros(n, np.uint64)
    lib().vsref_rng_u64(seed, _p(pa, C.c_uint64), len(path), n, _p(out, C.c_uint64))
    return out


def rng_draws(seed: int, path, kinds, lo=None, hi=None) -> np.ndarray:
    n = len(kinds)
    pa = np.ascontiguousarray(path if len(path) else [0], np.uint64)
    k = np.ascontiguousarray(kinds, np.int32)
    lo = np.ascontiguousarray(lo if lo is not None else np.zeros(n))
    hi = np.ascontiguousarray(hi if hi is not None else np.ones(n))
    out = np.zeros(n)
    lib().vsref_rng_draws(seed, _p(pa, C.c_uint64), len(path), _p(k, C.c_int32), _p(lo, C.c_double),
                          _p(hi, C.c_double), n, _p(out, C.c_double))
    return out


def random_smiles(seed: int, i: int) -> str:
    buf = C.create_string_buffer(4096)
    _chk(lib().vsref_random_smiles(seed, i, buf, 4096))
    return buf.value.decode()


def filter_poses(scores, keep_top, min_score):
    s = np.ascontiguousarray(scores, np.float64)
    out = np.zeros(max(len(s), 1), np.int32)
    n = lib().vsref_filter_poses(_p(s, C.c_double), len(s), keep_top, min_score, _p(out, C.c_int32))
    return [int(v) for v in out[:n]]


def rank_ligands(scores: dict):
    ids = list(scores)
    blob = b"".join(i.encode() + b"\0" for i in ids) or b"\0"
    s = np.array([scores[i] for i in ids], np.float64)
    out = np.zeros(max(len(ids), 1), np.int32)
    n = lib().vsref_rank_ligands(blob, _p(s, C.c_double), len(ids), _p(out, C.c_int32))
    return [(ids[i], float(s[i])) for i in out[:n]]


def size_class(atoms, rot, classes):
    c = np.ascontiguousarray(np.array(classes, np.int32).reshape(-1))
    return lib().vsref_size_class(atoms, rot, _p(c, C.c_int32), len(classes))


def target_batch_size(cap, fixed, per_atom, per_rot, atom_hi, rot_hi):
    out = C.c_long()
    rc = lib().vsref_target_batch_size(cap, fixed, per_atom, per_rot, atom_hi, rot_hi, C.byref(out))
    if rc < 0:
        raise RefError(rc)
    return out.value


def simulate_throughput(n, overhead, service):
    return lib().vsref_simulate_throughput(n, overhead, service)


def bucket_replay(atoms, rot, classes, cap, fixed, per_atom, per_rot):
    n = len(atoms)
    a = np.ascontiguousarray(atoms, np.int32)
    r = np.ascontiguousarray(rot, np.int32)
    c = np.ascontiguousarray(np.array(classes, np.int32).reshape(-1))
    ir, bc, bl, mem = (np.zeros(max(n, 1), np.int32) for _ in range(4))
    nb = _chk(lib().vsref_bucket_replay(_p(a, C.c_int32), _p(r, C.c_int32), n, _p(c, C.c_int32),
                                        len(classes), cap, fixed, per_atom, per_rot, _p(ir, C.c_int32),
                                        _p(bc, C.c_int32), _p(bl, C.c_int32), _p(mem, C.c_int32)))
    out, k = [], 0
    for b in range(nb):
        out.append((int(bc[b]), [int(v) for v in mem[k:k + bl[b]]]))
        k += int(bl[b])
    return ir[:n].astype(bool), out


def pocket_json(sites, lo, hi, clash_radius, clash_penalty) -> str:
    return json.dumps({"sites": [{"center": list(c), "weight": w, "sigma": s, "kind": k}
                                 for (c, w, s, k) in sites],
                       "bounds": {"min": list(lo), "max": list(hi)},
                       "clash_radius": clash_radius, "clash_penalty": clash_penalty})


def start_draws(seeds, n_tors, restarts: int, attempts: int, lo, hi) -> np.ndarray:
    """FP32 casts of the reference dock() start draws (dock.cpp:343-354)
    for every (ligand, restart, attempt): [n, R, A, 7 + max T] rows of t, q,
    theta (shim vsref_start_draws)."""
    seeds = np.ascontiguousarray(seeds, np.uint64)
    n_tors = np.ascontiguousarray(n_tors, np.int32)
    n = len(seeds)
    stride = 7 + (int(n_tors.max()) if n else 0)
    out = np.zeros(max(n * restarts * attempts * stride, 1), np.float32)
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    lib().vsref_start_draws(_p(seeds, C.c_uint64), _p(n_tors, C.c_int32), n, restarts, attempts,
                            _p(lo, C.c_double), _p(hi, C.c_double), stride, _p(out, C.c_float))
    return out[:n * restarts * attempts * stride].reshape(n, restarts, attempts, stride)


def parse_check(smiles: str):
    """("ok", n_atoms, n_bonds) or ("error", kind index, 1-based position) of
    the reference chem::parse_smiles (shim vsref_parse_check)."""
    k, p, na, nb = C.c_int(), C.c_long(), C.c_int(), C.c_int()
    rc = lib().vsref_parse_check(smiles.encode("latin-1"), C.byref(k), C.byref(p), C.byref(na),
                                 C.byref(nb))
    return ("error", k.value, p.value) if rc else ("ok", na.value, nb.value)


def pocket_json_bytes(text: str) -> str:
    """pocket_to_json(parse_pocket_json(text)) of the reference."""
    buf = C.create_string_buffer(1 << 20)
    _chk(lib().vsref_pocket_json(text.encode(), buf, 1 << 20))
    return buf.value.decode()


def pose_json_bytes(ligand: str, t, q, tors, geo: float, rescore) -> str:
    """pose_to_json of the reference for the given pose (rescore None = absent)."""
    t = np.ascontiguousarray(t, np.float64)
    q = np.ascontiguousarray(q, np.float64)
    th = np.ascontiguousarray(tors if len(tors) else [0.0], np.float64)
    buf = C.create_string_buffer(1 << 16)
    n = lib().vsref_pose_json(ligand.encode(), _p(t, C.c_double), _p(q, C.c_double),
                              _p(th, C.c_double), len(tors), float(geo),
                              0 if rescore is None else 1, float(rescore or 0.0), buf, 1 << 16)
    _chk(n)
    return buf.value.decode()


def report_bytes(spec: dict, which: int = 0) -> str:
    """CampaignReport::to_json (which 0) / results_tsv (1) of the reference."""
    buf = C.create_string_buffer(1 << 20)
    _chk(lib().vsref_report_bytes(json.dumps(spec).encode(), which, buf, 1 << 20))
    return buf.value.decode()


def smzc_compress(text: bytes, dict_path: str) -> bytes:
    """codec::compress_stream of the reference (the dictionary from a file)."""
    cap = 2 * len(text) + 4096
    buf = C.create_string_buffer(cap)
    n = _chk(lib().vsref_smzc_compress(text, len(text), dict_path.encode(), buf, cap))
    return buf.raw[:n]


def smzc_decompress(data: bytes, dict_path: str) -> bytes:
    cap = 16 * len(data) + 4096
    buf = C.create_string_buffer(cap)
    n = _chk(lib().vsref_smzc_decompress(data, len(data), dict_path.encode(), buf, cap))
    return buf.raw[:n]


def train_dictionary(text: bytes, max_entries: int) -> bytes:
    """codec::train_dictionary + save_dictionary: SMZ1 bytes."""
    buf = C.create_string_buffer(8192)
    n = _chk(lib().vsref_train_dictionary(text, len(text), max_entries, buf, 8192))
    return buf.raw[:n]


def run_campaign(cfg_path: str, trace_path: str, report_path: str, tsv_path: str) -> int:
    """The reference's run_campaign on a config file (outputs redirected)."""
    return _chk(lib().vsref_run_campaign(cfg_path.encode(), trace_path.encode(),
                                         report_path.encode(), tsv_path.encode()))


def dictionary_entries(path: str) -> list[str]:
    """codec::load_dictionary_file(path).entries of the reference."""
    buf = C.create_string_buffer(8192)
    n = _chk(lib().vsref_dictionary_entries(path.encode(), buf, 8192))
    return [x.decode() for x in buf.raw[:n].split(b"\0")[:-1]]
