"""Dock/score entry points — the Python mirror of proj/include/vscreen/dock.hpp
on top of the B200 kernels (through the C-ABI, capi.h).

Scoring (`geometric_score`, `rescore`) and pose generation (`dock`) run on
the GPU; there is no CPU path.  `apply_pose`, `rmsd` and the JSON helpers
are plain host utilities, as in the reference.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _capi
from ._capi import lib as _lib, ptr
from .chem import Conformer, Library, Ligand, TorsionTopology, id_ranks
from .errors import (AtomCountMismatch, EmptyBounds, LengthMismatch, PocketError, check)

KINDS = {"steric": 0, "hbond": 1, "lipophilic": 2}
KIND_NAMES = {v: k for k, v in KINDS.items()}


@dataclass
class Site:
    """dock::Site (dock.hpp:18-23)."""
    center: tuple[float, float, float]
    weight: float = 1.0
    sigma: float = 1.0
    kind: str = "steric"


@dataclass
class Pocket:
    """dock::Pocket (dock.hpp:32-37); bounds as (lo, hi) triples."""
    sites: list[Site] = field(default_factory=list)
    lo: tuple[float, float, float] = (0.0, 0.0, 0.0)
    hi: tuple[float, float, float] = (0.0, 0.0, 0.0)
    clash_radius: float = 0.8
    clash_penalty: float = 1.0

    def empty(self) -> bool:
        return any(h <= l for l, h in zip(self.lo, self.hi))

    def as_c(self):
        arr = (_capi.vs_site * max(1, len(self.sites)))()
        for i, s in enumerate(self.sites):
            arr[i].center[:] = [float(v) for v in s.center]
            arr[i].weight = float(s.weight)
            arr[i].sigma = float(s.sigma)
            arr[i].kind = KINDS[s.kind]
        p = _capi.vs_pocket()
        p.sites = C.cast(arr, C.POINTER(_capi.vs_site))
        p.n_sites = len(self.sites)
        p.lo[:] = [float(v) for v in self.lo]
        p.hi[:] = [float(v) for v in self.hi]
        p.clash_radius = float(self.clash_radius)
        p.clash_penalty = float(self.clash_penalty)
        p._keep = arr
        return p


@dataclass
class Pose:
    """dock::Pose (dock.hpp:39-46) plus the sweep-v1 index tuple."""
    ligand_id: str = ""
    translation: tuple[float, float, float] = (0.0, 0.0, 0.0)
    rotation: tuple[float, float, float, float] = (1.0, 0.0, 0.0, 0.0)
    torsions: list[float] = field(default_factory=list)
    geometric_score: float = 0.0
    rescore: float | None = None
    restart: int = -1
    attempt: int = -1
    rot_index: int = -1


# ------------------------------------------------------------------- JSON --
def parse_pocket_json(text: str) -> Pocket:
    """dock::parse_pocket_json (dock.cpp:432-450)."""
    try:
        j = json.loads(text)
        sites = []
        for js in j["sites"]:
            kind = js["kind"]
            if kind not in KINDS:
                raise PocketError(f"unknown site kind: {kind}")
            s = Site(tuple(float(v) for v in js["center"][:3]), float(js["weight"]),
                     float(js["sigma"]), kind)
            if not s.sigma > 0.0:
                raise PocketError("site sigma must be > 0")
            sites.append(s)
        p = Pocket(sites, tuple(float(v) for v in j["bounds"]["min"][:3]),
                   tuple(float(v) for v in j["bounds"]["max"][:3]),
                   float(j["clash_radius"]), float(j["clash_penalty"]))
    except PocketError:
        raise
    except (KeyError, TypeError, ValueError, IndexError) as e:
        raise PocketError(f"bad pocket JSON: {e}") from e
    if p.clash_penalty < 0.0:
        raise PocketError("clash_penalty must be >= 0")
    return p


def load_pocket_file(path: str) -> Pocket:
    """dock::load_pocket_file (dock.cpp:452-458)."""
    try:
        with open(path) as f:
            return parse_pocket_json(f.read())
    except OSError as e:
        raise PocketError(f"cannot open pocket file: {path}") from e


def _jnums(xs) -> list[str]:
    """Doubles as nlohmann::json 3.11 dumps them (the reference's JSON
    library; capi.h vs_json_format_doubles): Grisu2 digits, fixed notation
    for decimal exponents in (-4, 15], else d.ddde+XX, null if non-finite."""
    x = np.ascontiguousarray(xs, np.float64).reshape(-1)
    if x.size == 0:
        return []
    buf = C.create_string_buffer(32 * x.size)
    check(_lib.vs_json_format_doubles(ptr(x, C.c_double), x.size, buf, 32))
    raw = buf.raw
    return [raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode() for i in range(x.size)]


def _jnum(x) -> str:
    return _jnums([x])[0]


def _jstr(v: str) -> str:
    return json.dumps(v, ensure_ascii=False)  # same escapes as nlohmann (UTF-8 kept)


def pocket_to_json(p: Pocket) -> str:
    """dock::pocket_to_json (dock.cpp:460-474): the ordered_json dump(2)
    bytes of the reference (tests/test_json_bytes.py)."""
    def arr(v, ind):
        pad = " " * ind
        return "[\n" + ",\n".join(pad + "  " + _jnum(x) for x in v) + "\n" + pad + "]"

    sites = []
    for st in p.sites:
        sites.append("    {\n"
                     f'      "center": {arr(st.center, 6)},\n'
                     f'      "weight": {_jnum(st.weight)},\n'
                     f'      "sigma": {_jnum(st.sigma)},\n'
                     f'      "kind": {_jstr(st.kind)}\n'
                     "    }")
    site_block = "[\n" + ",\n".join(sites) + "\n  ]" if sites else "[]"
    return ("{\n"
            f'  "sites": {site_block},\n'
            '  "bounds": {\n'
            f'    "min": {arr(p.lo, 4)},\n'
            f'    "max": {arr(p.hi, 4)}\n'
            "  },\n"
            f'  "clash_radius": {_jnum(p.clash_radius)},\n'
            f'  "clash_penalty": {_jnum(p.clash_penalty)}\n'
            "}")


def pose_to_json(pose: Pose) -> str:
    """dock::pose_to_json (dock.cpp:476-489): compact ordered_json bytes."""
    t, q, th = list(pose.translation), list(pose.rotation), list(pose.torsions)
    v = _jnums(t + q + th + [pose.geometric_score] + ([] if pose.rescore is None else [pose.rescore]))
    nums = lambda a, b: "[" + ",".join(v[a:b]) + "]"
    n = 7 + len(th)
    resc = "null" if pose.rescore is None else v[n + 1]
    return (f'{{"ligand":{_jstr(pose.ligand_id)},"translation":{nums(0, 3)},'
            f'"rotation":{nums(3, 7)},"torsions":{nums(7, n)},'
            f'"geometric_score":{v[n]},"rescore":{resc}}}')


# --------------------------------------------------------------- params ---
@dataclass
class DockParams:
    """dock(restarts, diversity_delta) + StageKnobs keep_top/min_score
    (pipeline.hpp:33-40) + the sweep-v1 knobs (docs/SWEEP_V1.md)."""
    restarts: int = 30
    diversity_delta: float = 1.0
    rotations: int = 256
    flex_angles: int = 16
    flex_passes: int = 2
    keep_top: int = 4
    min_score: float = -1e30
    rotation_seed: int = 0x5EED
    write_all_poses: bool = False
    polish: int = 1  # 0 off, 1 rigid compass, 2 + fine torsion pass (SWEEP_V1.md §3.5)

    def as_c(self) -> _capi.vs_dock_params:
        p = _capi.vs_dock_params()
        p.restarts, p.rotations = self.restarts, self.rotations
        p.flex_angles, p.flex_passes = self.flex_angles, self.flex_passes
        p.diversity_delta, p.keep_top = self.diversity_delta, self.keep_top
        p.write_all_poses = 1 if self.write_all_poses else 0
        p.min_score, p.rotation_seed = self.min_score, self.rotation_seed
        p.polish = self.polish
        return p


POSE_DTYPE = np.dtype([("t", np.float32, 3), ("q", np.float32, 4), ("score", np.float32),
                       ("rescore", np.float32), ("restart", np.int16), ("attempt", np.int16),
                       ("rot", np.int16), ("reserved", np.int16)])
assert POSE_DTYPE.itemsize == C.sizeof(_capi.vs_pose)


@dataclass
class DockResults:
    best: np.ndarray          # (n,) float32, -inf when dropped
    n_kept: np.ndarray        # (n,) int32, -1 = out of every size class
    n_surv: np.ndarray
    surv: np.ndarray          # (n, keep_top) POSE_DTYPE
    surv_tors: np.ndarray
    keys: np.ndarray          # (n,) uint64
    all: np.ndarray | None = None
    all_tors: np.ndarray | None = None
    tors_off: np.ndarray | None = None
    keep_top: int = 0
    restarts: int = 0

    def poses(self, i: int, n_tors: int, which: str = "surv", ligand_id: str = "") -> list[Pose]:
        if which == "surv":
            cnt, rec, tors, slots = int(self.n_surv[i]), self.surv[i], self.surv_tors, self.keep_top
        else:
            cnt, rec, tors, slots = int(self.n_kept[i]), self.all[i], self.all_tors, self.restarts
        out = []
        base = int(self.tors_off[i]) * slots
        for s in range(max(cnt, 0)):
            r = rec[s]
            th = [float(v) for v in tors[base + s * n_tors: base + (s + 1) * n_tors]]
            resc = float(r["rescore"]) if (which == "surv" or s < int(self.n_surv[i])) else None
            out.append(Pose(ligand_id, tuple(float(v) for v in r["t"]),
                            tuple(float(v) for v in r["q"]), th, float(r["score"]), resc,
                            int(r["restart"]), int(r["attempt"]), int(r["rot"])))
        return out


def key_score(key: int) -> float:
    return float(_lib.vs_key_score(int(key)))


def key_id_rank(key: int) -> int:
    return int(_lib.vs_key_id_rank(int(key)))


# ---------------------------------------------------------------- engine ---
def _check_pose_arrays(lib: Library, pose_lig: np.ndarray, t: np.ndarray, q: np.ndarray,
                       tors: np.ndarray) -> None:
    """Sizes of flattened pose arrays against the library before they cross
    the C-ABI, which sizes its copies from pose_lig and the library: t[3n],
    q[4n], ligand indices in range, and the torsions of every pose's ligand
    (check_counts, dock.cpp:219-230)."""
    n = len(pose_lig)
    if t.size != 3 * n or q.size != 4 * n:
        raise ValueError(f"{n} poses need t of {3 * n} and q of {4 * n} values "
                         f"(got {t.size} and {q.size})")
    if n and (int(pose_lig.min()) < 0 or int(pose_lig.max()) >= len(lib)):
        raise ValueError("pose ligand index out of range")
    need = int(np.asarray(lib.n_tors, np.int64)[pose_lig].sum()) if n else 0
    if tors.size != need:
        raise AtomCountMismatch(f"poses need {need} torsion values, got {tors.size}")


class _PinnedOwner:
    def __init__(self, p: int):
        self.p = p

    def __del__(self):
        try:
            _lib.vs_host_free(C.c_void_p(self.p))
        except Exception:
            pass


def pinned_empty(shape, dtype) -> np.ndarray:
    """An uninitialised numpy array in page-locked host memory (capi.h
    vs_host_alloc); the memory is freed with the array's last view."""
    dtype = np.dtype(dtype)
    shape = (shape,) if np.isscalar(shape) else tuple(shape)
    nbytes = int(np.prod(shape, dtype=np.int64)) * dtype.itemsize
    p = C.c_void_p()
    check(_lib.vs_host_alloc(max(nbytes, 1), C.byref(p)), None, "pinned host allocation")
    buf = (C.c_uint8 * max(nbytes, 1)).from_address(p.value)
    buf._owner = _PinnedOwner(p.value)
    return np.frombuffer(buf, np.uint8, count=nbytes).view(dtype).reshape(shape)


class Engine:
    """One GPU handle (vs_handle): pocket + resident library + results."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(_lib.vs_create(device, C.byref(h)), None, f"vs_create(device={device})")
        self._h = h
        self.device = device
        self._lib = None
        self._prm = None
        self.pocket = None

    def close(self):
        if getattr(self, "_h", None):
            _lib.vs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def device_info(self) -> dict:
        name = C.create_string_buffer(256)
        sms, clk = C.c_int32(), C.c_int32()
        _lib.vs_device_info(self._h, name, C.byref(sms), C.byref(clk))
        return {"name": name.value.decode(), "sm_count": sms.value, "clock_khz": clk.value}

    def set_pocket(self, pocket: Pocket, grid_spacing: float = 0.0, grid_pad: float = 2.0):
        cp = pocket.as_c()
        check(_lib.vs_set_pocket(self._h, C.byref(cp), grid_spacing, grid_pad), self._h, "set_pocket")
        self.pocket = pocket

    def grid_maps(self):
        dims = (C.c_int32 * 3)()
        origin = (C.c_float * 3)()
        sp = C.c_float()
        check(_lib.vs_grid_info(self._h, dims, origin, C.byref(sp)), self._h, "grid_info")
        n = dims[0] * dims[1] * dims[2]
        maps = [np.zeros(n, np.float32) for _ in range(3)]
        check(_lib.vs_grid_fetch(self._h, *(ptr(m, C.c_float) for m in maps)), self._h, "grid_fetch")
        shape = (dims[2], dims[1], dims[0])
        return ([m.reshape(shape) for m in maps], tuple(origin), sp.value)

    def upload(self, lib: Library, classes=None):
        cl, ncl = _classes_c(classes)
        self._lib_c = lib.as_c()
        check(_lib.vs_upload_library(self._h, C.byref(self._lib_c), cl, ncl), self._h, "upload")
        self._lib = lib

    def dock(self, params: DockParams, stream: int | None = None):
        self._prm_c = params.as_c()
        check(_lib.vs_dock(self._h, C.byref(self._prm_c), C.c_void_p(stream or 0)), self._h, "dock")
        self._prm = params

    def fetch(self, out: DockResults | None = None) -> DockResults:
        """The last dock's results (into `out` from alloc_results, if given)."""
        return self._fetch(self._lib, self._prm, out)

    @staticmethod
    def alloc_results(lib: Library, prm: DockParams, pinned: bool = False) -> DockResults:
        """Result buffers for docking `lib` with `prm`; pinned=True places
        them in page-locked memory (pinned_empty), so vs_dock_host /
        vs_fetch_results DMA straight into them.  Pass them back as
        dock_host(..., out=) to reuse them across calls."""
        n, tt = len(lib), int(np.sum(lib.n_tors))
        kt, R = max(prm.keep_top, 1), prm.restarts
        mk = pinned_empty if pinned else (lambda shape, dt: np.zeros(shape, dt))
        res = DockResults(best=mk(max(n, 1), np.float32), n_kept=mk(max(n, 1), np.int32),
                          n_surv=mk(max(n, 1), np.int32), surv=mk((max(n, 1), kt), POSE_DTYPE),
                          surv_tors=mk(max(tt * kt, 1), np.float32), keys=mk(max(n, 1), np.uint64),
                          tors_off=np.concatenate([[0], np.cumsum(lib.n_tors, dtype=np.int64)]),
                          keep_top=prm.keep_top, restarts=R)
        if prm.write_all_poses:
            res.all = mk((max(n, 1), R), POSE_DTYPE)
            res.all_tors = mk(max(tt * R, 1), np.float32)
        return res

    def _alloc(self, lib: Library, prm: DockParams, out: DockResults | None = None):
        if out is None:
            res = self.alloc_results(lib, prm)
        else:
            n, tt = len(lib), int(np.sum(lib.n_tors))
            kt = max(prm.keep_top, 1)
            if (len(out.best) < n or out.surv.shape[1:] != (kt,) or len(out.surv) < n
                    or out.surv_tors.size < tt * kt or out.restarts != prm.restarts
                    or (prm.write_all_poses and out.all is None)):
                raise ValueError("out= buffers do not fit this library and parameters")
            res = out
        r = _capi.vs_results()
        r.best = ptr(res.best, C.c_float)
        r.n_kept = ptr(res.n_kept, C.c_int32)
        r.n_surv = ptr(res.n_surv, C.c_int32)
        r.surv = res.surv.ctypes.data_as(C.c_void_p)
        r.surv_tors = ptr(res.surv_tors, C.c_float)
        r.keys = ptr(res.keys, C.c_uint64)
        if prm.write_all_poses:
            r.all = res.all.ctypes.data_as(C.c_void_p)
            r.all_tors = ptr(res.all_tors, C.c_float)
        return res, r

    def _fetch(self, lib, prm, out=None):
        res, r = self._alloc(lib, prm, out)
        check(_lib.vs_fetch_results(self._h, C.byref(r)), self._h, "fetch")
        return _trim(res, len(lib))

    def dock_host(self, lib: Library, params: DockParams, classes=None,
                  out: DockResults | None = None, prefetch: Library | None = None) -> DockResults:
        """Upload + dock + fetch in one C-ABI call (host buffers in and out);
        out: result buffers from alloc_results to write into (reused);
        prefetch: the library of the next call, moved to the device under
        this dock (capi.h vs_dock_host_prefetch; keep it unchanged until
        then)."""
        cl, ncl = _classes_c(classes)
        lc = lib.as_c()
        pc = params.as_c()
        res, r = self._alloc(lib, params, out)
        if prefetch is not None:
            nc_ = prefetch.as_c()
            self._prefetch_keep = (prefetch, nc_)  # its arrays stay referenced until used
            check(_lib.vs_dock_host_prefetch(self._h, C.byref(lc), C.byref(nc_), cl, ncl,
                                             C.byref(pc), C.byref(r)), self._h, "dock_host")
        else:
            check(_lib.vs_dock_host(self._h, C.byref(lc), cl, ncl, C.byref(pc), C.byref(r)),
                  self._h, "dock_host")
        self._lib, self._prm = lib, params
        return _trim(res, len(lib))

    def topk(self, k: int) -> np.ndarray:
        out = np.zeros(k, np.uint64)
        check(_lib.vs_topk(self._h, k, ptr(out, C.c_uint64)), self._h, "topk")
        return out

    def topk_device(self, k: int, out_ptr: int, stream: int | None = None):
        check(_lib.vs_topk_device(self._h, k, C.c_void_p(out_ptr), C.c_void_p(stream or 0)),
              self._h, "topk_device")

    def topk_merge_device(self, keys_ptr: int, n: int, k: int, out_ptr: int,
                          stream: int | None = None):
        check(_lib.vs_topk_merge_device(self._h, C.c_void_p(keys_ptr), n, k, C.c_void_p(out_ptr),
                                        C.c_void_p(stream or 0)), self._h, "topk_merge")

    # ---- multi-GPU: NCCL top-k gather (capi.h vs_comm_init / vs_topk_allgather)
    def comm_init(self, nranks: int, rank: int, unique_id: bytes):
        """Join an NCCL communicator of `nranks` handles (one per GPU);
        unique_id = nccl_unique_id() of rank 0, broadcast by the caller."""
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(unique_id))
        check(_lib.vs_comm_init(self._h, nranks, rank, buf), self._h, "comm_init")

    def comm_attach(self, comm_ptr: int):
        check(_lib.vs_comm_attach(self._h, C.c_void_p(comm_ptr)), self._h, "comm_attach")

    def topk_allgather(self, k: int, out_ptr: int, stream: int | None = None, comm_ptr: int = 0):
        """Local top-k -> ncclAllGather of k keys per rank -> device merge,
        on `stream`; out_ptr: k device u64 keys (identical on every rank)."""
        check(_lib.vs_topk_allgather(self._h, C.c_void_p(comm_ptr or 0), k, C.c_void_p(out_ptr),
                                     C.c_void_p(stream or 0)), self._h, "topk_allgather")

    def start_draws(self, seeds, n_tors, restarts: int, attempts: int) -> np.ndarray:
        """FP32 restart start draws of the device dock (capi.h
        vs_start_draws): array [n, restarts, attempts, 7 + max T] of
        t(3), q(4), theta(T)."""
        seeds = np.ascontiguousarray(seeds, np.uint64)
        n_tors = np.ascontiguousarray(n_tors, np.int32)
        n = len(seeds)
        stride = 7 + (int(n_tors.max()) if n else 0)
        out = np.zeros(max(n * restarts * attempts * stride, 1), np.float32)
        check(_lib.vs_start_draws(self._h, ptr(seeds, C.c_uint64), ptr(n_tors, C.c_int32), n,
                                  restarts, attempts, stride, ptr(out, C.c_float)),
              self._h, "start_draws")
        return out[:n * restarts * attempts * stride].reshape(n, restarts, attempts, stride)

    def last_dock_ms(self) -> float:
        return float(_lib.vs_last_dock_ms(self._h))

    def last_rescore_ms(self) -> float:
        """Device ms of the rescore kernels of the last rescore() call."""
        return float(_lib.vs_last_rescore_ms(self._h))

    def launch_count(self) -> int:
        return int(_lib.vs_launch_count(self._h))

    def phase_ms(self) -> dict:
        """Device ms of the last dock per kernel (capi.h vs_last_phase_ms)."""
        out = (C.c_double * 4)()
        check(_lib.vs_last_phase_ms(self._h, out), self._h, "phase_ms")
        return dict(zip(("start", "sweep", "flex", "finish"), (float(v) for v in out)))

    def phase_ms_ex(self) -> dict:
        """Device ms of the last dock per kernel with the polish kernel on its
        own (capi.h vs_last_phase_ms_ex)."""
        out = (C.c_double * 5)()
        k = _lib.vs_last_phase_ms_ex(self._h, out, 5)
        if k < 0:
            check(k, self._h, "phase_ms_ex")
        return dict(zip(("start", "sweep", "flex", "finish", "polish"), (float(v) for v in out)))

    def measure_gather_peak(self) -> float:
        """Measured random 16 B gather rate (loads/s, capi.h vs_measure_gather_peak)."""
        v = C.c_double()
        check(_lib.vs_measure_gather_peak(self._h, C.byref(v)), self._h, "gather_peak")
        return v.value

    def measure_l2_gather_peak(self) -> float:
        """Measured random 32 B (one sector) gather rate from L2, bytes/s:
        the L2-gather roof of SURVEY §8(d) (capi.h vs_measure_gather_peak_ex)."""
        v = C.c_double()
        check(_lib.vs_measure_gather_peak_ex(self._h, 32, C.byref(v)), self._h, "gather_peak")
        return 32.0 * v.value

    def stats(self) -> dict:
        """Work counters of the last dock (capi.h vs_last_stats)."""
        out = np.zeros(10, np.uint64)
        check(_lib.vs_last_stats_ex(self._h, ptr(out, C.c_uint64), 10), self._h, "stats")
        cyc = [int(v) for v in out[4:8]]
        tot = max(sum(cyc), 1)
        return {"translation_iters": int(out[0]), "translation_iter_atoms": int(out[1]),
                "start_attempts": int(out[2]), "active_pairs": int(out[3]),
                "post_compass_iters": int(out[8]), "post_compass_iter_atoms": int(out[9]),
                "phase_cycle_share": {k: round(c / tot, 4) for k, c in
                                      zip(("start", "sweep", "flex", "keep"), cyc)}}

    def measure_peaks(self) -> dict:
        """Measured FP32 / FP64 FMA (flop/s) and MUFU ex2 (op/s) peaks."""
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        check(_lib.vs_measure_peaks(self._h, C.byref(a), C.byref(b), C.byref(c)), self._h, "peaks")
        return {"fp32_flops": a.value, "fp64_flops": b.value, "xu_ops": c.value}

    def score_gradient(self, lib: Library, pose_lig, t, q, tors):
        """FP64 score_gradient of given poses (capi.h vs_score_gradient):
        (score[n], grad_t[n, 3], grad_q[n, 4], grad_tors[sum T])."""
        pose_lig = np.ascontiguousarray(pose_lig, np.int32)
        n = len(pose_lig)
        t = np.ascontiguousarray(t, np.float64).reshape(-1)
        q = np.ascontiguousarray(q, np.float64).reshape(-1)
        tors = np.ascontiguousarray(tors, np.float64).reshape(-1)
        _check_pose_arrays(lib, pose_lig, t, q, tors)
        nt = tors.size
        if nt == 0:
            tors = np.zeros(1, np.float64)
        score = np.zeros(max(n, 1), np.float64)
        gt = np.zeros(max(n, 1) * 3, np.float64)
        gq = np.zeros(max(n, 1) * 4, np.float64)
        gtor = np.zeros(max(nt, 1), np.float64)
        lc = lib.as_c()
        check(_lib.vs_score_gradient(self._h, C.byref(lc), n, ptr(pose_lig, C.c_int32),
                                     ptr(t, C.c_double), ptr(q, C.c_double), ptr(tors, C.c_double),
                                     ptr(score, C.c_double), ptr(gt, C.c_double),
                                     ptr(gq, C.c_double), ptr(gtor, C.c_double)),
              self._h, "score_gradient")
        return score[:n], gt[:3 * n].reshape(n, 3), gq[:4 * n].reshape(n, 4), gtor[:nt]

    def ascend(self, lib: Library, pose_lig, t, q, tors, max_steps: int = 500):
        """The reference ascent on the device (capi.h vs_ascend): returns the
        refined (t[n, 3], q[n, 4], tors, score[n], steps[n]) in FP64."""
        pose_lig = np.ascontiguousarray(pose_lig, np.int32)
        n = len(pose_lig)
        t = np.array(t, np.float64).reshape(-1).copy()
        q = np.array(q, np.float64).reshape(-1).copy()
        tors = np.array(tors, np.float64).reshape(-1).copy()
        _check_pose_arrays(lib, pose_lig, t, q, tors)
        nt = tors.size
        if nt == 0:
            tors = np.zeros(1, np.float64)
        score = np.zeros(max(n, 1), np.float64)
        steps = np.zeros(max(n, 1), np.int32)
        lc = lib.as_c()
        check(_lib.vs_ascend(self._h, C.byref(lc), n, ptr(pose_lig, C.c_int32), ptr(t, C.c_double),
                             ptr(q, C.c_double), ptr(tors, C.c_double), max_steps,
                             ptr(score, C.c_double), ptr(steps, C.c_int32)), self._h, "ascend")
        return t[:3 * n].reshape(n, 3), q[:4 * n].reshape(n, 4), tors[:nt], score[:n], steps[:n]

    def score64(self, lib: Library, pose_lig, t, q, tors):
        """geometric_score and rescore of given poses in FP64 on the device
        (capi.h vs_score64): (geo[n], resc[n])."""
        pose_lig = np.ascontiguousarray(pose_lig, np.int32)
        n = len(pose_lig)
        t = np.ascontiguousarray(t, np.float64).reshape(-1)
        q = np.ascontiguousarray(q, np.float64).reshape(-1)
        tors = np.ascontiguousarray(tors, np.float64).reshape(-1)
        _check_pose_arrays(lib, pose_lig, t, q, tors)
        if tors.size == 0:
            tors = np.zeros(1, np.float64)
        geo = np.zeros(max(n, 1), np.float64)
        resc = np.zeros(max(n, 1), np.float64)
        lc = lib.as_c()
        check(_lib.vs_score64(self._h, C.byref(lc), n, ptr(pose_lig, C.c_int32), ptr(t, C.c_double),
                              ptr(q, C.c_double), ptr(tors, C.c_double), ptr(geo, C.c_double),
                              ptr(resc, C.c_double)), self._h, "score64")
        return geo[:n], resc[:n]

    def dock_refined(self, lib: Library, params: DockParams, max_steps: int = 500, classes=None):
        """dock() with the reference contract (capi.h vs_dock_refined_host):
        sweep-v1 restarts refined by the reference ascent, the keep rule on
        the refined poses, sorted by score.  Returns per ligand a list of
        (t[3], q[4], torsions, score, restart) tuples (FP64)."""
        n, R = len(lib), params.restarts
        tt = int(np.sum(lib.n_tors))
        cl, ncl = _classes_c(classes)
        npos = np.zeros(max(n, 1), np.int32)
        t = np.zeros(max(n, 1) * R * 3)
        q = np.zeros(max(n, 1) * R * 4)
        th = np.zeros(max(tt, 1) * R)
        sc = np.zeros(max(n, 1) * R)
        rs = np.zeros(max(n, 1) * R, np.int32)
        out = _capi.vs_refined(ptr(npos, C.c_int32), ptr(t, C.c_double), ptr(q, C.c_double),
                               ptr(th, C.c_double), ptr(sc, C.c_double), ptr(rs, C.c_int32))
        lc, pc = lib.as_c(), params.as_c()
        check(_lib.vs_dock_refined_host(self._h, C.byref(lc), cl, ncl, C.byref(pc), max_steps,
                                        C.byref(out)), self._h, "dock_refined")
        _, to, _ = lib.offsets()
        res = []
        for i in range(n):
            T = int(lib.n_tors[i])
            res.append([(t[3 * (i * R + r):3 * (i * R + r) + 3], q[4 * (i * R + r):4 * (i * R + r) + 4],
                         th[to[i] * R + r * T:to[i] * R + (r + 1) * T], float(sc[i * R + r]),
                         int(rs[i * R + r])) for r in range(max(int(npos[i]), 0))])
        return res

    def rescore_device(self, n_poses: int, pose_lig_ptr: int, t_ptr: int, q_ptr: int,
                       tors_ptr: int, geo_ptr: int, resc_ptr: int, stream: int | None = None):
        """K3a over poses already in device memory (capi.h vs_rescore_device),
        against the resident library; all pointers are device pointers."""
        check(_lib.vs_rescore_device(self._h, n_poses, C.c_void_p(pose_lig_ptr), C.c_void_p(t_ptr),
                                     C.c_void_p(q_ptr), C.c_void_p(tors_ptr), C.c_void_p(geo_ptr),
                                     C.c_void_p(resc_ptr), C.c_void_p(stream or 0)),
              self._h, "rescore_device")

    def rescore_survivors(self, geo_ptr: int, resc_ptr: int, stream: int | None = None):
        """The last dock's survivors re-scored in device memory against the
        current pocket (capi.h vs_rescore_survivors): device arrays
        [n * keep_top]."""
        check(_lib.vs_rescore_survivors(self._h, C.c_void_p(geo_ptr), C.c_void_p(resc_ptr),
                                        C.c_void_p(stream or 0)), self._h, "rescore_survivors")

    def rescore(self, lib: Library, pose_lig, t, q, tors, out=None):
        """K3a: canonical geometric score and rescore of given poses; out:
        (geo, resc) float32 arrays of >= n poses to write into (e.g.
        pinned_empty buffers, which the scores are DMA'd straight into)."""
        pose_lig = np.ascontiguousarray(pose_lig, np.int32)
        t = np.ascontiguousarray(t, np.float32).reshape(-1)
        q = np.ascontiguousarray(q, np.float32).reshape(-1)
        tors = np.ascontiguousarray(tors, np.float32).reshape(-1)
        n = len(pose_lig)
        if t.size != 3 * n or q.size != 4 * n:
            raise ValueError(f"{n} poses need t of {3 * n} and q of {4 * n} values "
                             f"(got {t.size} and {q.size})")
        n_tors_values = tors.size  # checked against the poses' ligands in C
        if tors.size == 0:
            tors = np.zeros(1, np.float32)
        if out is not None:
            geo, resc = out
            if (geo.dtype != np.float32 or resc.dtype != np.float32 or len(geo) < max(n, 1)
                    or len(resc) < max(n, 1) or not geo.flags.c_contiguous
                    or not resc.flags.c_contiguous):
                raise ValueError("out= needs two contiguous float32 arrays of >= n poses")
        else:
            geo = np.zeros(max(n, 1), np.float32)
            resc = np.zeros(max(n, 1), np.float32)
        lc = lib.as_c()
        check(_lib.vs_rescore_checked(self._h, C.byref(lc), n, ptr(pose_lig, C.c_int32),
                                      ptr(t, C.c_float), ptr(q, C.c_float), ptr(tors, C.c_float),
                                      n_tors_values, ptr(geo, C.c_float), ptr(resc, C.c_float)),
              self._h, "rescore")
        return geo[:n], resc[:n]


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId of the NCCL the process has (capi.h vs_nccl_unique_id)."""
    buf = (C.c_uint8 * 128)()
    check(_lib.vs_nccl_unique_id(buf), None, "nccl_unique_id")
    return bytes(buf)


def _classes_c(classes):
    if not classes:
        return None, 0
    arr = (_capi.vs_size_class * len(classes))()
    for i, c in enumerate(classes):
        arr[i].atom_lo, arr[i].atom_hi = c[0], c[1]
        arr[i].rot_lo, arr[i].rot_hi = c[2], c[3]
    return arr, len(classes)


def _trim(res: DockResults, n: int) -> DockResults:
    res.best, res.n_kept, res.n_surv = res.best[:n], res.n_kept[:n], res.n_surv[:n]
    res.surv, res.keys = res.surv[:n], res.keys[:n]
    if res.all is not None:
        res.all = res.all[:n]
    return res


_ENGINES: dict[int, Engine] = {}


def default_engine(device: int = 0) -> Engine:
    e = _ENGINES.get(device)
    if e is None:
        e = _ENGINES[device] = Engine(device)
    return e


# ------------------------------------------------- single-ligand drop-ins ---
def _one_ligand_library(conf: Conformer, topo: TorsionTopology, classes=None, seed: int = 0,
                        atom_class=None) -> Library:
    n = len(conf.coords)
    for ax in topo.axes:
        if ax.a >= n or ax.b >= n:
            raise AtomCountMismatch("torsion topology does not fit conformer")
    cls = np.zeros(n, np.int32) if atom_class is None else np.asarray(atom_class, np.int32)
    mv = [m for ax in topo.axes for m in ax.moving]
    return Library(ids=[conf.ligand_id or "x"], n_atoms=np.array([n], np.int32),
                   n_tors=np.array([len(topo.axes)], np.int32),
                   rot_bonds=np.array([len(topo.axes)], np.int32),
                   coords=np.asarray(conf.coords, np.float64).reshape(-1, 3), atom_class=cls,
                   axis_a=np.array([a.a for a in topo.axes], np.int32),
                   axis_b=np.array([a.b for a in topo.axes], np.int32),
                   moving_count=np.array([len(a.moving) for a in topo.axes], np.int32),
                   moving=np.array(mv, np.int32), seeds=np.array([seed & (2**64 - 1)], np.uint64),
                   id_rank=np.zeros(1, np.uint32))


def _check_counts(conf: Conformer, topo: TorsionTopology, pose: Pose):
    # dock.cpp:219-230
    if len(pose.torsions) != len(topo.axes):
        raise AtomCountMismatch(f"pose has {len(pose.torsions)} torsions, topology has "
                                f"{len(topo.axes)}")
    n = len(conf.coords)
    for ax in topo.axes:
        if ax.a >= n or ax.b >= n:
            raise AtomCountMismatch("torsion topology does not fit conformer")


def _score(conf, topo, poses, pocket, atom_class, engine=None):
    eng = engine or default_engine()
    if eng.pocket is not pocket:
        eng.set_pocket(pocket)
    if not len(conf.coords):
        raise AtomCountMismatch("conformer has no atoms")
    lib = _one_ligand_library(conf, topo, atom_class=atom_class)
    n = len(poses)
    t = np.array([p.translation for p in poses], np.float64)
    q = np.array([p.rotation for p in poses], np.float64)
    tors = np.array([v for p in poses for v in p.torsions], np.float64)
    return eng.score64(lib, np.zeros(n, np.int32), t, q, tors)


def geometric_score(conf: Conformer, topo: TorsionTopology, pose: Pose, pocket: Pocket,
                    engine: Engine | None = None) -> float:
    """dock::geometric_score (dock.cpp:278-282) on the GPU (canonical FP32)."""
    _check_counts(conf, topo, pose)
    return float(_score(conf, topo, [pose], pocket, None, engine)[0][0])


@dataclass
class ScoreGradient:
    """dock::ScoreGradient (dock.hpp:86-91)."""
    score: float
    translation: tuple
    rotation: tuple  # d/d(w, x, y, z)
    torsions: list


def score_gradient(conf: Conformer, topo: TorsionTopology, pose: Pose, pocket: Pocket,
                   engine: Engine | None = None) -> ScoreGradient:
    """dock::score_gradient (dock.cpp:284-295) on the GPU in FP64: analytic
    translation / rotation derivatives, central differences for torsions."""
    _check_counts(conf, topo, pose)
    if pocket.empty():
        raise EmptyBounds()
    eng = engine or default_engine()
    if eng.pocket is not pocket:
        eng.set_pocket(pocket)
    if not len(conf.coords):
        raise AtomCountMismatch("conformer has no atoms")
    lib = _one_ligand_library(conf, topo)
    s, gt, gq, gtor = eng.score_gradient(lib, np.zeros(1, np.int32), [pose.translation],
                                         [pose.rotation], list(pose.torsions))
    return ScoreGradient(float(s[0]), tuple(float(v) for v in gt[0]),
                         tuple(float(v) for v in gq[0]), [float(v) for v in gtor])


def rescore(ligand: Ligand, conf: Conformer, topo: TorsionTopology, pose: Pose, pocket: Pocket,
            engine: Engine | None = None) -> float:
    """dock::rescore (dock.cpp:297-316) on the GPU."""
    if ligand.heavy_atoms != len(conf.coords):
        raise AtomCountMismatch("graph and conformer disagree on atom count")
    _check_counts(conf, topo, pose)
    return float(_score(conf, topo, [pose], pocket, ligand.atom_classes(), engine)[1][0])


def dock(conf: Conformer, topo: TorsionTopology, pocket: Pocket, restarts: int,
         diversity_delta: float, seed: int, max_steps: int = 500, params: DockParams | None = None,
         engine: Engine | None = None, atom_class=None) -> list[Pose]:
    """dock::dock (dock.cpp:318-371): the sweep-v1 restarts refined by the
    reference ascent (max_steps, FP64 on the device), the reference's keep
    rule on the refined poses (pairwise RMSD >= diversity_delta, restart
    order) and a stable sort by geometric score descending
    (capi.h vs_dock_refined_host)."""
    if pocket.empty():
        raise EmptyBounds()
    if restarts < 1:
        raise ValueError("restarts must be >= 1")
    if diversity_delta < 0.0:
        raise ValueError("diversity_delta must be >= 0")
    if not len(conf.coords):
        raise AtomCountMismatch("conformer has no atoms")
    prm = params or DockParams()
    prm = DockParams(restarts=restarts, diversity_delta=diversity_delta, rotations=prm.rotations,
                     flex_angles=prm.flex_angles, flex_passes=prm.flex_passes,
                     keep_top=prm.keep_top, min_score=prm.min_score,
                     rotation_seed=prm.rotation_seed, polish=prm.polish)
    eng = engine or default_engine()
    if eng.pocket is not pocket:
        eng.set_pocket(pocket)
    lib = _one_ligand_library(conf, topo, seed=seed, atom_class=atom_class)
    (poses,) = eng.dock_refined(lib, prm, max_steps)
    return [Pose(conf.ligand_id, tuple(float(v) for v in t), tuple(float(v) for v in q),
                 [float(v) for v in th], sc, None, restart=r) for (t, q, th, sc, r) in poses]


def filter_poses(poses: Sequence[Pose], keep_top: int, min_score: float) -> list[Pose]:
    """dock::filter_poses (dock.cpp:373-390), via the native host function."""
    scores = np.array([p.geometric_score for p in poses], np.float64)
    out = np.zeros(max(len(poses), 1), np.int32)
    n = _lib.vs_filter_poses(ptr(scores, C.c_double), len(poses), int(min(keep_top, 2**62)),
                             float(min_score), ptr(out, C.c_int32))
    return [poses[i] for i in out[:n]]


def rmsd(a, b) -> float:
    """dock::rmsd (dock.cpp:392-401): no alignment."""
    a = np.asarray(a, np.float64).reshape(-1, 3)
    b = np.asarray(b, np.float64).reshape(-1, 3)
    if len(a) != len(b):
        raise LengthMismatch(f"coordinate sets have different lengths: {len(a)} vs {len(b)}")
    if len(a) == 0:
        return 0.0
    s = 0.0
    for (ax, ay, az), (bx, by, bz) in zip(a.tolist(), b.tolist()):
        dx, dy, dz = ax - bx, ay - by, az - bz
        s += dx * dx + dy * dy + dz * dz
    return math.sqrt(s / len(a))


def apply_pose(conf: Conformer, topo: TorsionTopology, pose: Pose) -> np.ndarray:
    """dock::apply_pose (dock.cpp:52-67, 272-276) in FP64 on the host."""
    _check_counts(conf, topo, pose)
    pts = [list(map(float, p)) for p in np.asarray(conf.coords, np.float64).reshape(-1, 3)]

    def qrot(w, x, y, z, v):
        ux, uy, uz = x, y, z
        cx, cy, cz = uy * v[2] - uz * v[1], uz * v[0] - ux * v[2], ux * v[1] - uy * v[0]
        dx, dy, dz = uy * cz - uz * cy, uz * cx - ux * cz, ux * cy - uy * cx
        return [v[0] + 2.0 * w * cx + 2.0 * dx, v[1] + 2.0 * w * cy + 2.0 * dy,
                v[2] + 2.0 * w * cz + 2.0 * dz]

    for j, ax in enumerate(topo.axes):
        o = pts[ax.a]
        d = [pts[ax.b][k] - o[k] for k in range(3)]
        n = math.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
        u = [v / n for v in d] if n > 0 else [0.0, 0.0, 0.0]
        h = 0.5 * pose.torsions[j]
        s = math.sin(h)
        for idx in ax.moving:
            r = qrot(math.cos(h), u[0] * s, u[1] * s, u[2] * s,
                     [pts[idx][k] - o[k] for k in range(3)])
            pts[idx] = [o[k] + r[k] for k in range(3)]
    w, x, y, z = pose.rotation
    n = math.sqrt(w * w + x * x + y * y + z * z)
    w, x, y, z = w / n, x / n, y / n, z / n
    return np.array([[a + b for a, b in zip(qrot(w, x, y, z, p), pose.translation)] for p in pts])


def pose_rmsd(conf: Conformer, topo: TorsionTopology, a: Pose, b: Pose) -> float:
    """dock::pose_rmsd (dock.cpp:403-406)."""
    return rmsd(apply_pose(conf, topo, a), apply_pose(conf, topo, b))
