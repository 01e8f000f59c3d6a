"""The dock funnel of run_campaign on the B200 path.

`run_dock_stages` runs the parse -> embed -> dock -> rescore -> filter -> rank
stages of `pipeline::run_campaign` (proj/src/pipeline.cpp:380-537) from the
reference's campaign JSON (`parse_config_json`, pipeline.cpp:76-160), with the
dock, rescore, filter and best-score stages in one GPU pass and the ranking
as the device top-k.  What it keeps from the reference, exactly:

- parse: records of `read_library_file`, unparsable lines skipped, duplicate
  ids rejected (pipeline.cpp:381-416);
- embed: seed `Rng(seed).split(1).split(i)` over the parsed ligands, the
  reference `embed_3d` bit for bit (:418-429);
- dock: ligands outside every size class dropped, the `BatchQueue` replay
  with its `dock.b{bi}` tasks and their simulated durations (:433-473), dock
  seed `Rng(seed).split(2).split(i)` over the in-class ligands (:480-484);
- filter / rank: `filter_poses(keep_top, min_score)`, best = max rescore,
  ligands without a surviving pose dropped, `rank_ligands` order and
  keep = min(n, max(1, floor(keep_after_dock * n))) (:502-537);
- the stage records {name, in, out, sim_seconds, tasks} of the report.

What it does not do: `sim_seconds` of the dock stage is the cluster
scheduler simulation (`sched::run_simulation`, out of scope here): the
stage carries the tasks instead so a caller's scheduler can replay them.
Compressed (.smzc) libraries decode through codec.decompress_file.  The
pose generator is sweep-v1 (docs/SWEEP_V1.md), so the ranked scores are
sweep-v1's, not the gradient ascent's.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

from ._capi import lib as _lib, ptr
from .batcher import DeviceModel, SizeClass, bucket_replay, default_classes
from .chem import build_library, read_library_file
from .dock import DockParams, Engine, load_pocket_file
from .errors import VscreenError
from .pipeline import RankedLigand, campaign_seeds, keep_count, rank_ligands


class ConfigError(VscreenError):
    """pipeline::ConfigError (pipeline.hpp)."""


@dataclass
class StageKnobs:
    """pipeline::StageKnobs (pipeline.hpp:33-40)."""
    embed_iterations: int = 200
    restarts: int = 4
    diversity_delta: float = 1.0
    keep_top: int = 4
    min_score: float = -1e30
    ls_max_steps: int = 500


@dataclass
class CampaignConfig:
    """The dock-funnel fields of pipeline::CampaignConfig (pipeline.hpp:42-65)."""
    library_path: str = ""
    dictionary_path: str = ""
    pocket_path: str = ""
    keep_after_dock: float = 0.2
    keep_for_fep: float = 0.5
    knobs: StageKnobs = field(default_factory=StageKnobs)
    device: DeviceModel = field(default_factory=DeviceModel)
    classes: list = field(default_factory=list)
    master_seed: int = 0
    threads: int = 1
    top_n: int = 10
    trace_path: str = "campaign_trace.jsonl"    # relative to the working directory
    report_path: str = "campaign_report.json"


@dataclass
class StageStats:
    """pipeline::StageStats (pipeline.hpp:71-77)."""
    name: str
    in_: int = 0
    out: int = 0
    sim_seconds: float | None = 0.0
    tasks: int = 0

    def to_json(self) -> dict:
        return {"name": self.name, "in": self.in_, "out": self.out,
                "sim_seconds": self.sim_seconds, "tasks": self.tasks}


@dataclass
class DockTask:
    """sched::Task of the dock stage (pipeline.cpp:462-473)."""
    id: str
    duration_s: float
    cls: int
    ligand_ids: list


@dataclass
class DockFunnel:
    stages: list
    ranked: list          # kept RankedLigand, rank order
    tasks: list           # DockTask per batch
    ids: list             # docked ligand ids (in-class, post-compaction order)
    best: np.ndarray      # best rescore per docked ligand (-inf: no surviving pose)
    dock_ms: float


def _resolve(base_dir: str, path: str) -> str:
    """pipeline.cpp:57-60."""
    if not path or os.path.isabs(path) or not base_dir:
        return path
    return os.path.join(base_dir, path)


def parse_config_json(text: str, base_dir: str = "") -> CampaignConfig:
    """pipeline::parse_config_json (pipeline.cpp:76-160), dock-funnel fields;
    missing required keys raise ConfigError like the reference."""
    try:
        j = json.loads(text)
    except ValueError as e:
        raise ConfigError(f"bad campaign JSON: {e}") from e
    c = CampaignConfig()
    try:
        c.library_path = _resolve(base_dir, j["library"])
        c.dictionary_path = _resolve(base_dir, j.get("dictionary", ""))
        c.pocket_path = _resolve(base_dir, j["pocket"])
        c.keep_after_dock = float(j["funnel"]["keep_after_dock"])
        c.keep_for_fep = float(j["funnel"]["keep_for_fep"])
        k = j.get("knobs", {})
        d = StageKnobs()
        c.knobs = StageKnobs(int(k.get("embed_iterations", d.embed_iterations)),
                             int(k.get("restarts", d.restarts)),
                             float(k.get("diversity_delta", d.diversity_delta)),
                             int(k.get("keep_top", d.keep_top)),
                             float(k.get("min_score", d.min_score)),
                             int(k.get("ls_max_steps", d.ls_max_steps)))
        jd = j["device"]
        c.device = DeviceModel(float(jd["memory_capacity"]), float(jd.get("mem_fixed", 0.0)),
                               float(jd["mem_per_atom"]), float(jd["mem_per_rotbond"]),
                               float(jd["launch_overhead_s"]),
                               [float(v) for v in jd["service_time_per_class_s"]])
        if "classes" in j:
            c.classes = [SizeClass(int(x["atom_lo"]), int(x["atom_hi"]), int(x["rot_lo"]),
                                   int(x["rot_hi"])) for x in j["classes"]]
        else:
            c.classes = default_classes()
        c.master_seed = int(j.get("seed", 0))
        c.threads = int(j.get("threads", 1))
        c.top_n = int(j.get("top_n", 10))
        # output paths stay relative to the working directory (pipeline.cpp:151-154)
        c.trace_path = str(j.get("trace", c.trace_path))
        c.report_path = str(j.get("report", c.report_path))
    except (KeyError, TypeError) as e:
        raise ConfigError(f"bad campaign config: missing or invalid {e}") from e
    _validate(c)
    return c


def _validate(c: CampaignConfig) -> None:
    """validate_config (pipeline.cpp:162-178), the dock-funnel fields."""
    if not (0.0 < c.keep_after_dock <= 1.0):
        raise ConfigError("funnel.keep_after_dock must be in (0, 1]")
    if not (0.0 < c.keep_for_fep <= 1.0):
        raise ConfigError("funnel.keep_for_fep must be in (0, 1]")
    if c.threads < 1:
        raise ConfigError("threads must be >= 1")
    for label, p in (("library", c.library_path), ("pocket", c.pocket_path)):
        if not os.path.exists(p):
            raise ConfigError(f"{label} file not found: {p}")
    if c.dictionary_path and not os.path.exists(c.dictionary_path):
        raise ConfigError(f"dictionary file not found: {c.dictionary_path}")


def load_config_file(path: str) -> CampaignConfig:
    """pipeline::load_config_file (pipeline.cpp:180-188)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError as e:
        raise ConfigError(f"cannot open campaign config: {path}") from e
    return parse_config_json(text, os.path.dirname(path))


def prepare(cfg: CampaignConfig, threads: int | None = None):
    """parse + embed + the dock stage's class filter and batch replay (no
    GPU).  Returns (library of in-class ligands with their campaign seeds,
    stage records so far, dock tasks, dock-stage input count)."""
    threads = threads or max(1, cfg.threads)
    if cfg.library_path.endswith(".smzc"):  # pipeline.cpp:384-396
        if not cfg.dictionary_path:
            raise ConfigError("compressed library needs a dictionary")
        from .codec import decompress, load_dictionary_file
        d = load_dictionary_file(cfg.dictionary_path)
        try:
            with open(cfg.library_path, "rb") as f:
                data = f.read()
        except OSError as e:
            raise ConfigError(f"cannot open library: {cfg.library_path}") from e
        text = decompress(d, data, threads=os.cpu_count())
        from .chem import read_library_records
        records = read_library_records(text.split("\n") if text else [])
    else:
        records = read_library_file(cfg.library_path)
    smiles = [r.smiles for r in records]
    ids = [r.id for r in records]
    # parse: graph, descriptors and topology only (no embedding)
    probe = build_library(smiles, ids, iterations=-1, threads=threads, drop_failed=False)
    from . import _capi
    parsed = [i for i in range(len(records)) if probe.status[i] == 0]
    bad = [i for i in range(len(records))
           if probe.status[i] not in (0, _capi.VS_ERR_PARSE)]
    if bad:
        raise VscreenError(f"ligand {ids[bad[0]]}: graph cannot be embedded "
                           f"(status {int(probe.status[bad[0]])})")
    p_ids = [ids[i] for i in parsed]
    if len(set(p_ids)) != len(p_ids):
        raise ConfigError("duplicate ligand id in library")
    stages = [StageStats("parse", len(records), len(parsed), 0.0, 0)]
    # embed: seeds over the parsed ligands (pipeline.cpp:418-429)
    n = len(parsed)
    es = campaign_seeds(cfg.master_seed, n, stage=1)
    # dock: class filter + batch replay over the parsed ligands (:433-461)
    atoms = probe.n_atoms[parsed]
    rot = probe.rot_bonds[parsed]
    in_range, batches = bucket_replay(atoms, rot, cfg.classes, cfg.device)
    usable = np.nonzero(in_range)[0]
    ds = campaign_seeds(cfg.master_seed, len(usable), stage=2)
    sm = [smiles[parsed[i]] for i in usable]
    lib = build_library(sm, [p_ids[i] for i in usable], es[usable], ds,
                        iterations=cfg.knobs.embed_iterations, threads=threads)
    stages.append(StageStats("embed", n, n, 0.0, 0))
    tasks = []
    for bi, (cls, members) in enumerate(batches):
        tasks.append(DockTask(f"dock.b{bi}",
                              cfg.device.launch_overhead + len(members) * cfg.device.service_time(cls),
                              cls, [p_ids[m] for m in members]))
    return lib, stages, tasks, n


class _TraceWriter:
    """TraceWriter (pipeline.cpp:335-352): stage_start / stage_end JSONL
    lines.  The scheduler simulation's events (sched_events) are out of
    scope, so the dock stage carries none."""

    def __init__(self, path: str):
        if not path:
            self.f = None
            return
        try:
            parent = os.path.dirname(path)
            if parent:
                os.makedirs(parent, exist_ok=True)
            self.f = open(path, "wb")
        except OSError as e:
            raise ConfigError(f"cannot open trace for writing: {path}") from e

    def stage(self, kind: str, name: str):
        if self.f is not None:
            self.f.write(f'{{"kind":"stage_{kind}","stage":"{name}"}}\n'.encode())

    def close(self):
        if self.f is not None:
            self.f.close()


def run_dock_stages(cfg: CampaignConfig, engine: Engine | None = None, grid_spacing: float = 0.0,
                    params: DockParams | None = None, write_outputs: bool = False) -> DockFunnel:
    """parse -> embed -> dock -> rescore -> filter -> rank on one GPU.  The
    pocket is analytic by default (as the reference scores it); grid_spacing
    > 0 docks on the grid maps.  write_outputs: the trace (stage lines) at
    cfg.trace_path and the report bytes at cfg.report_path, as
    run_campaign writes them (pipeline.cpp:357-379, 586-590)."""
    trace = _TraceWriter(cfg.trace_path if write_outputs else "")
    try:
        trace.stage("start", "parse")
        lib, stages, tasks, n_dock_in = prepare(cfg)
        trace.stage("end", "parse")
        trace.stage("start", "embed")
        trace.stage("end", "embed")
        trace.stage("start", "dock")
        pocket = load_pocket_file(cfg.pocket_path)
        own = engine is None
        eng = engine or Engine(0)
        try:
            eng.set_pocket(pocket, grid_spacing=grid_spacing)
            k = cfg.knobs
            prm = params or DockParams(restarts=k.restarts, diversity_delta=k.diversity_delta,
                                       keep_top=k.keep_top, min_score=k.min_score)
            res = eng.dock_host(lib, prm, classes=[c.astuple() for c in cfg.classes])
            dock_ms = eng.last_dock_ms()
        finally:
            if own:
                eng.close()
        # tasks = batches; sim_seconds needs the scheduler simulation (None here)
        stages.append(StageStats("dock", n_dock_in, len(lib), None, len(tasks)))
        trace.stage("end", "dock")
        # rescore, filter and best ran inside the dock pass (K3a, keep rule)
        for name in ("rescore", "filter", "rank"):
            trace.stage("start", name)
            if name == "rescore":
                stages.append(StageStats("rescore", len(lib), len(lib), 0.0, 0))
            elif name == "filter":
                kept = np.nonzero(res.n_surv > 0)[0]
                stages.append(StageStats("filter", len(lib), len(kept), 0.0, 0))
            else:
                scores = {lib.ids[i]: float(res.best[i]) for i in kept}
                ranked = rank_ligands(scores)
                keep = min(keep_count(len(kept), cfg.keep_after_dock), len(ranked))
                stages.append(StageStats("rank", len(kept), keep, 0.0, 0))
            trace.stage("end", name)
    finally:
        trace.close()
    f = DockFunnel(stages, [RankedLigand(i, s) for i, s in ranked[:keep]], tasks,
                   list(lib.ids), res.best, dock_ms)
    if write_outputs:
        parent = os.path.dirname(cfg.report_path)
        if parent:
            os.makedirs(parent, exist_ok=True)
        with open(cfg.report_path, "wb") as out:
            out.write(funnel_to_json(f, cfg.trace_path).encode())
    return f


def dock_library_jsonl(library_path: str, pocket_path: str, out_path: str, restarts: int = 8,
                       diversity: float = 1.0, keep_top: int = 4, min_score: float = -1e30,
                       do_rescore: bool = False, seed: int = 0, threads: int | None = None,
                       engine: Engine | None = None, max_steps: int = 500) -> int:
    """`vscreen dock` (vscreen_main.cpp:67-93) over the GPU path: per library
    record, make_ligand + embed_3d(Rng(seed).split(i).next_u64()) +
    torsion_topology, dock(..., Rng(seed).split(i).split(1).next_u64()) with
    the reference contract (sweep-v1 restarts refined by the ascent,
    capi.h vs_dock_refined_host), filter_poses, the FP64 rescore on request,
    and one pose_to_json line per kept pose.  A record that fails to parse
    stops the run after the lines of the records before it, with the
    reference's exception.  Returns the number of lines written."""
    from . import _capi
    from .chem import make_ligand, read_library_file
    from .dock import Pose, filter_poses, pose_to_json
    from .errors import check as _check
    threads = threads or os.cpu_count() or 1
    pocket = load_pocket_file(pocket_path)
    records = read_library_file(library_path)
    try:
        out = open(out_path, "wb")
    except OSError as e:
        raise ConfigError(f"cannot open output: {out_path}") from e
    n = len(records)
    es = np.zeros(max(n, 1), np.uint64)
    ds = np.zeros(max(n, 1), np.uint64)
    for i in range(n):
        path1 = np.array([i], np.uint64)
        path2 = np.array([i, 1], np.uint64)
        _check(_lib.vs_rng_u64(seed & (2**64 - 1), ptr(path1, C.c_uint64), 1, 1,
                               ptr(es[i:], C.c_uint64)))
        _check(_lib.vs_rng_u64(seed & (2**64 - 1), ptr(path2, C.c_uint64), 2, 1,
                               ptr(ds[i:], C.c_uint64)))
    lib = build_library([r.smiles for r in records], [r.id for r in records], es[:n], ds[:n],
                        threads=threads, drop_failed=False)
    bad = np.nonzero(lib.status[:n] != 0)[0]
    stop = int(bad[0]) if len(bad) else n
    lines = 0
    own = engine is None
    eng = engine or Engine(0)
    try:
        eng.set_pocket(pocket)
        if stop:
            head = lib.subset(np.arange(stop))
            prm = DockParams(restarts=restarts, diversity_delta=diversity)
            per_lig = eng.dock_refined(head, prm, max_steps)
            _, to, _ = head.offsets()
            for i, poses in enumerate(per_lig):
                ps = [Pose(head.ids[i], tuple(float(v) for v in t), tuple(float(v) for v in q),
                           [float(v) for v in th], sc, None, restart=r)
                      for (t, q, th, sc, r) in poses]
                ps = filter_poses(ps, keep_top, min_score)
                if do_rescore and ps:
                    _, resc = eng.score64(head, np.full(len(ps), i, np.int32),
                                          [p.translation for p in ps], [p.rotation for p in ps],
                                          [v for p in ps for v in p.torsions])
                    for p, v in zip(ps, resc):
                        p.rescore = float(v)
                for p in ps:
                    out.write((pose_to_json(p) + "\n").encode())
                    lines += 1
    finally:
        out.close()
        if own:
            eng.close()
    if stop < n:
        # the reference's make_ligand exception for that record
        make_ligand(records[stop].id, records[stop].smiles)
        raise VscreenError(f"ligand {records[stop].id}: status {int(lib.status[stop])}")
    return lines


def report_to_json(stages, ranked, pairs=(), trace_path: str = "") -> str:
    """CampaignReport::to_json (pipeline.cpp:269-301): the reference's report
    bytes (nlohmann ordered_json, indent 2).  stages: StageStats; ranked:
    RankedLigand; pairs: (pair_id, ligand_a, ligand_b, ddg_kT, sem_kT,
    replicas, target_met) tuples (the FEP stage itself is out of scope)."""
    from .dock import _jnum, _jstr

    def obj(fields, ind):
        pad = " " * ind
        return ("{\n" + ",\n".join(f'{pad}  "{k}": {v}' for k, v in fields) + "\n" + pad + "}")

    def arr(items, ind):
        pad = " " * ind
        return "[]" if not items else "[\n" + ",\n".join(pad + "  " + x for x in items) + "\n" + pad + "]"

    st = [obj([("name", _jstr(s.name)), ("in", str(int(s.in_))), ("out", str(int(s.out))),
               ("sim_seconds", _jnum(s.sim_seconds or 0.0)), ("tasks", str(int(s.tasks)))], 4)
          for s in stages]
    rk = [obj([("id", _jstr(r.id)), ("score", _jnum(r.score)),
               ("delta_g", "null" if r.delta_g is None else _jnum(r.delta_g))], 4) for r in ranked]
    pr = [obj([("pair_id", _jstr(p[0])), ("ligand_a", _jstr(p[1])), ("ligand_b", _jstr(p[2])),
               ("ddg_kT", _jnum(p[3])), ("sem_kT", _jnum(p[4])), ("replicas", str(int(p[5]))),
               ("target_met", "true" if p[6] else "false")], 4) for p in pairs]
    return obj([("stages", arr(st, 2)), ("ranked", arr(rk, 2)), ("pairs", arr(pr, 2)),
                ("trace_path", _jstr(trace_path))], 0)


def funnel_to_json(f: DockFunnel, trace_path: str = "") -> str:
    """The dock funnel's stage records and ranked ligands as the reference's
    report bytes (report_to_json; no pairs: the FEP stages are out of scope)."""
    return report_to_json(f.stages, f.ranked, (), trace_path)


__all__ = ["CampaignConfig", "ConfigError", "DockFunnel", "DockTask", "StageKnobs", "StageStats",
           "dock_library_jsonl", "funnel_to_json", "load_config_file", "report_to_json", "parse_config_json", "prepare", "run_dock_stages"]
