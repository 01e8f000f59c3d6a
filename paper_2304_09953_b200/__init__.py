"""B200-native dock-and-score path of the LIGATE virtual-screening stack
(arXiv 2304.09953), drop-in for the reference `vscreen` API on that path.

Python surface of proj/bindings/module.cpp restricted to the hot path:
`dock_smiles`, `rmsd`, `target_batch_size`, `simulate_throughput`,
`rank_ligands`, `run_campaign` (its dock funnel), the codec read side
(`load_dictionary`, `decompress_line`), plus the chem loaders that feed it.  Library-scale
screening is `pipeline.screen` / `dock.Engine`.
"""
from __future__ import annotations

import json as _json

from . import _capi  # noqa: F401  (fails loudly if the native library is missing)
from .batcher import (BatchQueue, DeviceModel, SizeClass, bucket_replay, default_classes,
                      simulate_throughput, size_class, target_batch_size)
from .chem import (Conformer, Library, Ligand, build_library, embed_3d, make_ligand,
                   parse_smiles, random_smiles, read_library_file, rotatable_bonds,
                   torsion_topology)
from .dock import (DockParams, Engine, Pocket, Pose, ScoreGradient, Site, apply_pose, dock,
                   filter_poses, geometric_score, load_pocket_file, parse_pocket_json,
                   pocket_to_json, pose_rmsd, pose_to_json, rescore, rmsd, score_gradient)
from .codec import decompress_line, load_dictionary
from .errors import (AtomCountMismatch, EmptyBounds, ItemTooLarge, LengthMismatch, OutOfRange,
                     ParseError)
from .pipeline import RankedLigand, rank_ligands, screen

__version__ = "0.1.0"


def run_campaign(config_path: str) -> dict:
    """module.cpp:320-325 restricted to the hot path: the dock funnel of
    pipeline::run_campaign (parse -> embed -> dock -> rescore -> filter ->
    rank) on the GPU for the campaign config at `config_path`, writing the
    trace stage lines and the report like the reference; returns the report
    as a dict.  The pair / FEP stages are out of scope, so
    `pairs` is empty and the report ends at the rank stage."""
    from .campaign import load_config_file, run_dock_stages, funnel_to_json
    cfg = load_config_file(config_path)
    f = run_dock_stages(cfg, write_outputs=True)
    return _json.loads(funnel_to_json(f, cfg.trace_path))


def dock_smiles(smiles: str, pocket_json: str, restarts: int = 4, diversity_delta: float = 1.0,
                seed: int = 0) -> list[dict]:
    """module.cpp:128-145: parse -> embed_3d(seed) -> torsion_topology ->
    dock(seed) -> pose dicts sorted by geometric score.  The same seed feeds
    the embedding and the dock, as in the reference."""
    lig = make_ligand("", smiles, embed_seed=seed)
    pocket = parse_pocket_json(pocket_json)
    poses = dock(lig.conformer, lig.topology, pocket, restarts, diversity_delta, seed,
                 atom_class=lig.atom_classes())
    return [_json.loads(pose_to_json(p)) for p in poses]
