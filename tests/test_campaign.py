"""The dock funnel of run_campaign (paper_2304_09953_b200.campaign, SURVEY §8
f3) against the reference's own pieces: config parsing
(pipeline.cpp:76-160), parse / embed stages and seeds (:381-429), the size
class filter and BatchQueue replay that make the dock.b{bi} tasks
(:433-473), filter / best / rank / keep (:502-537).  Fixtures:
tests/golden/campaign/ holds the reference's proj/data/campaign_100.json,
sample_library_100.smi and pocket.json (data files, copied verbatim)."""
import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, gpu_available, need_ref

CAMP = os.path.join(GOLDEN, "campaign")


@pytest.fixture(scope="module")
def Cm():
    from paper_2304_09953_b200 import campaign
    return campaign


def test_config_matches_reference_json(Cm):
    cfg = Cm.load_config_file(os.path.join(CAMP, "campaign_100.json"))
    j = json.load(open(os.path.join(CAMP, "campaign_100.json")))
    assert cfg.library_path == os.path.join(CAMP, "sample_library_100.smi")
    assert cfg.pocket_path == os.path.join(CAMP, "pocket.json")
    assert cfg.keep_after_dock == 0.2 and cfg.master_seed == 2024 and cfg.threads == 4
    assert cfg.knobs.restarts == 4 and cfg.knobs.keep_top == 4 and cfg.knobs.min_score == -5.0
    assert cfg.knobs.ls_max_steps == 300 and cfg.knobs.embed_iterations == 200
    assert [c.astuple() for c in cfg.classes] == [
        (c["atom_lo"], c["atom_hi"], c["rot_lo"], c["rot_hi"]) for c in j["classes"]]
    assert cfg.device.service_time_per_class == j["device"]["service_time_per_class_s"]
    bad = dict(j)
    del bad["pocket"]
    with pytest.raises(Cm.ConfigError):
        Cm.parse_config_json(json.dumps(bad), CAMP)
    with pytest.raises(Cm.ConfigError):
        Cm.parse_config_json("{not json", CAMP)
    smzc = dict(j, library="lib.smzc")
    with pytest.raises(Cm.ConfigError):
        Cm.prepare(Cm.parse_config_json(json.dumps(smzc), CAMP))


def _library_with_edge_cases(tmp_path):
    """The sample library plus unparsable lines and a ligand outside every
    size class (>= 96 heavy atoms)."""
    from paper_2304_09953_b200.chem import random_smiles
    lines = open(os.path.join(CAMP, "sample_library_100.smi")).read().splitlines()
    big = "".join(random_smiles(99, i) for i in range(40))
    lines[5:5] = ["C1CC(\tBAD1", "Xq\tBAD2", big + "\tBIG0"]
    (tmp_path / "lib.smi").write_text("\n".join(lines) + "\n")
    for f in ("pocket.json", "smiles.dict"):
        shutil.copy(os.path.join(CAMP, f), tmp_path / f)
    j = json.load(open(os.path.join(CAMP, "campaign_100.json")))
    j["library"] = "lib.smi"
    (tmp_path / "c.json").write_text(json.dumps(j))
    return str(tmp_path / "c.json")


def test_prepare_matches_reference_stages(Cm, tmp_path):
    R = need_ref()
    cfg = Cm.load_config_file(_library_with_edge_cases(tmp_path))
    lib, stages, tasks, n_in = Cm.prepare(cfg, threads=8)
    from paper_2304_09953_b200.chem import read_library_file
    recs = read_library_file(cfg.library_path)
    parsed = []
    for r in recs:
        try:
            parsed.append((r, R.RefLigand(r.smiles, iterations=-1)))
        except R.RefError:
            pass
    assert [s.to_json()["out"] for s in stages] == [len(parsed), len(parsed)]
    assert stages[0].in_ == len(recs) and n_in == len(parsed)
    classes = [c.astuple() for c in cfg.classes]
    d = cfg.device
    in_range, batches = R.bucket_replay([p[1].n_atoms for p in parsed],
                                        [p[1].rot_bonds for p in parsed], classes,
                                        d.memory_capacity, d.mem_fixed, d.mem_per_atom,
                                        d.mem_per_rotbond)
    assert not in_range.all()  # BIG0 is outside every class
    assert [t.id for t in tasks] == [f"dock.b{i}" for i in range(len(batches))]
    for t, (cls, members) in zip(tasks, batches):
        assert t.cls == cls
        assert t.ligand_ids == [parsed[m][0].id for m in members]
        assert t.duration_s == d.launch_overhead + len(members) * d.service_time(cls)
    usable = [i for i in range(len(parsed)) if in_range[i]]
    assert list(lib.ids) == [parsed[i][0].id for i in usable]
    # embed seeds over the parsed index, dock seeds over the in-class index
    ao, _, _ = lib.offsets()
    for k in range(0, len(usable), 7):
        i = usable[k]
        es = int(R.rng_u64(cfg.master_seed, [1, i], 1)[0])
        ref = R.RefLigand(parsed[i][0].smiles, embed_seed=es, iterations=200)
        np.testing.assert_array_equal(lib.coords[ao[k]:ao[k + 1]], ref.coords())
        assert int(lib.seeds[k]) == int(R.rng_u64(cfg.master_seed, [2, k], 1)[0])


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_dock_funnel_on_gpu(Cm, tmp_path):
    from oracle import sweep
    import paper_2304_09953_b200 as V
    cfg = Cm.load_config_file(_library_with_edge_cases(tmp_path))
    f = Cm.run_dock_stages(cfg)
    names = [s.name for s in f.stages]
    assert names == ["parse", "embed", "dock", "rescore", "filter", "rank"]
    st = {s.name: s for s in f.stages}
    assert st["dock"].tasks == len(f.tasks) and st["dock"].out == len(f.ids)
    assert st["dock"].sim_seconds is None  # scheduler simulation: out of scope
    # the GPU pass is the oracle's, bit for bit
    lib, _, _, _ = Cm.prepare(cfg, threads=8)
    pocket = V.load_pocket_file(cfg.pocket_path)
    k = cfg.knobs
    prm = V.DockParams(restarts=k.restarts, diversity_delta=k.diversity_delta,
                       keep_top=k.keep_top, min_score=k.min_score)
    ora = sweep.dock_library(sweep.OraclePocket(pocket), lib, prm, threads=8)
    kept = ora["n_surv"][:len(lib)] > 0
    np.testing.assert_array_equal(f.best[kept].view(np.uint32),
                                  ora["best"][:len(lib)][kept].view(np.uint32))
    assert st["filter"].out == int(kept.sum())
    # rank_ligands order of the kept best scores, keep fraction
    scores = {lib.ids[i]: float(ora["best"][i]) for i in np.nonzero(kept)[0]}
    ranked = V.rank_ligands(scores)
    n_keep = min(len(ranked), max(1, int(np.floor(cfg.keep_after_dock * len(scores)))))
    assert [(r.id, r.score) for r in f.ranked] == ranked[:n_keep]
    assert st["rank"].out == n_keep
    json.loads(Cm.funnel_to_json(f))
