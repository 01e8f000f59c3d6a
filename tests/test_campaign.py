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


def _stage_lines(path, upto="rank"):
    out = []
    for line in open(path, "rb").read().decode().splitlines():
        j = json.loads(line)
        if j["kind"] in ("stage_start", "stage_end"):
            out.append(line)
            if j["kind"] == "stage_end" and j["stage"] == upto:
                break
    return out


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_campaign_trace_and_report_on_gpu(Cm, tmp_path):
    """run_campaign's trace stage lines (TraceWriter, pipeline.cpp:335-352)
    and report stage records for parse / embed / dock against the reference's
    own run on campaign_100.json (tests/golden/campaign/ref_*, made by
    make_campaign_golden.py).  The scheduler events and sim_seconds belong to
    the simulated cluster (out of scope)."""
    for f in ("campaign_100.json", "pocket.json", "sample_library_100.smi", "smiles.dict"):
        shutil.copy(os.path.join(CAMP, f), tmp_path / f)
    cfg = Cm.load_config_file(str(tmp_path / "campaign_100.json"))
    cfg.trace_path = str(tmp_path / "out" / "trace.jsonl")
    cfg.report_path = str(tmp_path / "out" / "report.json")
    f = Cm.run_dock_stages(cfg, write_outputs=True)
    assert _stage_lines(cfg.trace_path) == _stage_lines(os.path.join(CAMP, "ref_trace.jsonl"))
    assert open(cfg.trace_path).read().count("\n") == 12
    rep = open(cfg.report_path, "rb").read().decode()
    assert rep == Cm.funnel_to_json(f, cfg.trace_path)
    ours = json.loads(rep)["stages"]
    ref = json.load(open(os.path.join(CAMP, "ref_report.json")))["stages"]
    for a, b in zip(ours[:3], ref[:3]):
        assert (a["name"], a["in"], a["out"], a["tasks"]) == (b["name"], b["in"], b["out"], b["tasks"])
    assert [s["name"] for s in ours] == [s["name"] for s in ref[:6]]
    assert ours[3]["in"] == ref[3]["in"] and ours[4]["in"] == ref[4]["in"]
    # the pybind-style entry point (module.cpp:320-325) over the same config
    import paper_2304_09953_b200 as V
    j = json.load(open(tmp_path / "campaign_100.json"))
    j["trace"] = str(tmp_path / "out2" / "trace.jsonl")
    j["report"] = str(tmp_path / "out2" / "report.json")
    (tmp_path / "c2.json").write_text(json.dumps(j))
    rep2 = V.run_campaign(str(tmp_path / "c2.json"))
    assert rep2 == json.loads(rep) | {"trace_path": j["trace"]}
    assert _stage_lines(j["trace"]) == _stage_lines(cfg.trace_path)


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_dock_jsonl_on_gpu(Cm, tmp_path):
    """`vscreen dock` pose JSONL (vscreen_main.cpp:67-93) through the GPU
    path: the reference's seeds and conformers (the reference re-scores every
    written pose to the written scores within 1e-9), pose_to_json bytes, the
    filter's order and limits, the records' order; a bad record stops the
    run after the earlier records' lines with the reference's exception."""
    R = need_ref()
    from paper_2304_09953_b200.chem import read_library_file
    from paper_2304_09953_b200.errors import ParseError
    lib_path = os.path.join(CAMP, "sample_library_100.smi")
    pocket_path = os.path.join(CAMP, "pocket.json")
    out = tmp_path / "poses.jsonl"
    n = Cm.dock_library_jsonl(lib_path, pocket_path, str(out), restarts=4, diversity=1.0,
                              keep_top=3, min_score=-5.0, do_rescore=True, seed=11)
    lines = open(out, "rb").read().decode().splitlines()
    assert n == len(lines) > 0
    recs = read_library_file(lib_path)
    order = {r.id: k for k, r in enumerate(recs)}
    rp = R.RefPocket(open(pocket_path).read())
    by_lig = {}
    for line in lines:
        j = json.loads(line)
        by_lig.setdefault(j["ligand"], []).append(j)
        assert line == R.pose_json_bytes(j["ligand"], j["translation"], j["rotation"],
                                         j["torsions"], j["geometric_score"], j["rescore"])
    assert list(by_lig) == sorted(by_lig, key=order.get)  # record order
    for lid, poses in list(by_lig.items())[::7]:
        assert len(poses) <= 3
        sc = [p["geometric_score"] for p in poses]
        assert sc == sorted(sc, reverse=True) and min(sc) >= -5.0
        i = order[lid]
        es = int(R.rng_u64(11, [i], 1)[0])
        ref = R.RefLigand(recs[i].smiles, embed_seed=es, iterations=200, ligand_id=lid)
        for p in poses:
            g = ref.geometric_score(rp, p["translation"], p["rotation"], p["torsions"])
            r = ref.rescore(rp, p["translation"], p["rotation"], p["torsions"])
            assert abs(g - p["geometric_score"]) <= 1e-9 * max(abs(g), 1.0)
            assert abs(r - p["rescore"]) <= 1e-9 * max(abs(r), 1.0)
    # a bad record: the lines before it, then ParseError
    lines_in = open(lib_path).read().splitlines()
    bad = tmp_path / "bad.smi"
    bad.write_text("\n".join(lines_in[:5] + ["C1CC(\tBADX"] + lines_in[5:]) + "\n")
    with pytest.raises(ParseError):
        Cm.dock_library_jsonl(str(bad), pocket_path, str(tmp_path / "b.jsonl"), restarts=2,
                              keep_top=2, seed=11)
    ids = [json.loads(x)["ligand"] for x in open(tmp_path / "b.jsonl").read().splitlines()]
    assert ids and set(ids) <= {r.id for r in recs[:5]}


def test_trace_writer_and_config_paths(Cm, tmp_path):
    """TraceWriter (pipeline.cpp:335-352): parent directories created, the
    stage lines' bytes, ConfigError when the trace cannot be opened; the
    config's output paths (trace / report) stay as given (pipeline.cpp:151-154)."""
    tw = Cm._TraceWriter(str(tmp_path / "a" / "b" / "t.jsonl"))
    tw.stage("start", "parse")
    tw.stage("end", "parse")
    tw.close()
    assert open(tmp_path / "a" / "b" / "t.jsonl", "rb").read() == (
        b'{"kind":"stage_start","stage":"parse"}\n{"kind":"stage_end","stage":"parse"}\n')
    (tmp_path / "f").write_text("x")
    with pytest.raises(Cm.ConfigError, match="cannot open trace for writing"):
        Cm._TraceWriter(str(tmp_path / "f" / "t.jsonl"))
    for f in ("pocket.json", "sample_library_100.smi", "smiles.dict"):
        shutil.copy(os.path.join(CAMP, f), tmp_path / f)
    j = json.load(open(os.path.join(CAMP, "campaign_100.json")))
    cfg = Cm.parse_config_json(json.dumps(dict(j, trace="out/t.jsonl", report="out/r.json")),
                               str(tmp_path))
    assert cfg.trace_path == "out/t.jsonl" and cfg.report_path == "out/r.json"
    j2 = {k: v for k, v in j.items() if k not in ("trace", "report")}
    d = Cm.parse_config_json(json.dumps(j2), str(tmp_path))  # pipeline.hpp:62-63 defaults
    assert d.trace_path == "campaign_trace.jsonl" and d.report_path == "campaign_report.json"
    bad = dict(j, funnel={"keep_after_dock": 0.0, "keep_for_fep": 0.5})
    with pytest.raises(Cm.ConfigError, match="keep_after_dock"):
        Cm.parse_config_json(json.dumps(bad), str(tmp_path))
