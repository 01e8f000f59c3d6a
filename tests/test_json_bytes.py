"""JSON I/O byte parity (dock.cpp:432-489): pocket_to_json
(parse_pocket_json(text)) and pose_to_json of the Python layer and of the
C++ drop-in (libvscreen_core.so) produce the reference's exact bytes
(nlohmann ordered_json) on random pockets and poses: tiny / huge / negative
/ integral values, non-finite scores, escaped ids."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, need_ref


def _values(rng, n):
    pool = [0.0, -0.0, 1.0, 2.0, 1e-5, 1e-4, 0.1, 1e15, 1e16, 1e-300, 1e300, -3.5e20, 123456.789,
            1 / 3, 2 ** 53, 7.0]
    out = []
    for k in range(n):
        out.append(float(pool[k % len(pool)]) if k % 2 else float(rng.normal() * 10.0 ** int(rng.integers(-8, 9))))
    return out


def _pocket(rng, n_sites):
    v = iter(_values(rng, 6 * n_sites + 8))
    kinds = ["steric", "hbond", "lipophilic"]
    sites = [{"center": [next(v), next(v), next(v)], "weight": next(v), "sigma": abs(next(v)) + 0.5,
              "kind": kinds[i % 3]} for i in range(n_sites)]
    return {"sites": sites, "bounds": {"min": [-5, -6.5, next(v)], "max": [5, 6, 7]},
            "clash_radius": 0.7, "clash_penalty": abs(next(v))}


@pytest.fixture(scope="module")
def json_exe(tmp_path_factory):
    exe = tmp_path_factory.mktemp("json") / "json_bytes"
    libdir = os.path.join(ROOT, "paper_2304_09953_b200")
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "cpp", "json_bytes.cpp"), f"-L{libdir}",
                    "-lvscreen_core", "-lvscreen_gpu", f"-Wl,-rpath,{libdir}", "-o", str(exe)],
                   check=True)
    return str(exe)


def test_json_bytes_match_reference(json_exe):
    R = need_ref()
    import paper_2304_09953_b200 as V
    rng = np.random.default_rng(11)
    for case in range(40):
        text = json.dumps(_pocket(rng, case % 5))
        ref = R.pocket_json_bytes(text)
        assert V.pocket_to_json(V.parse_pocket_json(text)) == ref
        t = _values(rng, 3)
        q = _values(rng, 4)
        tors = _values(rng, case % 4)
        geo = [1.5, float("nan"), -0.0, 1e-5][case % 4]
        resc = None if case % 3 == 0 else _values(rng, 1)[0]
        lig = ["L1", "MOL\"9\\x", "é-ligand", "tab\there"][case % 4]
        ref_pose = R.pose_json_bytes(lig, t, q, tors, geo, resc)
        pose = V.Pose(lig, tuple(t), tuple(q), list(tors), geo, resc)
        assert V.pose_to_json(pose) == ref_pose
        if "\t" not in lig:  # argv carries the id as is
            args = [json_exe, lig] + [repr(x) for x in t + q] + [repr(geo),
                                                              "none" if resc is None else repr(resc)]
            args += [repr(x) for x in tors]
            out = subprocess.run(args, input=text, capture_output=True, text=True, check=True).stdout
            cpp_pocket, cpp_pose = out.split("\n--\n")
            assert cpp_pocket == ref
            assert cpp_pose == ref_pose


REPORT_SPEC = {"stages": [["parse", 100, 98, 0.0, 0], ["dock", 98, 91, 12.345678901234567, 7],
                          ["rank", 91, 9, 0.0, 0]],
               "ranked": [["L10", 45.25, None], ["L2", -1e-5, 0.1], ["é\"x", 1e20, -3.5]],
               "pairs": [["P0", "L10", "L2", -1.234567890123, 0.05, 4, True]],
               "trace_path": "out/campaign_trace.jsonl"}


def test_campaign_report_bytes_match_reference(tmp_path):
    """CampaignReport::to_json / results_tsv (pipeline.cpp:269-313): the
    Python report writer and the C++ drop-in give the reference's bytes."""
    R = need_ref()
    from paper_2304_09953_b200.campaign import StageStats, report_to_json
    from paper_2304_09953_b200.pipeline import RankedLigand
    ref = R.report_bytes(REPORT_SPEC, 0)
    ref_tsv = R.report_bytes(REPORT_SPEC, 1)
    st = [StageStats(s[0], s[1], s[2], s[3], s[4]) for s in REPORT_SPEC["stages"]]
    rk = [RankedLigand(*x) for x in REPORT_SPEC["ranked"]]
    assert report_to_json(st, rk, [tuple(p) for p in REPORT_SPEC["pairs"]],
                          REPORT_SPEC["trace_path"]) == ref
    assert report_to_json([], [], (), "") == R.report_bytes(
        {"stages": [], "ranked": [], "pairs": [], "trace_path": ""}, 0)
    exe = tmp_path / "report_bytes"
    libdir = os.path.join(ROOT, "paper_2304_09953_b200")
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "cpp", "report_bytes.cpp"), f"-L{libdir}",
                    "-lvscreen_core", "-lvscreen_gpu", f"-Wl,-rpath,{libdir}", "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    cpp_json, cpp_tsv = out.split("\n--\n")
    assert cpp_json == ref
    assert cpp_tsv == ref_tsv


def test_number_text_matches_reference_on_random_doubles():
    """nlohmann's Grisu2 digits are not always the shortest round-trip ones
    (about 1 value in 600 differs from Python's repr): every number the
    Python writers print comes from capi.h vs_json_format_doubles."""
    R = need_ref()
    from paper_2304_09953_b200.dock import _jnums
    rng = np.random.default_rng(7)
    v = rng.normal(size=60000) * 10.0 ** rng.integers(-12, 13, size=60000)
    v[::97] = np.round(v[::97])
    bits = rng.integers(0, 2**63, size=3000, dtype=np.uint64).view(np.float64)
    v = np.concatenate([v, bits[np.isfinite(bits)]])
    mine = _jnums(v)
    for k in range(0, len(v), 3):
        chunk = v[k:k + 3]
        if len(chunk) < 3:
            break
        s = R.pose_json_bytes("a", chunk, [1, 0, 0, 0], [], 0.5, None)
        assert s.split('"translation":[')[1].split("]")[0].split(",") == mine[k:k + 3], chunk
