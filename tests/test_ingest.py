"""Host ligand ingest (parse, descriptors, embed, torsion topology, corpus,
library text) — bit-exact against the reference library, plus the
reference's own known answers (test_chem / test_dock / test_smoke)."""
import math

import numpy as np
import pytest

from conftest import need_ref


@pytest.fixture(scope="module")
def V():
    import paper_2304_09953_b200 as V
    return V


def test_smoke_known_answers(V):
    # tests/python/test_smoke.py:12-28
    g = V.parse_smiles("CCO")
    assert g["atoms"] == [("C", False), ("C", False), ("O", False)]
    assert g["bonds"] == [(0, 1, 1), (1, 2, 1)]
    assert V.rotatable_bonds("CCCC") == 1
    assert V.rotatable_bonds("C1CCCCC1") == 0
    with pytest.raises(V.ParseError):
        V.parse_smiles("C(")
    a = V.embed_3d("CCO", seed=5)
    assert a == V.embed_3d("CCO", seed=5)
    assert len(a) == 3
    assert 1.3 < math.dist(a[0], a[1]) < 1.7


def test_torsion_topology_known_answer(V):
    # test_dock.cpp:378-385
    t = V.torsion_topology("CCCC")
    assert len(t.axes) == 1 and (t.axes[0].a, t.axes[0].b) == (1, 2) and t.axes[0].moving == [3]


@pytest.mark.parametrize("bad,kind", [("C(", "UnbalancedBranch"), ("C)", "UnbalancedBranch"),
                                      ("C1CC", "UnclosedRingBond"), ("CX", "UnknownToken"),
                                      ("=C", "UnknownToken"), ("", "UnknownToken")])
def test_parse_errors(V, bad, kind):
    with pytest.raises(V.ParseError) as e:
        V.parse_smiles(bad)
    assert e.value.kind == kind


def test_corpus_and_embed_bit_exact_vs_reference(V):
    R = need_ref()
    for i in range(400):
        smi = V.random_smiles(99, i)
        assert smi == R.random_smiles(99, i)
        lig = V.make_ligand("x", smi, embed_seed=7 * i + 1)
        r = R.RefLigand(smi, 7 * i + 1)
        assert np.array_equal(lig.conformer.coords, r.coords()), smi
        assert [(a.a, a.b, a.moving) for a in lig.topology.axes] == r.axes()
        assert lig.rotatable_bonds == r.rot_bonds
        assert np.array_equal(lig.atom_classes(), r.classes())
        rb = r.bonds()
        assert [tuple(b) for b in lig.graph.bonds] == [tuple(int(v) for v in row[:3]) for row in rb]
        assert lig.graph.ring_bond_flags == [bool(v) for v in rb[:, 3]]


def test_library_builder_matches_single_builds(V):
    smis = [V.random_smiles(5, i) for i in range(64)]
    lib = V.build_library(smis, embed_seeds=list(range(64)), threads=4)
    ao, to, mo = lib.offsets()
    for i, s in enumerate(smis):
        lg = V.make_ligand("x", s, embed_seed=i)
        assert np.array_equal(lib.coords[ao[i]:ao[i + 1]], lg.conformer.coords)
        assert int(lib.n_tors[i]) == len(lg.topology.axes)


def test_read_library_records(V, tmp_path):
    p = tmp_path / "lib.smi"
    p.write_bytes(b"# header\nCCO\tethanol\n\nc1ccccc1\nCCN\t\r\n")
    recs = V.chem.read_library_file(str(p))
    assert [(r.smiles, r.id, r.line_number) for r in recs] == [
        ("CCO", "ethanol", 2), ("c1ccccc1", "L4", 4), ("CCN", "L5", 5)]


def test_aromatic_atoms_count_as_carbon(V):
    lig = V.make_ligand("b", "c1ccccc1O")
    assert list(lig.atom_classes()) == [1] * 6 + [2]


def test_flexible_selection_deterministic_and_in_bounds(V):
    """C4 population (capi.h vs_flexible_select): chunked parallel scan, so the
    selection must not depend on scheduling; every pick is a concatenation of
    consecutive corpus entries inside the atom / torsion-axis bounds."""
    from paper_2304_09953_b200.chem import flexible_smiles, random_smiles
    a = flexible_smiles(7, 12)
    b = flexible_smiles(7, 12)
    assert a == b and len(a) == 12
    assert flexible_smiles(7, 5) == a[:5]
    for s in a[:6]:
        lg = V.make_ligand("f", s, embed_seed=1)
        assert 60 <= lg.heavy_atoms <= 80
        assert 15 <= len(lg.topology.axes) <= 20
    # each pick is random_smiles(7, i) + random_smiles(7, i + 1) + ...
    assert a[0].startswith(random_smiles(7, 0)) or any(
        a[0].startswith(random_smiles(7, i)) for i in range(1, 5000))


def test_bench_configs_declared():
    """bench.py --config names the BASELINE.json configs it measures."""
    import bench
    assert set(bench.CONFIGS) == {"c2", "c3", "c4", "c5"}
    assert bench.CONFIGS["c3"]["scaling"] == "strong"
    assert bench.CONFIGS["c5"]["grid_spacing"] == 0.2


def _fuzz_smiles(rng, n):
    """Malformed and well-formed strings over the grammar's alphabet plus
    noise: random token soups, corpus entries with one edit, truncations."""
    toks = ["C", "N", "O", "S", "P", "F", "I", "B", "Cl", "Br", "c", "n", "o", "s", "p", "b",
            "-", "=", "#", "(", ")", "1", "2", "3", "9", "%12", "%10", "%1", "%0a", "%", "X", "[",
            "l", "r", "0", " "]
    out = []
    import paper_2304_09953_b200 as V
    for k in range(n):
        mode = k % 3
        if mode == 0:
            out.append("".join(rng.choice(toks) for _ in range(rng.integers(0, 9))))
        else:
            s = V.random_smiles(99, int(rng.integers(0, 10_000)))
            if mode == 1 and s:
                i = int(rng.integers(0, len(s)))
                s = s[:i] + rng.choice(toks) + s[i + 1:]
            else:
                s = s[:int(rng.integers(0, len(s) + 1))]
            out.append(s)
    return out


def test_parse_errors_match_reference_kind_and_position(V):
    """The parser (vs_ingest.cpp, streaming lexer + graph builder) reports
    the reference's outcome on 6000 fuzzed strings: parsed (same atom and
    bond counts) or ParseError with the same kind and 1-based position."""
    R = need_ref()
    rng = np.random.default_rng(2026)
    n_err = 0
    for s in _fuzz_smiles(rng, 6000):
        ref = R.parse_check(s)
        try:
            g = V.parse_smiles(s)
            ours = ("ok", len(g["atoms"]), len(g["bonds"]))
        except V.ParseError as e:
            ours = ("error", V.ParseError.KINDS.index(e.kind), e.position)
            n_err += 1
        assert ours == ref, (s, ours, ref)
    assert 1500 < n_err < 5500
