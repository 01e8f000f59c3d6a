"""Shared fixtures.  `-m gpu` tests need a B200 and the in-tree native
library; everything else runs on CPU.  The reference library
(oracle/_ref/libvsref.so) is optional: tests that need it skip without it and
the committed golden fixtures under tests/golden/ pin the oracle instead."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def pocket_json():
    with open(os.path.join(GOLDEN, "pocket.json")) as f:
        return f.read()


@pytest.fixture(scope="session")
def ref_available():
    from oracle import ref
    return ref.available()


def need_ref():
    from oracle import ref
    if not ref.available():
        pytest.skip("reference library oracle/_ref/libvsref.so not built")
    return ref


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def corpus_library(n, seed=99, max_atoms=40, max_tors=8, min_atoms=1, embed_master=2024,
                   dock_master=2024, threads=8):
    """C1-style synthetic library: reference corpus sampler rejection-filtered
    to the size bounds, embed seeds Rng(master).split(1).split(i), dock seeds
    .split(2).split(i) (pipeline.cpp:422-484)."""
    import paper_2304_09953_b200 as V
    from paper_2304_09953_b200.pipeline import campaign_seeds
    smis, i = [], 0
    while len(smis) < n:
        s = V.random_smiles(seed, i)
        i += 1
        lig = V.make_ligand("x", s)
        if min_atoms <= lig.heavy_atoms <= max_atoms and len(lig.topology.axes) <= max_tors:
            smis.append(s)
    es = campaign_seeds(embed_master, n, stage=1)
    ds = campaign_seeds(dock_master, n, stage=2)
    ids = [f"MOL{k}" for k in range(n)]
    return V.build_library(smis, ids, es, ds, threads=threads), smis
