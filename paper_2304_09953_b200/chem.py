"""Ligand loaders: SMILES parsing, descriptors, 3D
embedding, torsion topology and the library file format, all served by the
native host code in libvscreen_gpu.so (vs_ingest.cpp).

Mirrors proj/include/vscreen/chem.hpp and the chem part of
proj/bindings/module.cpp:79-95.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _capi
from ._capi import lib as _lib, ptr
from .errors import ParseError, check

BOND_ORDER = {1: "single", 2: "double", 3: "triple", 4: "aromatic"}



EMBED_PLACE_ONLY = -2  # capi.h VS_EMBED_PLACE_ONLY: BFS placement only
EMBED_DEVICE = -3      # capi.h VS_EMBED_DEVICE: parse + topology; embed_3d on the device

@dataclass
class Axis:
    """TorsionTopology::Axis (dock.hpp:66-69)."""
    a: int
    b: int
    moving: list[int]


@dataclass
class TorsionTopology:
    axes: list[Axis] = field(default_factory=list)


@dataclass
class MolecularGraph:
    """chem::MolecularGraph (chem.hpp:15-23)."""
    elements: list[str]
    aromatic: list[bool]
    bonds: list[tuple[int, int, int]]
    ring_bond_flags: list[bool]

    def atom_count(self) -> int:
        return len(self.elements)


@dataclass
class Conformer:
    """chem::Conformer (chem.hpp:78-81); coords (N, 3) float64."""
    ligand_id: str
    coords: np.ndarray


@dataclass
class Ligand:
    """chem::Ligand (chem.hpp:55-61) plus its conformer and topology."""
    id: str
    smiles: str
    graph: MolecularGraph
    heavy_atoms: int
    rotatable_bonds: int
    conformer: Conformer | None = None
    topology: TorsionTopology | None = None

    def atom_classes(self) -> np.ndarray:
        return np.array([1 if e == "C" else 2 if e in ("N", "O") else 0
                         for e in self.graph.elements], dtype=np.int32)


def _build(smiles: str, seed: int, iterations: int):
    cap_a = max(8, 2 * len(smiles) + 8)
    cap_b = cap_a * 2
    cap_t = cap_b
    cap_m = cap_a * cap_t
    bufs = dict(
        coords=np.zeros(3 * cap_a, np.float64), atom_class=np.zeros(cap_a, np.int32),
        elements=C.create_string_buffer(3 * cap_a), aromatic=np.zeros(cap_a, np.uint8),
        bonds=np.zeros(3 * cap_b, np.int32), ring=np.zeros(cap_b, np.uint8),
        axis_a=np.zeros(cap_t, np.int32), axis_b=np.zeros(cap_t, np.int32),
        moving_count=np.zeros(cap_t, np.int32), moving=np.zeros(cap_m, np.int32))
    b = _capi.vs_ligand_buf()
    b.cap_atoms, b.cap_bonds, b.cap_tors, b.cap_moving = cap_a, cap_b, cap_t, cap_m
    b.coords = ptr(bufs["coords"], C.c_double)
    b.atom_class = ptr(bufs["atom_class"], C.c_int32)
    b.elements = C.cast(bufs["elements"], C.c_char_p)
    b.aromatic = ptr(bufs["aromatic"], C.c_uint8)
    b.bonds = ptr(bufs["bonds"], C.c_int32)
    b.ring = ptr(bufs["ring"], C.c_uint8)
    b.axis_a = ptr(bufs["axis_a"], C.c_int32)
    b.axis_b = ptr(bufs["axis_b"], C.c_int32)
    b.moving_count = ptr(bufs["moving_count"], C.c_int32)
    b.moving = ptr(bufs["moving"], C.c_int32)
    rc = _lib.vs_ligand_build(smiles.encode(), seed & (2**64 - 1), iterations, C.byref(b))
    if rc == _capi.VS_ERR_PARSE:
        raise ParseError(b.parse_kind, b.parse_pos, smiles)
    check(rc, None, "ligand build")
    n, nb, nt = b.n_atoms, b.n_bonds, b.n_tors
    raw = bufs["elements"].raw
    elements = [raw[3 * i:3 * i + 3].split(b"\0")[0].decode() for i in range(n)]
    graph = MolecularGraph(
        elements=elements,
        aromatic=[bool(x) for x in bufs["aromatic"][:n]],
        bonds=[tuple(int(v) for v in bufs["bonds"][3 * e:3 * e + 3]) for e in range(nb)],
        ring_bond_flags=[bool(x) for x in bufs["ring"][:nb]])
    axes, k = [], 0
    for j in range(nt):
        c = int(bufs["moving_count"][j])
        axes.append(Axis(int(bufs["axis_a"][j]), int(bufs["axis_b"][j]),
                         [int(v) for v in bufs["moving"][k:k + c]]))
        k += c
    coords = bufs["coords"][:3 * n].reshape(n, 3).copy()
    return graph, b.rot_bonds, coords, TorsionTopology(axes)


def parse_smiles(text: str) -> dict:
    """Graph dict as the pybind module returns it (module.cpp:46-58, 79-83)."""
    g, _, _, _ = _build(text, 0, -1)
    return {"atoms": [(e, a) for e, a in zip(g.elements, g.aromatic)],
            "bonds": list(g.bonds), "ring_bond_flags": list(g.ring_bond_flags)}


def rotatable_bonds(smiles: str) -> int:
    """chem::rotatable_bonds (chem.cpp:319-331)."""
    return _build(smiles, 0, -1)[1]


def embed_3d(smiles: str, seed: int = 0, iterations: int = 200) -> list[tuple[float, float, float]]:
    """chem::embed_3d (chem.cpp:406-446) as (x, y, z) tuples (module.cpp:88-95)."""
    coords = _build(smiles, seed, iterations)[2]
    return [tuple(float(v) for v in row) for row in coords]


def make_ligand(id: str, smiles: str, embed_seed: int | None = None,
                iterations: int = 200) -> Ligand:
    """chem::make_ligand (chem.cpp:333-341); with embed_seed also embeds and
    builds the torsion topology (dock.cpp:234)."""
    g, rot, coords, topo = _build(smiles, embed_seed or 0, iterations if embed_seed is not None else -1)
    lig = Ligand(id=id, smiles=smiles, graph=g, heavy_atoms=len(g.elements), rotatable_bonds=rot,
                 topology=topo)
    if embed_seed is not None:
        lig.conformer = Conformer(id, coords)
    return lig


def torsion_topology(smiles_or_ligand) -> TorsionTopology:
    """dock::torsion_topology (dock.cpp:234-270)."""
    if isinstance(smiles_or_ligand, Ligand):
        return smiles_or_ligand.topology
    return _build(smiles_or_ligand, 0, -1)[3]


def random_smiles(seed: int, index: int) -> str:
    """corpus::random_smiles(Rng(seed).split(index)) (tools/smiles_corpus.hpp:13-49)."""
    buf = C.create_string_buffer(4096)
    check(_lib.vs_random_smiles(seed, index, buf, 4096))
    return buf.value.decode()


@dataclass
class LibraryRecord:
    smiles: str
    id: str
    line_number: int


def read_library_records(lines: Iterable[str]) -> list[LibraryRecord]:
    """chem::read_library_records (chem.cpp:448-470)."""
    out = []
    for n, line in enumerate(lines, start=1):
        line = line.rstrip("\n")
        if line.endswith("\r"):
            line = line[:-1]
        if not line or line[0] == "#":
            continue
        if "\t" in line:
            smi, lid = line.split("\t", 1)
            lid = lid or f"L{n}"
        else:
            smi, lid = line, f"L{n}"
        out.append(LibraryRecord(smi, lid, n))
    return out


def read_library_file(path: str) -> list[LibraryRecord]:
    """chem::read_library_file (chem.cpp:472-476)."""
    try:
        with open(path, "rb") as f:
            text = f.read().decode("latin-1")
    except OSError as e:
        raise RuntimeError(f"cannot open library file: {path}") from e
    return read_library_records(text.split("\n") if text else [])


# ------------------------------------------------------------------ library
@dataclass
class Library:
    """A flattened ligand library in the C-ABI layout (capi.h vs_library)."""
    ids: list[str]
    n_atoms: np.ndarray
    n_tors: np.ndarray
    rot_bonds: np.ndarray
    coords: np.ndarray        # (A, 3) float64
    atom_class: np.ndarray    # (A,) int32
    axis_a: np.ndarray
    axis_b: np.ndarray
    moving_count: np.ndarray
    moving: np.ndarray
    seeds: np.ndarray         # uint64
    id_rank: np.ndarray       # uint32

    def __len__(self) -> int:
        return len(self.ids)

    def offsets(self):
        ao = np.concatenate([[0], np.cumsum(self.n_atoms, dtype=np.int64)])
        to = np.concatenate([[0], np.cumsum(self.n_tors, dtype=np.int64)])
        mo = np.concatenate([[0], np.cumsum(self.moving_count, dtype=np.int64)])
        return ao, to, mo

    def as_c(self) -> _capi.vs_library:
        for name in ("n_atoms", "n_tors", "rot_bonds", "atom_class", "axis_a", "axis_b",
                     "moving_count", "moving"):
            setattr(self, name, np.ascontiguousarray(getattr(self, name), dtype=np.int32))
        self.coords = np.ascontiguousarray(self.coords, dtype=np.float64)
        self.seeds = np.ascontiguousarray(self.seeds, dtype=np.uint64)
        self.id_rank = np.ascontiguousarray(self.id_rank, dtype=np.uint32)
        L = _capi.vs_library()
        L.n_ligands = len(self.ids)
        L.n_atoms = ptr(self.n_atoms, C.c_int32)
        L.n_tors = ptr(self.n_tors, C.c_int32)
        L.rot_bonds = ptr(self.rot_bonds, C.c_int32)
        L.coords = ptr(self.coords, C.c_double)
        L.atom_class = ptr(self.atom_class, C.c_int32)
        L.axis_a = ptr(self.axis_a, C.c_int32)
        L.axis_b = ptr(self.axis_b, C.c_int32)
        L.moving_count = ptr(self.moving_count, C.c_int32)
        L.moving = ptr(self.moving, C.c_int32)
        L.seeds = ptr(self.seeds, C.c_uint64)
        L.id_rank = ptr(self.id_rank, C.c_uint32)
        return L

    def subset(self, idx: Sequence[int]) -> "Library":
        ao, to, mo = self.offsets()
        idx = [int(i) for i in idx]
        a_sl = [np.arange(ao[i], ao[i + 1]) for i in idx]
        t_sl = [np.arange(to[i], to[i + 1]) for i in idx]
        m_sl = [np.arange(mo[to[i]], mo[to[i + 1]]) for i in idx]
        cat = lambda parts, dt: (np.concatenate(parts).astype(np.int64) if parts else np.zeros(0, np.int64))
        a_i, t_i, m_i = cat(a_sl, None), cat(t_sl, None), cat(m_sl, None)
        ids = [self.ids[i] for i in idx]
        return Library(ids=ids, n_atoms=self.n_atoms[idx], n_tors=self.n_tors[idx],
                       rot_bonds=self.rot_bonds[idx], coords=self.coords[a_i],
                       atom_class=self.atom_class[a_i], axis_a=self.axis_a[t_i],
                       axis_b=self.axis_b[t_i], moving_count=self.moving_count[t_i],
                       moving=self.moving[m_i], seeds=self.seeds[idx],
                       id_rank=id_ranks(ids))

    @staticmethod
    def from_ligands(ligs: Sequence[Ligand], seeds: Sequence[int]) -> "Library":
        coords, cls, aa, ab, mc, mv = [], [], [], [], [], []
        for lg in ligs:
            coords.append(np.asarray(lg.conformer.coords, np.float64).reshape(-1, 3))
            cls.append(lg.atom_classes())
            for ax in lg.topology.axes:
                aa.append(ax.a); ab.append(ax.b); mc.append(len(ax.moving)); mv.extend(ax.moving)
        ids = [lg.id for lg in ligs]
        return Library(
            ids=ids, n_atoms=np.array([lg.heavy_atoms for lg in ligs], np.int32),
            n_tors=np.array([len(lg.topology.axes) for lg in ligs], np.int32),
            rot_bonds=np.array([lg.rotatable_bonds for lg in ligs], np.int32),
            coords=np.concatenate(coords) if coords else np.zeros((0, 3)),
            atom_class=np.concatenate(cls) if cls else np.zeros(0, np.int32),
            axis_a=np.array(aa, np.int32), axis_b=np.array(ab, np.int32),
            moving_count=np.array(mc, np.int32), moving=np.array(mv, np.int32),
            seeds=np.array([int(s) & (2**64 - 1) for s in seeds], np.uint64),
            id_rank=id_ranks(ids))


def id_ranks(ids: Sequence[str]) -> np.ndarray:
    """Rank of each id in std::map (bytewise) order — the rank_ligands tie-break."""
    blob = b"".join(i.encode() + b"\0" for i in ids) or b"\0"
    out = np.zeros(max(len(ids), 1), np.uint32)
    check(_lib.vs_id_ranks(blob, len(ids), ptr(out, C.c_uint32)))
    return out[:len(ids)]


def corpus_indices(seed: int, n: int, atoms: tuple[int, int], tors: tuple[int, int],
                   threads: int = 8, max_scan: int | None = None) -> np.ndarray:
    """Indices of the first n corpus entries random_smiles(Rng(seed).split(i))
    whose heavy atoms / torsion axes lie in the inclusive bounds."""
    out = np.zeros(max(n, 1), np.int64)
    got = _lib.vs_corpus_select(seed, n, atoms[0], atoms[1], tors[0], tors[1],
                                max_scan or 50 * n + 100000, threads, ptr(out, C.c_int64))
    check(got)
    return out[:got]


def _relax_on(engine, h, iterations, place=False):
    """Placement-only build -> the spring relaxation of embed_3d on the GPU;
    place: a VS_EMBED_DEVICE build -> the BFS placement there too."""
    try:
        fn = _lib.vs_libbuild_embed if place else _lib.vs_libbuild_relax
        check(fn(engine._h, h, iterations), engine._h, "device embed")
    except Exception:
        _lib.vs_libbuild_free(h)
        raise


def _embed_mode(engine, device_place, iterations):
    if engine is None:
        return iterations
    return EMBED_DEVICE if device_place else EMBED_PLACE_ONLY


def corpus_library(seed: int, n: int, atoms: tuple[int, int], tors: tuple[int, int],
                   embed_master: int = 2024, dock_master: int = 2024, iterations: int = 200,
                   threads: int = 8, engine=None, device_place: bool = False) -> Library:
    """Synthetic library: corpus entries filtered to the size
    bounds; embed seed Rng(master).split(1).split(i), dock seed .split(2)
    .split(i) with i the index in the library (pipeline.cpp:422-484).
    With `engine`, embed_3d's spring relaxation runs on that GPU (bit-identical);
    device_place also moves the BFS placement there (CUDA log/cos in the
    jitter: coordinates within a tolerance of the host embed)."""
    from .pipeline import campaign_seeds
    idx = corpus_indices(seed, n, atoms, tors, threads)
    m = len(idx)
    es = campaign_seeds(embed_master, m, stage=1)
    ds = campaign_seeds(dock_master, m, stage=2)
    h = C.c_void_p()
    check(_lib.vs_libbuild_corpus(seed, ptr(idx, C.c_int64), m, ptr(es, C.c_uint64),
                                  _embed_mode(engine, device_place, iterations), threads,
                                  C.byref(h)))
    if engine is not None:
        _relax_on(engine, h, iterations, device_place)
    ids = [f"Z{int(i)}" for i in idx]
    return _fetch_built(h, m, ids, ds)


def flexible_smiles(seed: int, n: int, atoms=(60, 80), tors=(15, 20), max_scan: int = 400000):
    """C4 population: concatenations of consecutive corpus
    entries random_smiles(Rng(seed).split(i)) until the graph has >= atoms[0]
    heavy atoms; kept when atoms and torsion axes fall inside the bounds."""
    first = np.zeros(max(n, 1), np.int64)
    count = np.zeros(max(n, 1), np.int32)
    got = check(_lib.vs_flexible_select(seed, n, atoms[0], atoms[1], tors[0], tors[1], max_scan,
                                        ptr(first, C.c_int64), ptr(count, C.c_int32)))
    return ["".join(random_smiles(seed, int(first[k]) + c) for c in range(int(count[k])))
            for k in range(got)]


def _fetch_built(h, n, ids, ds, drop_failed=True) -> Library:
    try:
        A, T, M = C.c_int64(), C.c_int64(), C.c_int64()
        _lib.vs_libbuild_sizes(h, C.byref(A), C.byref(T), C.byref(M))
        st = np.zeros(max(n, 1), np.int32)
        na, nt, rb = (np.zeros(max(n, 1), np.int32) for _ in range(3))
        coords = np.zeros((max(A.value, 1), 3), np.float64)
        cls = np.zeros(max(A.value, 1), np.int32)
        aa, ab, mc = (np.zeros(max(T.value, 1), np.int32) for _ in range(3))
        mv = np.zeros(max(M.value, 1), np.int32)
        _lib.vs_libbuild_fetch(h, ptr(st, C.c_int32), ptr(na, C.c_int32), ptr(nt, C.c_int32),
                               ptr(rb, C.c_int32), ptr(coords, C.c_double), ptr(cls, C.c_int32),
                               ptr(aa, C.c_int32), ptr(ab, C.c_int32), ptr(mc, C.c_int32),
                               ptr(mv, C.c_int32))
    finally:
        _lib.vs_libbuild_free(h)
    st, na, nt, rb = st[:n], na[:n], nt[:n], rb[:n]
    lib = Library(ids=list(ids), n_atoms=na, n_tors=nt, rot_bonds=rb, coords=coords[:A.value],
                  atom_class=cls[:A.value], axis_a=aa[:T.value], axis_b=ab[:T.value],
                  moving_count=mc[:T.value], moving=mv[:M.value],
                  seeds=np.asarray(ds, np.uint64), id_rank=id_ranks(ids))
    lib.status = st
    if drop_failed and (st != 0).any():
        keep = np.nonzero(st == 0)[0]
        status = st[keep]
        lib = lib.subset(keep)
        lib.status = status
    return lib


def build_library(smiles: Sequence[str], ids: Sequence[str] | None = None,
                  embed_seeds: Sequence[int] | None = None, dock_seeds: Sequence[int] | None = None,
                  iterations: int = 200, threads: int = 8, drop_failed: bool = True,
                  engine=None, device_place: bool = False) -> Library:
    """Parse + embed + topology for many ligands on `threads` host threads
    (the parse/embed stages of run_campaign, pipeline.cpp:383-431).  With
    `engine` (a dock.Engine), the host does parse, topology and embed_3d's
    BFS placement, and the spring relaxation runs on the GPU (bit-identical
    coordinates); with device_place the whole embed_3d runs on
    the GPU (coordinates within a tolerance: CUDA log/cos in the jitter)."""
    n = len(smiles)
    ids = list(ids) if ids is not None else [f"L{i + 1}" for i in range(n)]
    es = np.array([int(s) & (2**64 - 1) for s in (embed_seeds if embed_seeds is not None else [0] * n)],
                  np.uint64)
    blob = b"".join(s.encode() + b"\0" for s in smiles) or b"\0"
    h = C.c_void_p()
    check(_lib.vs_libbuild_run(blob, n, ptr(es, C.c_uint64),
                               _embed_mode(engine, device_place, iterations), threads, C.byref(h)))
    if engine is not None:
        _relax_on(engine, h, iterations, device_place)
    ds = np.array([int(s) & (2**64 - 1) for s in (dock_seeds if dock_seeds is not None else [0] * n)],
                  np.uint64)
    return _fetch_built(h, n, ids, ds, drop_failed)
