"""Size-class batcher — mirror of proj/include/vscreen/batcher.hpp backed by the
native host functions (vs_host.cpp).  The same classes are the packer's
device launch buckets."""
from __future__ import annotations

import ctypes as C
from collections import deque
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _capi
from ._capi import lib as _lib, ptr
from .errors import ItemTooLarge, OutOfRange, check


@dataclass(frozen=True)
class SizeClass:
    """batcher::SizeClass (batcher.hpp:33-40): half-open ranges."""
    atom_lo: int
    atom_hi: int
    rot_lo: int
    rot_hi: int

    def contains(self, atoms: int, rot: int) -> bool:
        return self.atom_lo <= atoms < self.atom_hi and self.rot_lo <= rot < self.rot_hi

    def astuple(self):
        return (self.atom_lo, self.atom_hi, self.rot_lo, self.rot_hi)


@dataclass
class DeviceModel:
    """batcher::DeviceModel (batcher.hpp:17-29)."""
    memory_capacity: float = 0.0
    mem_fixed: float = 0.0
    mem_per_atom: float = 0.0
    mem_per_rotbond: float = 0.0
    launch_overhead: float = 0.0
    service_time_per_class: list[float] = field(default_factory=list)

    def service_time(self, cls: int) -> float:
        s = self.service_time_per_class
        return s[cls] if cls < len(s) else s[-1]


def _cls_array(classes: Sequence[SizeClass]):
    arr = (_capi.vs_size_class * max(1, len(classes)))()
    for i, c in enumerate(classes):
        arr[i].atom_lo, arr[i].atom_hi, arr[i].rot_lo, arr[i].rot_hi = c.astuple()
    return arr


def default_classes() -> list[SizeClass]:
    """batcher::default_classes (batcher.cpp:7-17)."""
    arr = (_capi.vs_size_class * 8)()
    n = check(_lib.vs_default_classes(arr, 8))
    return [SizeClass(arr[i].atom_lo, arr[i].atom_hi, arr[i].rot_lo, arr[i].rot_hi) for i in range(n)]


def size_class(heavy_atoms: int, rotatable_bonds: int, classes: Sequence[SizeClass],
               ligand_id: str = "L") -> int:
    """batcher::size_class (batcher.cpp:19-26)."""
    rc = _lib.vs_size_class_of(heavy_atoms, rotatable_bonds, _cls_array(classes), len(classes))
    if rc < 0:
        raise OutOfRange(f"ligand {ligand_id} ({heavy_atoms} atoms, {rotatable_bonds} rotatable "
                         "bonds) fits no size class")
    return rc


def target_batch_size(memory_capacity: float, mem_fixed: float, mem_per_atom: float,
                      mem_per_rotbond: float, atom_hi: int, rot_hi: int) -> int:
    """batcher::target_batch_size (batcher.cpp:28-38), pybind signature
    (module.cpp:163-176)."""
    c = _capi.vs_size_class(0, atom_hi, 0, rot_hi)
    out = C.c_int64()
    rc = _lib.vs_target_batch_size(C.byref(c), memory_capacity, mem_fixed, mem_per_atom,
                                   mem_per_rotbond, C.byref(out))
    if rc == _capi.VS_ERR_ITEM_TOO_LARGE:
        item = mem_per_atom * atom_hi + mem_per_rotbond * rot_hi
        raise ItemTooLarge(f"worst-case item memory {item} exceeds device budget "
                           f"{memory_capacity - mem_fixed}")
    check(rc)
    return int(out.value)


def simulate_throughput(n_items: int, launch_overhead_s: float, service_time_s: float) -> float:
    """batcher::simulate_throughput (batcher.cpp:40-43), pybind signature."""
    return float(_lib.vs_simulate_throughput(n_items, launch_overhead_s, service_time_s))


@dataclass
class Batch:
    cls: int
    ligand_ids: list[str]


class BatchQueue:
    """batcher::BatchQueue (batcher.cpp:45-86): per-class FIFO flushed at the
    class target size or when the oldest entry is older than max_age."""

    def __init__(self, classes: Sequence[SizeClass], dev: DeviceModel, max_age: float = 1.0):
        self.classes = list(classes)
        self.targets = [target_batch_size(dev.memory_capacity, dev.mem_fixed, dev.mem_per_atom,
                                          dev.mem_per_rotbond, c.atom_hi, c.rot_hi)
                        for c in self.classes]
        self.buffers = [deque() for _ in self.classes]
        self.max_age = max_age

    def _drain(self, cls: int) -> Batch:
        b = Batch(cls, [e[0] for e in self.buffers[cls]])
        self.buffers[cls].clear()
        return b

    def enqueue(self, ligand_id: str, cls: int, now: float) -> Batch | None:
        if cls >= len(self.classes):
            raise OutOfRange("class index out of range")
        self.buffers[cls].append((ligand_id, now))
        if len(self.buffers[cls]) >= self.targets[cls]:
            return self._drain(cls)
        return None

    def flush_aged(self, now: float) -> list[Batch]:
        return [self._drain(c) for c, b in enumerate(self.buffers)
                if b and now - b[0][1] > self.max_age]

    def flush_all(self) -> list[Batch]:
        return [self._drain(c) for c, b in enumerate(self.buffers) if b]

    def buffered(self, cls: int) -> int:
        return len(self.buffers[cls])

    def target(self, cls: int) -> int:
        return self.targets[cls]


def bucket_replay(atoms: Sequence[int], rot: Sequence[int], classes: Sequence[SizeClass],
                  dev: DeviceModel, max_age: float = 1.0):
    """The dock-stage bucket replay of run_campaign (pipeline.cpp:439-461) in
    native code: returns (in_range[n], [(class, [ligand indices])...])."""
    n = len(atoms)
    a = np.ascontiguousarray(atoms, np.int32)
    r = np.ascontiguousarray(rot, np.int32)
    in_range = np.zeros(max(n, 1), np.int32)
    bc = np.zeros(max(n, 1), np.int32)
    bl = np.zeros(max(n, 1), np.int32)
    mem = np.zeros(max(n, 1), np.int32)
    nb = _lib.vs_bucket_replay(ptr(a, C.c_int32), ptr(r, C.c_int32), n, _cls_array(classes),
                               len(classes), dev.memory_capacity, dev.mem_fixed, dev.mem_per_atom,
                               dev.mem_per_rotbond, max_age, ptr(in_range, C.c_int32),
                               ptr(bc, C.c_int32), ptr(bl, C.c_int32), ptr(mem, C.c_int32))
    if nb == _capi.VS_ERR_ITEM_TOO_LARGE:
        raise ItemTooLarge("worst-case item memory exceeds device budget")
    check(nb)
    batches, k = [], 0
    for b in range(nb):
        batches.append((int(bc[b]), [int(v) for v in mem[k:k + bl[b]]]))
        k += int(bl[b])
    return in_range[:n].astype(bool), batches
