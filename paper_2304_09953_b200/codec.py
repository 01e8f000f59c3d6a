"""SMZC compressed-library decompression (the reference codec's read side,
codec.hpp:41-79) over the native multithreaded decoder
(capi.h vs_smzc_decompress): the text equals the reference's
decompress_stream output byte for byte, so read_library_records over it
gives the reference's records."""
from __future__ import annotations

import ctypes as C
import os
import re

from ._capi import lib as _lib
from .errors import BadFormat, UnknownCode, check


def decompress(dictionary: bytes, data: bytes, threads: int | None = None) -> str:
    """Decode an SMZC library (bytes) with its SMZ1 dictionary (bytes)."""
    threads = threads or os.cpu_count() or 1
    need = C.c_int64()
    rc = _lib.vs_smzc_decompress(dictionary, len(dictionary), data, len(data), threads, None, 0,
                                 C.byref(need))
    if rc < 0:
        _raise_last()
    buf = C.create_string_buffer(max(need.value, 1))
    rc = _lib.vs_smzc_decompress(dictionary, len(dictionary), data, len(data), threads, buf,
                                 need.value, C.byref(need))
    check(rc, None, "smzc")
    return buf.raw[:need.value].decode("latin-1")


def _raise_last() -> None:
    msg = _lib.vs_codec_last_error().decode()
    m = re.fullmatch(r"unknown code byte 0x([0-9a-f]+) at offset (\d+)", msg)
    if m:
        raise UnknownCode(int(m.group(1), 16), int(m.group(2)))
    raise BadFormat(msg)


def load_dictionary_file(path: str) -> bytes:
    """codec::load_dictionary_file (codec.cpp:217-221): the validated SMZ1
    bytes; BadFormat as the reference raises it."""
    try:
        with open(path, "rb") as f:
            d = f.read()
    except OSError as e:
        raise BadFormat(f"cannot open dictionary: {path}") from e
    n = C.c_int32()
    if _lib.vs_smz1_check(d, len(d), C.byref(n)) < 0:
        _raise_last()
    return d


def decompress_file(path: str, dictionary_path: str, threads: int | None = None) -> str:
    """codec::decompress_stream of a .smzc file with its dictionary file."""
    d = load_dictionary_file(dictionary_path)
    with open(path, "rb") as f:
        data = f.read()
    return decompress(d, data, threads)


def load_dictionary(path: str) -> list[str]:
    """module.cpp:123-125: the entries of an SMZ1 dictionary file (code byte
    0x80 + i <-> entries[i]); BadFormat as the reference raises it."""
    d = load_dictionary_file(path)
    out, o = [], 5
    for _ in range(d[4]):
        n = d[o]
        out.append(d[o + 1:o + 1 + n].decode("ascii"))
        o += 1 + n
    return out


def decompress_line(data: bytes, entries: list[str]) -> str:
    """module.cpp:114-121 / codec.cpp:147-161: one record's bytes expanded
    with the dictionary entries; UnknownCode(code, offset) for a code byte
    without an entry."""
    out = []
    for i, b in enumerate(bytes(data)):
        if b < 0x80:
            out.append(chr(b))
        elif b - 0x80 < len(entries):
            out.append(entries[b - 0x80])
        else:
            raise UnknownCode(b, i)
    return "".join(out)
