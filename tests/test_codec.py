"""SMZC compressed-library reading (the ingest feed of
run_campaign, pipeline.cpp:384-396) against the reference codec.

Golden: tests/golden/codec/ holds SMZC files written by the reference's
codec::compress_stream (tests/golden/make_codec_golden.py); decoding them
must give the sample library byte for byte.  With oracle/_ref present, a
random corpus is compressed and decoded by the reference and decoded by the
native multithreaded decoder, and the error cases (codec.cpp:183-289) raise
the reference's exception type with the reference's message."""
import hashlib
import json
import os
import shutil

import pytest

from conftest import GOLDEN, need_ref

CODEC = os.path.join(GOLDEN, "codec")
CAMP = os.path.join(GOLDEN, "campaign")


@pytest.fixture(scope="module")
def K():
    from paper_2304_09953_b200 import codec
    return codec


def _sample():
    return open(os.path.join(CAMP, "sample_library_100.smi"), "rb").read().decode("latin-1")


@pytest.mark.parametrize("lib,dic", [("library_100.smzc", "../campaign/smiles.dict"),
                                     ("library_trained.smzc", "trained.dict")])
def test_golden_smzc_decodes_to_sample_library(K, lib, dic):
    for threads in (1, 4):
        text = K.decompress_file(os.path.join(CODEC, lib), os.path.join(CODEC, dic),
                                 threads=threads)
        assert text == _sample()


def test_golden_hash_pins_the_dictionary(K):
    with pytest.raises(K.BadFormat, match="dictionary hash mismatch"):
        K.decompress_file(os.path.join(CODEC, "library_100.smzc"),
                          os.path.join(CODEC, "trained.dict"))
    with pytest.raises(K.BadFormat, match="cannot open dictionary"):
        K.decompress_file(os.path.join(CODEC, "library_100.smzc"), "/nonexistent.dict")


def _corpus(R, n, seed):
    lines = [R.random_smiles(seed, i) + f"\tZ{i}" for i in range(n)]
    lines[3:3] = ["", "# comment", "C" * 300]  # empty, comment, long record (2-byte varint)
    return ("\n".join(lines) + "\n").encode()


def test_random_corpus_matches_reference_decoder(K, tmp_path):
    R = need_ref()
    text = _corpus(R, 6000, 17)  # > 4096 records: the threaded path
    dic = R.train_dictionary(text, 128)
    dp = tmp_path / "c.dict"
    dp.write_bytes(dic)
    data = R.smzc_compress(text, str(dp))
    ref = R.smzc_decompress(data, str(dp))
    assert ref == text
    for threads in (1, 3, 16):
        assert K.decompress(dic, data, threads=threads).encode("latin-1") == ref
    # no trailing newline: getline still yields the last line
    t2 = text.rstrip(b"\n")
    d2 = R.smzc_compress(t2, str(dp))
    assert K.decompress(dic, d2).encode("latin-1") == R.smzc_decompress(d2, str(dp))
    # empty library: header only
    d0 = R.smzc_compress(b"", str(dp))
    assert len(d0) == 36 and K.decompress(dic, d0) == ""


def _ref_message(R, fn):
    with pytest.raises(R.RefError) as e:
        fn()
    return str(e.value).split(": ", 1)[1]


def test_error_cases_match_reference(K, tmp_path):
    R = need_ref()
    text = _corpus(R, 50, 5)
    dic = R.train_dictionary(text, 32)
    dp = tmp_path / "c.dict"
    dp.write_bytes(dic)
    data = R.smzc_compress(text, str(dp))
    digest = hashlib.sha256(dic).digest()
    n_entries = dic[4]
    cases = {
        "magic": b"SMZX" + data[4:],
        "short_hash": data[:20],
        "trunc_payload": data[:-3],
        "trunc_varint": data[:36] + b"\x85",
        "varint_overflow": data[:36] + b"\xff" * 10 + b"\x01",
        # an unknown code in record 1 comes before a truncation later on
        "unknown_code": b"SMZC" + digest + b"\x02CC" + bytes([2, 0x41, 0x80 + n_entries]) + b"\x05C",
    }
    for name, blob in cases.items():
        ref_msg = _ref_message(R, lambda: R.smzc_decompress(blob, str(dp)))
        exc = K.UnknownCode if name == "unknown_code" else K.BadFormat
        with pytest.raises(exc) as e:
            K.decompress(dic, blob)
        assert str(e.value) == ref_msg, name
        if name == "unknown_code":
            assert e.value.code == 0x80 + n_entries and e.value.offset == 1
    # malformed dictionaries: load_dictionary's checks, in its order
    bad_dicts = {
        "magic": b"SMZ2" + dic[4:],
        "header": b"SMZ1",
        "count": b"SMZ1" + bytes([129]),
        "entry_len": b"SMZ1\x01\x01C",
        "entry_trunc": b"SMZ1\x02\x02CC\x03CC",
        "printable": b"SMZ1\x01\x02C\x01",
        "duplicate": b"SMZ1\x02\x02CC\x02CC",
    }
    for name, d in bad_dicts.items():
        p = tmp_path / f"{name}.dict"
        p.write_bytes(d)
        ref_msg = _ref_message(R, lambda: R.smzc_decompress(data, str(p)))
        with pytest.raises(K.BadFormat) as e:
            K.load_dictionary_file(str(p))
        assert str(e.value) == ref_msg, name


def test_campaign_reads_a_compressed_library(tmp_path):
    """prepare() on an .smzc library equals prepare() on the plain .smi."""
    from paper_2304_09953_b200 import campaign as Cm
    for f in ("pocket.json", "sample_library_100.smi"):
        shutil.copy(os.path.join(CAMP, f), tmp_path / f)
    shutil.copy(os.path.join(CODEC, "library_100.smzc"), tmp_path / "lib.smzc")
    shutil.copy(os.path.join(CAMP, "smiles.dict"), tmp_path / "smiles.dict")
    j = json.load(open(os.path.join(CAMP, "campaign_100.json")))
    plain = Cm.parse_config_json(json.dumps(j), str(tmp_path))
    jz = dict(j, library="lib.smzc", dictionary="smiles.dict")
    packed = Cm.parse_config_json(json.dumps(jz), str(tmp_path))
    assert packed.dictionary_path.endswith("smiles.dict")
    a = Cm.prepare(plain, threads=4)
    b = Cm.prepare(packed, threads=4)
    assert list(a[0].ids) == list(b[0].ids)
    assert (a[0].coords == b[0].coords).all() and (a[0].seeds == b[0].seeds).all()
    assert [s.to_json() for s in a[1]] == [s.to_json() for s in b[1]]
    assert [t.ligand_ids for t in a[2]] == [t.ligand_ids for t in b[2]]
    nodict = dict(jz)
    del nodict["dictionary"]
    with pytest.raises(Cm.ConfigError, match="needs a dictionary"):
        Cm.prepare(Cm.parse_config_json(json.dumps(nodict), str(tmp_path)))
    # validate_config (pipeline.cpp:172-178): missing files at parse time
    with pytest.raises(Cm.ConfigError, match="dictionary file not found"):
        Cm.parse_config_json(json.dumps(dict(jz, dictionary="x.dict")), str(tmp_path))
    with pytest.raises(Cm.ConfigError, match="library file not found"):
        Cm.parse_config_json(json.dumps(dict(jz, library="x.smzc")), str(tmp_path))
    # a dictionary that is not SMZ1: BadFormat from the parse stage
    (tmp_path / "bad.dict").write_bytes(b"nope")
    from paper_2304_09953_b200.codec import BadFormat
    with pytest.raises(BadFormat, match="bad dictionary magic"):
        Cm.prepare(Cm.parse_config_json(json.dumps(dict(jz, dictionary="bad.dict")),
                                        str(tmp_path)))


def test_cpp_dropin_codec_read_side(tmp_path):
    """include/vscreen/codec.hpp + libvscreen_core.so as a reference C++
    caller reads an SMZC library (pipeline.cpp:390-396): tests/cpp/codec_read.cpp."""
    import subprocess
    from conftest import ROOT
    exe = tmp_path / "codec_read"
    libdir = os.path.join(ROOT, "paper_2304_09953_b200")
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "cpp", "codec_read.cpp"), f"-L{libdir}",
                    "-lvscreen_core", "-lvscreen_gpu", f"-Wl,-rpath,{libdir}", "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe), CODEC, CAMP], capture_output=True, text=True)
    assert out.returncode == 0 and "codec ok" in out.stdout, out.stdout + out.stderr


def test_pybind_codec_read_functions(tmp_path):
    """load_dictionary / decompress_line as module.cpp:114-125 expose them
    (known answers of test_codec.cpp:92-108 and the golden dictionary)."""
    import paper_2304_09953_b200 as V
    assert V.decompress_line(bytes([0x80, ord("O")]), ["CC"]) == "CCO"
    assert V.decompress_line(b"", []) == ""
    with pytest.raises(V.codec.UnknownCode) as e:
        V.decompress_line(bytes([0x90]), [])
    assert e.value.code == 0x90 and e.value.offset == 0
    entries = V.load_dictionary(os.path.join(CAMP, "smiles.dict"))
    raw = open(os.path.join(CAMP, "smiles.dict"), "rb").read()
    assert len(entries) == raw[4] and all(2 <= len(x) <= 8 for x in entries)
    R = need_ref()
    assert entries == R.dictionary_entries(os.path.join(CAMP, "smiles.dict"))
