"""The C-ABI library loads and exports every symbol include/vscreen_gpu/capi.h
declares; without a GPU the runtime reports VS_ERR_NO_DEVICE instead of
falling back to the CPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ROOT, gpu_available

HEADER = os.path.join(ROOT, "include", "vscreen_gpu", "capi.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("vs_create", "vs_set_pocket", "vs_upload_library", "vs_dock", "vs_dock_host",
                 "vs_fetch_results", "vs_topk", "vs_topk_merge_device", "vs_rescore",
                 "vs_bucket_replay", "vs_rank_ligands", "vs_filter_poses"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2304_09953_b200 import _capi
    lib = C.CDLL(_capi.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes table binds exactly what the header declares
    assert set(_capi.EXPORTED) == set(declared())


def test_exports_via_nm():
    from paper_2304_09953_b200 import _capi
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    assert set(declared()) <= syms


def test_kernels_are_sm100a():
    from paper_2304_09953_b200 import _capi
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(gpu_available(), reason="CPU-only check")
def test_no_device_is_an_error_not_a_fallback():
    import paper_2304_09953_b200 as V
    from paper_2304_09953_b200.errors import DeviceError
    with pytest.raises(DeviceError):
        V.Engine(0)


def test_key_encoding_roundtrip():
    from paper_2304_09953_b200 import _capi
    import numpy as np
    for s in (1.5, -2.25, 0.0, 123.0, -1e-3):
        f = np.float32(s)
        b = int(f.view(np.uint32))
        ordv = (~b & 0xFFFFFFFF) if b & 0x80000000 else (b | 0x80000000)
        key = ((~ordv & 0xFFFFFFFF) << 32) | 17
        assert _capi.lib.vs_key_score(key) == f
        assert _capi.lib.vs_key_id_rank(key) == 17


def test_no_device_entry_points_fail_loudly():
    """Without a GPU the device entry points report it (no CPU fallback):
    page-locked allocation and handle creation."""
    import ctypes as C
    from conftest import gpu_available
    if gpu_available():
        pytest.skip("a GPU is present")
    import numpy as np
    from paper_2304_09953_b200 import _capi
    from paper_2304_09953_b200.dock import pinned_empty
    from paper_2304_09953_b200.errors import VscreenError
    with pytest.raises(VscreenError):
        pinned_empty(16, np.float32)
    h = C.c_void_p()
    assert _capi.lib.vs_create(0, C.byref(h)) == _capi.VS_ERR_NO_DEVICE
    p = C.c_void_p()
    assert _capi.lib.vs_host_alloc(64, C.byref(p)) == _capi.VS_ERR_NO_DEVICE and not p.value
