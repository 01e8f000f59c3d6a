"""A reference-style C++ caller (tests/cpp/dropin_example.cpp: the
reference's own API from include/vscreen/ plus the library-scale C-ABI)
compiles, links libvscreen_core.so and runs: host functions on the CPU; the
GPU entry points fail loudly without a device and return the reference's
known answers (test_dock.cpp:45-47, 172-184) with one."""
import os
import subprocess

import pytest

from conftest import ROOT, gpu_available


def _build(tmp_path):
    exe = tmp_path / "dropin"
    libdir = os.path.join(ROOT, "paper_2304_09953_b200")
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp"), f"-L{libdir}",
                    "-lvscreen_core", "-lvscreen_gpu", f"-Wl,-rpath,{libdir}", "-o", str(exe)],
                   check=True)
    return str(exe)


def test_cpp_dropin_builds_and_runs(tmp_path):
    out = subprocess.run([_build(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "dropin ok" in out.stdout


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_cpp_dropin_on_gpu(tmp_path):
    out = subprocess.run([_build(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "gpu ok" in out.stdout and "batch ok" in out.stdout
