"""Build the in-tree native library ``libvscreen_gpu.so`` (sm_100a).

One shared object holds the CUDA kernels, the GPU runtime and the host-side
C-ABI (ingest, batcher, rank).  Built in-tree so it travels to the GPU box
with the repo snapshot.  ``--fmad=false`` keeps the device arithmetic exactly
the spec's (every FMA is an explicit ``fmaf``); host code is compiled by the
system g++ with its defaults so FP64 ingest matches the reference bit for bit.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvscreen_gpu.so")
# the C++ drop-in for the reference's own API (include/vscreen/*.hpp): the
# library reference callers link instead of the CPU vscreen_core
CORE = os.path.join(HERE, "libvscreen_core.so")
DROPIN = ["vs_dropin_chem.cpp", "vs_dropin_dock.cpp", "vs_dropin_batcher.cpp",
          "vs_dropin_report.cpp", "vs_dropin_codec.cpp"]
SOURCES = ["vs_kernels.cu", "vs_dock.cu", "vs_grad.cu", "vs_embed.cu", "vs_pack.cu", "vs_runtime.cu",
           "vs_host.cpp", "vs_ingest.cpp", "vs_codec.cpp", "vs_json.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "--fmad=false", "-ccbin", "/usr/bin/g++",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-diag-suppress", "550"]


def _stale(lib=LIB, extra=()) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + list(extra)
    deps.append(os.path.join(HERE, "..", "include", "vscreen_gpu", "capi.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _json_dir() -> str:
    import sysconfig
    return os.path.join(sysconfig.get_paths()["purelib"], "include", "cudnn_frontend", "thirdparty")


def build_core(force: bool = False, verbose: bool = False) -> str:
    """libvscreen_core.so: the drop-in for the reference's C++ API, linked
    against libvscreen_gpu.so (found next to it at run time)."""
    inc = os.path.join(HERE, "..", "include")
    srcs = [os.path.join(CSRC, "dropin", f) for f in DROPIN]
    extra = srcs + [os.path.join(inc, "vscreen", f) for f in os.listdir(os.path.join(inc, "vscreen"))]
    if not force and not _stale(CORE, extra) and os.path.getmtime(CORE) >= os.path.getmtime(LIB):
        return CORE
    cmd = ["/usr/bin/g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", f"-I{inc}",
           f"-I{_json_dir()}", *srcs, f"-L{HERE}", "-lvscreen_gpu", "-Wl,-rpath,$ORIGIN",
           "-o", CORE + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(CORE + ".tmp", CORE)
    return CORE


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Build the library; `defines`/`out` produce experiment variants
    (e.g. defines=("VS_MINB=5",), out=".../libvscreen_gpu.minb5.so")."""
    lib = out or LIB
    if not force and not defines and out is None and not _stale():
        build_core(verbose=verbose)
        return LIB
    tag = "_".join(d.replace("=", "") for d in defines) or "default"
    objs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, "_build", tag, src + ".o")
        os.makedirs(os.path.dirname(obj), exist_ok=True)
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src),
               "-o", obj]
        if src == "vs_json.cpp":
            cmd[1:1] = [f"-I{_json_dir()}"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(obj)
    cmd = [NVCC, *ARCH, "-shared", "-ccbin", "/usr/bin/g++", *objs, "-o", lib + ".tmp", "-lpthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(lib + ".tmp", lib)
    if out is None and not defines:
        build_core(force=True, verbose=verbose)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
