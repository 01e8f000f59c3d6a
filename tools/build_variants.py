"""Build experiment variants of the library into variants/ (git-ignored,
travels with gpurun):  python tools/build_variants.py NAME=DEF1,DEF2 ...
then on the GPU: VSCREEN_GPU_LIB=variants/lib_NAME.so python tools/profile_dock.py"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2304_09953_b200 import build as B  # noqa: E402


def one(spec):
    name, _, defs = spec.partition("=")
    defines = tuple(d for d in defs.split(",") if d)
    out = os.path.join(ROOT, "variants", f"lib_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    B.build(force=True, defines=defines or ("VS_VARIANT_" + name,), out=out)
    return out


if __name__ == "__main__":
    with ThreadPoolExecutor(8) as ex:
        for o in ex.map(one, sys.argv[1:]):
            print(o)
