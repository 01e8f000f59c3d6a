"""Host embed_3d vs placement-only + GPU relaxation on a
corpus library: wall time of each stage."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(n=20000):
    import paper_2304_09953_b200 as V
    from paper_2304_09953_b200 import chem
    from paper_2304_09953_b200._capi import lib as L, ptr
    from paper_2304_09953_b200.errors import check
    from paper_2304_09953_b200.pipeline import campaign_seeds
    th = os.cpu_count()
    idx = chem.corpus_indices(5, n, (10, 40), (0, 10), th)
    m = len(idx)
    es = campaign_seeds(2024, m, stage=1)
    eng = V.Engine(0)
    for rep in range(2):
        for it in (200, chem.EMBED_PLACE_ONLY, chem.EMBED_DEVICE):
            h = C.c_void_p()
            t0 = time.perf_counter()
            check(L.vs_libbuild_corpus(5, ptr(idx, C.c_int64), m, ptr(es, C.c_uint64), it, th,
                                       C.byref(h)))
            t1 = time.perf_counter()
            msg = f"n={m} threads={th} build(iter={it}) {1e3 * (t1 - t0):.1f} ms"
            if it in (chem.EMBED_PLACE_ONLY, chem.EMBED_DEVICE):
                t2 = time.perf_counter()
                fn = L.vs_libbuild_relax if it == chem.EMBED_PLACE_ONLY else L.vs_libbuild_embed
                check(fn(eng._h, h, 200), eng._h, "device embed")
                what = "relax" if it == chem.EMBED_PLACE_ONLY else "place + relax"
                msg += f"  gpu {what} {1e3 * (time.perf_counter() - t2):.1f} ms"
            L.vs_libbuild_free(h)
            print(msg, flush=True)
    eng.close()


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
