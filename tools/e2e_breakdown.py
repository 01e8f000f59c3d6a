"""Host-clock breakdown of the end-to-end path (vs_dock_host) on the C2
workload: upload (pack + H2D), dock (device), fetch (D2H + unpack), top-k."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(n=100_000, pinned=0):
    import bench
    import paper_2304_09953_b200 as V
    lib, _, _ = bench.build_workload(n, 0, 1, os.cpu_count() or 1)
    if pinned:
        bench.pin_library(lib)
    eng = V.Engine(0)
    eng.set_pocket(bench.make_pocket(), grid_spacing=0.4, grid_pad=2.0)
    prm = bench.params()
    out = eng.alloc_results(lib, prm, pinned=bool(pinned))
    eng.dock_host(lib, prm, out=out)
    for _ in range(2):
        t0 = time.perf_counter()
        eng.upload(lib)
        t1 = time.perf_counter()
        eng.dock(prm)
        eng.last_dock_ms()  # synchronizes on the dock's end event
        t2 = time.perf_counter()
        eng.fetch(out)
        t3 = time.perf_counter()
        eng.topk(1000)
        t4 = time.perf_counter()
        print(f"upload {1e3 * (t1 - t0):.1f} ms  dock {1e3 * (t2 - t1):.1f} ms  "
              f"fetch {1e3 * (t3 - t2):.1f} ms  topk {1e3 * (t4 - t3):.1f} ms  "
              f"total {1e3 * (t4 - t0):.1f} ms  -> {n / (t4 - t0):.0f} ligands/s")
        t0 = time.perf_counter()
        eng.dock_host(lib, prm, out=out)
        t1 = time.perf_counter()
        eng.topk(1000)
        print(f"dock_host {1e3 * (t1 - t0):.1f} ms (device span {eng.last_dock_ms():.1f} ms) "
              f"+ topk {1e3 * (time.perf_counter() - t1):.1f} ms")
    eng.close()


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
