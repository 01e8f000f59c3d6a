"""Summarise one profiling round (tools/profile_round.sh TAG) into profiles/:

  profiles/<TAG>_launches.json     per-kernel share of the bench launch list
  profiles/<TAG>_dock_ncu.json     key metrics + stall breakdown of the dock kernel
  profiles/<TAG>_dock_functions.txt per-subroutine samples (tools/ncu_funcs.py)
  profiles/<TAG>_dock_lines.txt    hottest source lines (tools/sass_lines.py)
  profiles/ncu_dock_traffic.json   DRAM bytes per C2 dock launch (bench roofline.traffic)

  python tools/ncu_summary.py TAG     (reads gpurun_out/*_TAG.*, needs ncu + nvdisasm)
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys
import tempfile
from contextlib import redirect_stdout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]


def launches(tag):
    rows = [r for r in csv.reader(open(os.path.join(OUT, f"launches_{tag}.csv"))) if len(r) > 10]
    h = rows[0]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        name = r[ik].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    return {"source": f"ncu --metrics gpu__time_duration.sum --clock-control none (bench.py --steps 2 "
                      f"--warmup 3 --no-cpu --no-e2e), gpurun_out/launches_{tag}.csv",
            "note": "serialised, cold-cache launches: compare shares, not absolute times",
            "kernels": [{"kernel": k, "launches": v[0], "ms": round(v[1] / 1e6, 3),
                         "share": round(v[1] / tot, 4)}
                        for k, v in sorted(agg.items(), key=lambda x: -x[1][1])]}


def traffic(tag):
    rows = [r for r in csv.reader(open(os.path.join(OUT, f"traffic_{tag}.csv"))) if len(r) > 10]
    h = rows[0]
    vals = {r[h.index("Metric Name")]: float(r[h.index("Metric Value")].replace(",", ""))
            for r in rows[1:]}
    rd, wr = vals["dram__bytes_read.sum"], vals["dram__bytes_write.sum"]
    return {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k vs_dock_kernel "
                      f"-c 1 on bench.py (C2, 100k ligands, one launch), gpurun_out/traffic_{tag}.csv",
            "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
            "kernel_ns": vals.get("gpu__time_duration.sum")}


def dock_report(tag):
    rep = os.path.join(OUT, f"prof_dock_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rows[0], rows[2]))
    out = {"source": f"ncu --set full --clock-control none --import-source on, tools/profile_dock.py "
                     f"--ligands 20000 (C2 library prefix), gpurun_out/prof_dock_{tag}.ncu-rep",
           "metrics": {k: d.get(k) for k in METRICS}, "stalls_per_issue": {}}
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith(
                "_per_issue_active.ratio"):
            try:
                if float(v) >= 0.05:
                    out["stalls_per_issue"][k[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]] = round(float(v), 3)
            except ValueError:
                pass
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    return out, src


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    json.dump(launches(tag), open(os.path.join(PROF, f"{tag}_launches.json"), "w"), indent=1)
    t = traffic(tag)
    json.dump(t, open(os.path.join(PROF, "ncu_dock_traffic.json"), "w"), indent=1)
    summ, src = dock_report(tag)
    summ["dram_traffic_c2_launch"] = t
    json.dump(summ, open(os.path.join(PROF, f"{tag}_dock_ncu.json"), "w"), indent=1)
    with tempfile.TemporaryDirectory() as td:
        lib = os.path.join(ROOT, "paper_2304_09953_b200", "libvscreen_gpu.so")
        subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=td, capture_output=True)
        sass = os.path.join(td, "dock.sass")
        with open(sass, "w") as f:
            subprocess.run(["nvdisasm", "-g", os.path.join(td, "vs_dock.sm_100a.cubin")], stdout=f)
        csvp = os.path.join(td, "src.csv")
        open(csvp, "w").write(src)
        import ncu_funcs
        import sass_lines
        kp = "_ZN2vs14vs_dock_kernelILi1EE"
        for name, fn in (("functions", lambda: ncu_funcs.main(csvp, sass, kp)),
                         ("lines", lambda: sass_lines.main(csvp, sass, kp, 40))):
            buf = io.StringIO()
            with redirect_stdout(buf):
                fn()
            open(os.path.join(PROF, f"{tag}_dock_{name}.txt"), "w").write(buf.getvalue())
    print("wrote", sorted(f for f in os.listdir(PROF) if f.startswith(tag) or f.startswith("ncu_")))


if __name__ == "__main__":
    main(sys.argv[1])
