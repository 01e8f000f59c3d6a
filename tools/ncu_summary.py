"""Summarise one profiling round (tools/profile_round.sh TAG) into profiles/:

  profiles/<TAG>_launches.json     per-kernel share of the bench launch list
  profiles/<TAG>_dock_ncu.json     key metrics + stall breakdown of each profiled dock kernel
  profiles/<TAG>_<kernel>_functions.txt per-subroutine samples (tools/ncu_funcs.py)
  profiles/<TAG>_<kernel>_lines.txt    hottest source lines (tools/sass_lines.py)
  profiles/ncu_dock_traffic.json   DRAM bytes per C2 launch of each dock kernel (bench
                                   roofline.traffic)

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
        name = r[ik].split("(")[0].replace("void ", "").split("<")[0]
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
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = {}
    for r in rows[1:]:
        name = r[ik].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        d = per.setdefault(name, {})
        if r[im] not in d:  # first launch of each kernel
            d[r[im]] = float(r[iv].replace(",", ""))
    kernels = {}
    for name, v in per.items():
        rd, wr = v.get("dram__bytes_read.sum", 0.0), v.get("dram__bytes_write.sum", 0.0)
        kernels[name] = {"dram_bytes_read": rd, "dram_bytes_write": wr,
                         "dram_bytes_per_launch": rd + wr, "kernel_ns": v.get("gpu__time_duration.sum")}
    return {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum on the first C2 "
                      f"launch of each dock kernel (bench.py, 100k ligands), gpurun_out/traffic_{tag}.csv",
            "kernels": kernels}


def dock_report(tag):
    rep = os.path.join(OUT, f"prof_dock_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    out = {"source": f"ncu --set full --clock-control none --import-source on, tools/profile_dock.py "
                     f"--ligands 20000 (C2 library prefix), gpurun_out/prof_dock_{tag}.ncu-rep",
           "kernels": {}}
    for row in rows[2:]:
        d = dict(zip(rows[0], row))
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "").split("<")[0]
        name = name.split("::")[-1]
        k = {"metrics": {m: d.get(m) for m in METRICS}, "stalls_per_issue": {}}
        for key, v in d.items():
            if key.startswith("smsp__average_warps_issue_stalled_") and key.endswith(
                    "_per_issue_active.ratio"):
                try:
                    if float(v) >= 0.05:
                        k["stalls_per_issue"][key[len("smsp__average_warps_issue_stalled_"):-len(
                            "_per_issue_active.ratio")]] = round(float(v), 3)
                except ValueError:
                    pass
        out["kernels"][name] = k
    return out, rep


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    t = None
    if os.path.exists(os.path.join(OUT, f"launches_{tag}.csv")):  # (a full-capture-only round skips these)
        json.dump(launches(tag), open(os.path.join(PROF, f"{tag}_launches.json"), "w"), indent=1)
        t = traffic(tag)
        json.dump(t, open(os.path.join(PROF, "ncu_dock_traffic.json"), "w"), indent=1)
    summ, rep = dock_report(tag)
    if t:
        summ["dram_traffic_c2_first_launch"] = t["kernels"]
    json.dump(summ, open(os.path.join(PROF, f"{tag}_dock_ncu.json"), "w"), indent=1)
    import ncu_funcs
    import sass_lines
    with tempfile.TemporaryDirectory() as td:
        lib = os.path.join(ROOT, "paper_2304_09953_b200", "libvscreen_gpu.so")
        subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=td, capture_output=True)
        sass = os.path.join(td, "dock.sass")
        with open(sass, "w") as f:
            subprocess.run(["nvdisasm", "-g", os.path.join(td, "vs_dock.sm_100a.cubin")], stdout=f)
        for kname in summ["kernels"]:
            src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                                  "sass", "--kernel-name", f"regex:{kname}"],
                                 capture_output=True, text=True).stdout
            csvp = os.path.join(td, f"{kname}.csv")
            open(csvp, "w").write(src)
            # the profiled instantiation (e.g. vs_flex_kernel<(int)1, (int)8>) as its
            # mangled prefix
            import re
            m = re.search(kname + r"<([^>]*)>", src.splitlines()[0] if src else "")
            targs = re.findall(r"\(int\)(\d+)", m.group(1)) if m else ["1"]
            kp = f"_ZN2vs{len(kname)}{kname}I" + "".join(f"Li{a}E" for a in targs) + "EE"
            for part, fn in (("functions", lambda: ncu_funcs.main(csvp, sass, kp)),
                             ("lines", lambda: sass_lines.main(csvp, sass, kp, 40))):
                buf = io.StringIO()
                with redirect_stdout(buf):
                    fn()
                open(os.path.join(PROF, f"{tag}_{kname}_{part}.txt"), "w").write(buf.getvalue())
    print("wrote", sorted(f for f in os.listdir(PROF) if f.startswith(tag) or f.startswith("ncu_")))


if __name__ == "__main__":
    main(sys.argv[1])
