#!/bin/bash
# One GPU profiling pass (run under gpurun from the repo root):
#   1. the default bench line (no profiler)             -> gpurun_out/bench_$TAG.json
#   2. ncu launch list of a short bench run              -> gpurun_out/launches_$TAG.csv
#   3. DRAM traffic of the first launch of each dock kernel (C2) -> gpurun_out/traffic_$TAG.csv
#   4. ncu --set full of one sweep and one flex launch (profile_dock) -> gpurun_out/prof_dock_$TAG.ncu-rep
# Each ncu step runs only if the same command exited 0 without ncu first.
TAG=${1:-r1}
NLIG=${2:-20000}
mkdir -p gpurun_out
set -o pipefail
timeout 900 python bench.py --json-out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1 || { echo "bench failed"; tail -20 gpurun_out/bench_$TAG.log; exit 1; }
tail -1 gpurun_out/bench_$TAG.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_short_$TAG.log 2>&1 || { echo "short bench failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/ncu_launch_$TAG.log 2>&1 || echo "launch list failed"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:"vs_(start|sweep|flex|polish|finish)_kernel" -c 5 --csv \
    --log-file gpurun_out/traffic_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_traffic_$TAG.log 2>&1 || echo "traffic failed"
timeout 300 python tools/profile_dock.py --ligands $NLIG > gpurun_out/profile_dock_$TAG.log 2>&1 || { echo "profile_dock failed"; exit 1; }
cat gpurun_out/profile_dock_$TAG.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"vs_(start|sweep|flex|polish)_kernel" -s 160 -c 4 \
    -f -o gpurun_out/prof_dock_$TAG python tools/profile_dock.py --ligands $NLIG \
    > gpurun_out/ncu_full_$TAG.log 2>&1 || echo "full capture failed"
tail -3 gpurun_out/ncu_full_$TAG.log
