#!/bin/bash
# ncu --set full of one launch of each dock kernel (second dock, restart 10)
# of tools/profile_dock.py --ligands $2, after the same command ran clean.
TAG=${1:-r2}
NLIG=${2:-20000}
mkdir -p gpurun_out
timeout 300 python tools/profile_dock.py --ligands $NLIG > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:"vs_(start|sweep|flex|polish)_kernel" -s 160 -c 4 \
    -f -o gpurun_out/prof_$TAG python tools/profile_dock.py --ligands $NLIG \
    > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full_$TAG.log
