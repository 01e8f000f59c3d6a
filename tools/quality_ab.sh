#!/bin/bash
# Docking quality (tools/quality_vs_reference.py, cached reference arm) and
# dock throughput (tools/profile_dock.py) of library variants on one box:
#   bash tools/quality_ab.sh "new c31i24 ..." [n_ligands]
VARIANTS=${1:-"new"}
N=${2:-384}
for v in $VARIANTS; do
  if [ $v = new ]; then unset VSCREEN_GPU_LIB; else export VSCREEN_GPU_LIB=variants/lib_$v.so; fi
  q=$(timeout 600 python tools/quality_vs_reference.py $N --grid 2>&1 | tail -1)
  t=$(timeout 300 python tools/profile_dock.py --ligands 60000 2>&1 | tail -1 | cut -c1-60)
  echo "$v | $t | $(echo $q | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["mean_ours"],3), round(d["frac_ours_ge_ref"],3), round(d["mean_ref"],3))' 2>/dev/null || echo $q)"
done
