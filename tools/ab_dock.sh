#!/bin/bash
# Same-box A/B of dock throughput (tools/profile_dock.py, C2 prefix) between
# variants/lib_<name>.so builds and the in-tree library ("new"), after the
# GPU test suite:  bash tools/ab_dock.sh "head new" [ligands] [rounds]
VARIANTS=${1:-"head new"}
NLIG=${2:-60000}
ROUNDS=${3:-2}
mkdir -p gpurun_out
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab_pytest.log
fi
for r in $(seq $ROUNDS); do
 for v in $VARIANTS; do
  if [ $v = new ]; then unset VSCREEN_GPU_LIB; else export VSCREEN_GPU_LIB=variants/lib_$v.so; fi
  echo -n "$v: "; timeout 300 python tools/profile_dock.py --ligands $NLIG 2>&1 | tail -1 | cut -c1-200
 done
done
