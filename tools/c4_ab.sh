#!/bin/bash
# Same-box A/B of the C4 bench line (flexible ligands) between the in-tree
# library ("new") and variants/lib_<name>.so builds (tools/build_variants.py)
for v in ${1:-new}; do
  if [ $v = new ]; then unset VSCREEN_GPU_LIB; else export VSCREEN_GPU_LIB=variants/lib_$v.so; fi
  python bench.py --config c4 --no-cpu --no-e2e --steps 3 --warmup 3 --json-out gpurun_out/c4_$v.json > /dev/null 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/c4_$v.json').read().strip().splitlines()[-1])
print('$v', d['value'], {k: v.get('ms') for k, v in d['roofline']['per_kernel'].items()})"
done
