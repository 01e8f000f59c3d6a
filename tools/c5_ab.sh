#!/bin/bash
# Same-box A/B of the C5 bench line (rescoring-only) between the in-tree
# library ("new") and variants/lib_<name>.so builds (tools/build_variants.py)
for v in ${1:-new}; do
  if [ $v = new ]; then unset VSCREEN_GPU_LIB; else export VSCREEN_GPU_LIB=variants/lib_$v.so; fi
  python bench.py --config c5 --no-cpu --steps 5 --warmup 3 --json-out gpurun_out/c5_$v.json > /dev/null 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/c5_$v.json').read().strip().splitlines()[-1])
print('$v', round(d['value']), d['ms_per_step'], round(d['e2e']['value']))"
done
