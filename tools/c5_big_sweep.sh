#!/bin/bash
# C5 rescoring: the largest-footprint size class capped at VSCREEN_RESCORE_BIG
# blocks per SM (the others get the remaining 8 - big), swept over 1..4
for b in 1 2 3 4; do VSCREEN_RESCORE_BIG=$b python bench.py --config c5 --no-cpu --no-e2e --steps 5 --warmup 3 --json-out gpurun_out/c5b$b.json > /dev/null 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c5b$b.json').read().strip().splitlines()[-1]); print('big=$b', round(d['value']), d['ms_per_step'])"; done
