#!/bin/bash
# e2e A/B of the vs_dock_host pipeline shapes (tools/e2e_breakdown.py)
for cfg in "0.3|0" "0.25,0.5,0.75|1" "0.2,0.6|0" "0.35|0" "0.15,0.6|0"; do  # split|concurrent
  split=${cfg%|*}; conc=${cfg#*|}
  echo "== split $split concurrent $conc"
  VSCREEN_PIPE_SPLIT=$split VSCREEN_PIPE_CONCURRENT=$conc VSCREEN_UPLOAD_TIMING=1 timeout 300 \
    python tools/e2e_breakdown.py 2>&1 | grep -E "dock_host|pipeline" | tail -2
done
