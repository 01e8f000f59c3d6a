#!/bin/bash
# GPU test + bench pass (run under gpurun from the repo root):
#   gpurun_out/pytest_$TAG.log  -m gpu suite
#   gpurun_out/bench_$TAG.json  default C2 bench line (no profiler)
TAG=${1:-r2}
SKIP_TESTS=${SKIP_TESTS:-0}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
if [ "$SKIP_TESTS" != "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_$TAG.log 2>&1
  echo "pytest rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
fi
timeout 900 python bench.py ${BENCH_ARGS:-} --json-out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_$TAG.log
