#!/bin/bash
# Multi-GPU lines (one process per GPU over NCCL; the top-k gather is the
# C-ABI's vs_topk_allgather):  bash tools/scale_run.sh TAG "1 2 4" [config]
TAG=${1:-r2}
NS=${2:-"1 2 4"}
CFG=${3:-c3}
mkdir -p gpurun_out
for n in $NS; do
  if [ $n = 1 ]; then
    timeout 1200 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu \
      --json-out gpurun_out/bench_${TAG}_${CFG}_n1.json > gpurun_out/bench_${TAG}_${CFG}_n1.log 2>&1
  else
    NCCL_DEBUG=INFO timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --config $CFG --gpus $n \
      --steps 3 --warmup 3 --no-cpu --json-out gpurun_out/bench_${TAG}_${CFG}_n$n.json \
      > gpurun_out/bench_${TAG}_${CFG}_n$n.log 2>&1
  fi
  echo "n=$n rc=$?"
  python -c "
import json,sys
d=json.load(open('gpurun_out/bench_${TAG}_${CFG}_n$n.json'))
print(d['n_gpus'], d['value'], (d.get('e2e') or {}).get('value'), d['ms_per_step'], d.get('topk_check'))" 2>&1 | tail -1
done
grep -h "NVLS\|nranks" gpurun_out/bench_${TAG}_${CFG}_n*.log | head -4
