#!/bin/bash
# N-GPU bench lines (one process per GPU over NCCL) for N in $1 (default "2"),
# then the C2 reference arm under torchrun (rank 0 runs, the others exit).
mkdir -p gpurun_out
for n in ${1:-2}; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + n)) bench.py --gpus $n --steps 3 --warmup 3 --no-cpu \
      > gpurun_out/bench_n$n.log 2>&1; echo "n=$n rc=$?"; grep '^{' gpurun_out/bench_n$n.log | tail -1 | cut -c1-300
done
