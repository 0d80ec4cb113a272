#!/bin/bash
# The peer workloads at N = 2, 4, 8 ranks, all on the ONE GPU of this box (DV_BENCH_SAME_DEVICE=1,
# gloo plumbing, CUDA IPC between the processes): functional full-shape runs of the multi-rank
# code paths with their parity checks. The ranks share one HBM, so the GB/s are not NVLink numbers.
export DV_BENCH_SAME_DEVICE=1
for w in c5 c3; do
  for n in 2 4 8; do
    port=$((29500 + RANDOM % 1000))
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $port bench.py --workload $w --gpus $n --steps 20 --warmup 3 --dist-backend gloo 2>/dev/null \
      | grep '^{'
  done
done
