#!/bin/bash
# Multi-GPU measurement session (for a box with >= 2 B200s; one process per GPU, NCCL plumbing):
# the link probe across all pairs, then the peer workloads at N = 2, 4, 8 -- dvstream's CUDA-IPC peer
# stores and the NCCL send/recv baseline side by side -- and the headline C2 workload's weak scaling.
# Outputs: gpurun_out/nvlink_${TAG}.jsonl (one JSON line per run).
T=${TAG:-r02}
G=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/nvlink_$T.jsonl
mkdir -p gpurun_out
: > $OUT
timeout 900 python tools/probe_links.py >> $OUT 2> gpurun_out/nvlink_links_$T.err
for n in 2 4 8; do
  [ $n -gt $G ] && break
  for w in c5 c3 c4; do
    for base in none nccl; do
      [ $w = c4 ] && [ $base = nccl ] && continue
      port=$((29500 + RANDOM % 1000))
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $port bench.py --workload $w --gpus $n --steps 20 --warmup 3 --peer-baseline $base \
        2>> gpurun_out/nvlink_$T.err | grep '^{' >> $OUT
    done
  done
  port=$((29500 + RANDOM % 1000))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $n --steps 200 --warmup 10 --no-extras --no-cpu-baseline \
    2>> gpurun_out/nvlink_$T.err | grep '^{' >> $OUT
done
wc -l $OUT
