#!/bin/bash
# Multi-GPU measurement session (for a box with >= 2 B200s; one process per GPU, NCCL plumbing):
#  1. the link probe across all pairs (one process driving every GPU);
#  2. at N = 2, 4, 8: the headline with the full "nvlink" suite in its JSON line (link peaks, C5 ring,
#     C3 disaggregation by SM stores / copy engine / into FT6D caches with both transposes, NCCL
#     baselines, put latency, C4 on every rank; every delivered word verified);
#  3. the standalone peer workloads and their NCCL baselines;
#  4. NVLink counters of the peer-put kernels on rank 0 (ncu on a 2-rank C5 run: nvltx / nvlrx bytes).
# Outputs: gpurun_out/nvlink_${TAG}.jsonl (one JSON line per run), gpurun_out/nvlink_ncu_${TAG}.csv.
T=${TAG:-r02}
G=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/nvlink_$T.jsonl
mkdir -p gpurun_out
: > $OUT
timeout 900 python tools/probe_links.py >> $OUT 2> gpurun_out/nvlink_links_$T.err
for n in 2 4 8; do
  [ $n -gt $G ] && break
  port=$((29500 + RANDOM % 1000))
  timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $n --steps 200 --warmup 10 --no-cpu-baseline \
    2>> gpurun_out/nvlink_$T.err | grep '^{' >> $OUT
  for w in c5 c3 c4; do
    for base in none nccl; do
      [ $w = c4 ] && [ $base = nccl ] && continue
      port=$((29500 + RANDOM % 1000))
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $port bench.py --workload $w --gpus $n --steps 20 --warmup 3 --peer-baseline $base \
        2>> gpurun_out/nvlink_$T.err | grep '^{' >> $OUT
    done
  done
done
if [ $G -ge 2 ]; then
  # ncu profiles one process; rank 1 runs unprofiled (its kernels are the receivers)
  port=$((29500 + RANDOM % 1000))
  (RANK=1 LOCAL_RANK=1 WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=$port timeout 900 python bench.py \
     --workload c5 --gpus 2 --steps 20 --warmup 3 > /dev/null 2>> gpurun_out/nvlink_$T.err &)
  RANK=0 LOCAL_RANK=0 WORLD_SIZE=2 MASTER_ADDR=127.0.0.1 MASTER_PORT=$port timeout 900 ncu --clock-control none \
    --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum \
    -k regex:"k_run_copy|k_copy_cluster" -c 60 --csv python bench.py --workload c5 --gpus 2 --steps 20 --warmup 3 \
    > gpurun_out/nvlink_ncu_$T.csv 2>> gpurun_out/nvlink_$T.err
fi
wc -l $OUT
