#!/bin/bash
# Round-2 (session b) refresh at HEAD on one B200: GPU parity suite + smoke, then every committed
# measurement (tools/gpu_round_full.sh with TAG=r02b), then the N = 2 peer suite with both ranks on
# this GPU (full shapes) -- the multi-GPU code path the driver's N-GPU run takes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG:-r02b}.log 2>&1; echo "pytest_rc=$?"
tail -2 gpurun_out/pytest_gpu_${TAG:-r02b}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG:-r02b}.log 2>&1; echo "smoke_rc=$?"
TAG=${TAG:-r02b} bash tools/gpu_round_full.sh > gpurun_out/full_${TAG:-r02b}.log 2>&1; echo "full_rc=$?"
DV_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 3 --no-extras --no-cpu-baseline --dist-backend gloo > gpurun_out/bench_${TAG:-r02b}_n2_one_gpu_full.json 2> gpurun_out/bench_${TAG:-r02b}_n2_one_gpu_full.err; echo "n2_rc=$?"
head -c 400 gpurun_out/bench_${TAG:-r02b}.json
# session-c additions: SM partitions and the fused producer (latency, idle and loaded)
timeout 400 python tools/probe_green_ctx.py > gpurun_out/green_${TAG:-r02b}.jsonl 2>&1; echo "green_rc=$?"
GREEN_SMS=16 timeout 400 python tools/probe_green_ctx.py > gpurun_out/green16_${TAG:-r02b}.jsonl 2>&1
timeout 300 python tools/probe_fused_latency.py > gpurun_out/fused_${TAG:-r02b}.jsonl 2>&1; echo "fused_rc=$?"
LOADED=1 timeout 300 python tools/probe_fused_latency.py >> gpurun_out/fused_${TAG:-r02b}.jsonl 2>&1
