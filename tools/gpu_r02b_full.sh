#!/bin/bash
# Round-2 (session b) refresh at HEAD on one B200: GPU parity suite + smoke, then every committed
# measurement (tools/gpu_round_full.sh with TAG=r02b), then the N = 2 peer suite with both ranks on
# this GPU (full shapes) -- the multi-GPU code path the driver's N-GPU run takes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02b.log 2>&1; echo "pytest_rc=$?"
tail -2 gpurun_out/pytest_gpu_r02b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02b.log 2>&1; echo "smoke_rc=$?"
TAG=r02b bash tools/gpu_round_full.sh > gpurun_out/full_r02b.log 2>&1; echo "full_rc=$?"
DV_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 3 --no-extras --no-cpu-baseline --dist-backend gloo > gpurun_out/bench_r02b_n2_one_gpu_full.json 2> gpurun_out/bench_r02b_n2_one_gpu_full.err; echo "n2_rc=$?"
head -c 400 gpurun_out/bench_r02b.json
