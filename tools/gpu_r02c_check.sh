#!/bin/bash
# Session-c check at HEAD (one B200): GPU suite, smoke, headline bench (with the fused-producer and
# loaded-latency extras), C5 workload, the N = 2 peer suite with both ranks on this GPU.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02c.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_gpu_r02c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02c.log 2>&1; echo "smoke_rc=$?"
timeout 900 python bench.py > gpurun_out/bench_r02c2.json 2> gpurun_out/bench_r02c2.err; echo "bench_rc=$?"
timeout 600 python bench.py --workload c5 --steps 300 > gpurun_out/c5_r02c2.json 2> gpurun_out/c5_r02c2.err; echo "c5_rc=$?"
DV_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 3 --no-extras --no-cpu-baseline --dist-backend gloo > gpurun_out/bench_r02c_n2_full.json 2> gpurun_out/bench_r02c_n2_full.err; echo "n2_rc=$?"
