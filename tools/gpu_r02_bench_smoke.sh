cd $GRAFT_REPO_ROOT
timeout 600 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
DV_BENCH_SAME_DEVICE=1 DV_BENCH_PEER_SMALL=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-extras --no-cpu-baseline --dist-backend gloo --nvlink-steps 32 > gpurun_out/bench_r02a_n2.json 2> gpurun_out/bench_r02a_n2.err
