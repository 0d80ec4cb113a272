mkdir -p gpurun_out
TAG=r01c bash tools/gpu_round.sh > gpurun_out/round_r01c.log 2>&1
timeout 900 python tools/bench_configs.py > gpurun_out/configs_r01c.jsonl 2> gpurun_out/configs_r01c.err
tail -3 gpurun_out/configs_r01c.err
python tools/probe_latency.py > gpurun_out/latency_r01c.jsonl 2>&1
ls gpurun_out
