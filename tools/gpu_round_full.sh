#!/bin/bash
# Refresh every committed measurement at HEAD in one GPU session (one B200):
#   bench line + ncu launch list + ncu --set full of the headline pack kernel + DRAM/PCIe counters
#   (tools/gpu_round.sh), the per-config suite, latency stamps, the FT6D direction probe, the
#   HBM-kernel ncu capture and the link probe. Outputs land in gpurun_out/ with the tag ${TAG}.
T=${TAG:-r01g}
mkdir -p gpurun_out
TAG=$T bash tools/gpu_round.sh > gpurun_out/round_$T.log 2>&1
timeout 900 python tools/bench_configs.py > gpurun_out/configs_$T.jsonl 2> gpurun_out/configs_$T.err
tail -3 gpurun_out/configs_$T.err
timeout 300 python tools/probe_latency.py > gpurun_out/latency_$T.jsonl 2>&1
timeout 300 python tools/probe_ft6d_dirs.py > gpurun_out/ft6d_dirs_$T.jsonl 2>&1
timeout 600 python tools/probe_links.py > gpurun_out/links_$T.jsonl 2>&1
timeout 900 ncu --set full --metrics pcie__read_bytes.sum,pcie__write_bytes.sum --clock-control none \
  -k regex:"k_run_copy|k_packet_transpose|k_transpose_run|k_copy_cluster" -o gpurun_out/hbm_$T -f \
  python tools/ncu_hbm_kernels.py > gpurun_out/ncu_hbm_$T.log 2>&1
timeout 300 python bench.py --workload c5 --steps 300 > gpurun_out/c5_$T.json 2>&1
timeout 300 python bench.py --workload c3 --steps 3 > gpurun_out/c3_$T.json 2>&1
timeout 300 python bench.py --workload c4 > gpurun_out/c4_$T.json 2>&1
timeout 300 python tools/probe_latency_loaded.py > gpurun_out/latency_loaded_$T.jsonl 2>&1
DST=host timeout 300 python tools/probe_latency_loaded.py >> gpurun_out/latency_loaded_$T.jsonl 2>&1
ls gpurun_out
