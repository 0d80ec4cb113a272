#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/probe_e2e_order.py > gpurun_out/e2e_order_r02b.jsonl 2>&1; echo "e2e_rc=$?"
: > gpurun_out/tma_r02b2.dirs.jsonl
for sp in 0.6 1.0 1.5; do
  DV_TMA=1 DV_TMA_TSPLIT=$sp timeout 300 python tools/probe_ft6d_dirs.py | sed "s/^{/{\"tma\": 1, \"split\": $sp, /" >> gpurun_out/tma_r02b2.dirs.jsonl
done
DV_TMA=0 timeout 300 python tools/probe_ft6d_dirs.py | sed "s/^{/{\"tma\": 0, /" >> gpurun_out/tma_r02b2.dirs.jsonl
cat gpurun_out/e2e_order_r02b.jsonl gpurun_out/tma_r02b2.dirs.jsonl
