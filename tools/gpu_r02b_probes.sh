#!/bin/bash
# Round-2 probes (one B200): TMA tensor-map FT6D transpose forms vs the register transpose, and the
# token-step pack's fixed cost vs marginal rate under launch-shape variants.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/probes_r02b.jsonl
: > $O
timeout 120 ./tools/tma_ft6d_probe 1000 >> $O 2>&1
timeout 120 ./tools/tma_ft6d_probe 64 >> $O 2>&1
timeout 300 python tools/probe_token_floor.py >> $O 2>&1
for u in 1 2 8; do DV_U=$u timeout 300 python tools/probe_token_floor.py >> $O 2>&1; done
DV_VEC=16 timeout 300 python tools/probe_token_floor.py >> $O 2>&1
cat $O
