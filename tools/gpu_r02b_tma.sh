#!/bin/bash
# TMA-row FT6D transpose: parity (its own tests + the FT6D suites with DV_TMA=1), then the C2
# prompt-layer forms (tools/probe_ft6d_dirs.py) with the register form vs the TMA form, TS and split sweeps.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/tma_r02b
timeout 600 python -m pytest tests/test_gpu_tma.py -x -q > $O.pytest.log 2>&1; echo "tma tests rc=$?"; tail -3 $O.pytest.log
DV_TMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -x -q -k "ft6d or FT6D or fuzz" > $O.pytest_env.log 2>&1; echo "ft6d suites DV_TMA=1 rc=$?"; tail -3 $O.pytest_env.log
: > $O.dirs.jsonl
for rep in 1 2; do
  DV_TMA=0 timeout 300 python tools/probe_ft6d_dirs.py | sed 's/^{/{"tma": 0, /' >> $O.dirs.jsonl
  DV_TMA=1 timeout 300 python tools/probe_ft6d_dirs.py | sed 's/^{/{"tma": 1, /' >> $O.dirs.jsonl
done
for ts in 32 64; do for sp in 0.8 1.0 1.3; do
  DV_TMA=1 DV_TMA_TS=$ts DV_TMA_TSPLIT=$sp timeout 300 python tools/probe_ft6d_dirs.py | sed "s/^{/{\"tma\": 1, \"ts\": $ts, \"split\": $sp, /" >> $O.dirs.jsonl
done; done
cat $O.dirs.jsonl
