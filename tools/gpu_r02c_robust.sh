#!/bin/bash
# Session-c robustness pass (one B200): differential fuzz at 10x scale (default forms) and at 5x
# with the TMA-row FT6D transposes on, compute-sanitizer memcheck / racecheck over the SM-partition
# tests (cluster-publish fallback on an 8-SM green context).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
DV_FUZZ_SCALE=10 timeout 1500 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/fuzz_r02c_10x.log 2>&1; echo "fuzz10 rc=$?"; tail -1 gpurun_out/fuzz_r02c_10x.log
DV_TMA=1 DV_FUZZ_SCALE=5 timeout 1500 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/fuzz_r02c_tma_5x.log 2>&1; echo "fuzz_tma rc=$?"; tail -1 gpurun_out/fuzz_r02c_tma_5x.log
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --print-limit 20 --tool $tool python -m pytest -q -p no:cacheprovider tests/test_gpu_green.py > gpurun_out/sanitizer/r02c_green_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer/r02c_green_$tool.txt
  tail -3 gpurun_out/sanitizer/r02c_green_$tool.txt
done
