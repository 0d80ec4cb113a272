#!/bin/bash
# Round-2 re-entry check at HEAD (one B200): the GPU parity suite, smoke(), and the headline bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02b.log 2>&1; echo "pytest_rc=$?"
tail -3 gpurun_out/pytest_gpu_r02b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02b.log 2>&1; echo "smoke_rc=$?"
tail -2 gpurun_out/smoke_r02b.log
timeout 600 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo "bench_rc=$?"
head -c 600 gpurun_out/bench_r02b.json
