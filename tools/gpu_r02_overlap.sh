cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_r02.py -k concurrent_compute -q -p no:cacheprovider --timeout 200 > gpurun_out/ovl_test.log 2>&1
timeout 600 python tools/bench_overlap.py > gpurun_out/ovl_r02a.jsonl 2> gpurun_out/ovl_r02a.err
timeout 600 python tools/bench_overlap.py --xfer fused >> gpurun_out/ovl_r02a.jsonl 2>> gpurun_out/ovl_r02a.err
timeout 600 python tools/bench_overlap.py --pairs 24 >> gpurun_out/ovl_r02a.jsonl 2>> gpurun_out/ovl_r02a.err
