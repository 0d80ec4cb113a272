cd $GRAFT_REPO_ROOT
O=gpurun_out/ft6d_pp_r02.jsonl; : > $O
for pp in 1 2 1 2; do DV_PP=$pp timeout 300 python tools/probe_ft6d_dirs.py | sed "s/^{/{\"pp\": $pp, /" >> $O; done
DV_PP=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -k "ft6d or fuzz" -q -x -p no:cacheprovider --timeout 300 > gpurun_out/ft6d_pp2_tests.log 2>&1
tail -3 gpurun_out/ft6d_pp2_tests.log
