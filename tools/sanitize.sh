# compute-sanitizer runs over the hot path (one GPU): smoke() under memcheck/racecheck/synccheck,
# and memcheck over the flag/publish, FT6D (every PK) and decoupled parity tests.
mkdir -p gpurun_out/sanitizer
CS="compute-sanitizer --print-limit 20"
for tool in memcheck racecheck synccheck; do
  timeout 600 $CS --tool $tool python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer/${TAG}_smoke_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer/${TAG}_smoke_$tool.txt
done
for pk in 4 16; do
  DV_PK=$pk timeout 900 $CS --tool memcheck python -m pytest -q tests/test_gpu_parity.py -k "ft6d or FT6D or decoupled or flag or poller or transpose" > gpurun_out/sanitizer/${TAG}_memcheck_tests_pk$pk.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer/${TAG}_memcheck_tests_pk$pk.txt
done
tail -n 3 gpurun_out/sanitizer/*.txt
