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
# the newer paths: 16-CTA cluster publish, half-slab staging, tile transposes to host, in-kernel consumer
timeout 900 $CS --tool memcheck python -m pytest -q tests/test_gpu_parity.py -k "half_slab or auto_falls or enomem or in_kernel_consumer or release_scope or every_packet_group" > gpurun_out/sanitizer/${TAG}_memcheck_new_paths.txt 2>&1
echo "rc=$?" >> gpurun_out/sanitizer/${TAG}_memcheck_new_paths.txt
timeout 900 $CS --tool racecheck python -m pytest -q tests/test_gpu_parity.py -k "in_kernel_consumer or flag_orders or every_packet_group" > gpurun_out/sanitizer/${TAG}_racecheck_new_paths.txt 2>&1
echo "rc=$?" >> gpurun_out/sanitizer/${TAG}_racecheck_new_paths.txt
tail -n 3 gpurun_out/sanitizer/*.txt
