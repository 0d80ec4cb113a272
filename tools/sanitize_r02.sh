# compute-sanitizer over the round-2 paths (one GPU): smoke() (prompt per layer + credited ring) under
# memcheck / racecheck / synccheck; memcheck over the round-2 GPU tests (rings + credits, DV_EBUSY,
# ordering fixes, bulk reads in subprocesses excluded, overlap, engine); racecheck over the engine
# and ring tests.
mkdir -p gpurun_out/sanitizer
T=${TAG:-r02}
CS="compute-sanitizer --print-limit 20"
for tool in memcheck racecheck synccheck; do
  timeout 600 $CS --tool $tool python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer/${T}_smoke_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer/${T}_smoke_$tool.txt
done
# (not the engine: the sanitizer serialises kernels, and a resident engine never yields)
timeout 1200 $CS --tool memcheck python -m pytest -q -p no:cacheprovider tests/test_gpu_r02.py -k "not bulk_host_reads and not captured_publishes and not engine" > gpurun_out/sanitizer/${T}_memcheck_r02_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/sanitizer/${T}_memcheck_r02_tests.txt
DV_RDBULK=1 timeout 600 $CS --tool memcheck python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "scatter_gather_random_shapes and True" > gpurun_out/sanitizer/${T}_memcheck_bulk_reads.txt 2>&1
echo "rc=$?" >> gpurun_out/sanitizer/${T}_memcheck_bulk_reads.txt
timeout 900 $CS --tool racecheck python -m pytest -q -p no:cacheprovider tests/test_gpu_r02.py -k "engine_per_layer or ring_credits or ebusy" > gpurun_out/sanitizer/${T}_racecheck_r02.txt 2>&1
echo "rc=$?" >> gpurun_out/sanitizer/${T}_racecheck_r02.txt
for f in gpurun_out/sanitizer/${T}_*.txt; do echo "== $f"; tail -n 3 $f; done
