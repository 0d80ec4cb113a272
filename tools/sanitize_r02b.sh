# compute-sanitizer over the TMA-row FT6D transpose (tests/test_gpu_tma.py): memcheck, racecheck
# (shared-memory hazards between the threads' and the TMA engine's accesses), synccheck.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
T=${TAG:-r02b}
CS="compute-sanitizer --print-limit 20"
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool python -m pytest -q -p no:cacheprovider tests/test_gpu_tma.py -k "not full_size" > gpurun_out/sanitizer/${T}_tma_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer/${T}_tma_$tool.txt
done
timeout 1200 $CS --tool memcheck python -m pytest -q -p no:cacheprovider tests/test_gpu_tma.py -k "full_size" > gpurun_out/sanitizer/${T}_tma_memcheck_full_size.txt 2>&1
echo "rc=$?" >> gpurun_out/sanitizer/${T}_tma_memcheck_full_size.txt
for f in gpurun_out/sanitizer/${T}_*.txt; do echo "== $f"; tail -n 4 $f; done
