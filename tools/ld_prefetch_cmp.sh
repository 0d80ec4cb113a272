for n in 0 128 256; do
  DV_NVCC_EXTRA="-DDV_LD_PREFETCH=$n" python -m paper_2403_01876_b200.build -f > /dev/null 2>&1
  echo "== DV_LD_PREFETCH=$n"
  python tools/probe_small_reads.py | tail -2
  python tools/probe_token_pack.py
  python tools/bench_configs.py --only C4 2>/dev/null | grep -E "fused_zero_copy" | head -2 | cut -c1-160
  python tools/probe_ft6d_dirs.py | grep kv5d
done
