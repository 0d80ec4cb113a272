#!/bin/bash
# Swap in each library variant under variants/ and time the HBM-side shapes (probe_ft6d.py +
# the C3/C5 config subset). Restores the original library at the end.
cp paper_2403_01876_b200/libdvstream.so /tmp/orig.so
for v in variants/*.so; do
  cp $v paper_2403_01876_b200/libdvstream.so
  touch paper_2403_01876_b200/libdvstream.so
  echo "== $v"
  python tools/probe_ft6d.py
  python tools/bench_configs.py --only C3,C5 2>/dev/null | grep -E "16_layers_stream_out_direct|prompt_replica|token_step_per_stage" | cut -c1-200
done
cp /tmp/orig.so paper_2403_01876_b200/libdvstream.so
