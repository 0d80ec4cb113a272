"""ncu driver: one C2 layer (160 KiB) streamed to pinned host by (a) the producer then the separate
stream-out kernel and (b) the producer fused with the stream-out through a device plan; three of
each (the last measured). Run under: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum,pcie__write_bytes.sum -k regex:"k_fill_rows|k_run_copy" python tools/ncu_fused_producer.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
LAYER = 2 * B * H * D * 2
k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
cache = dv.cache(k, v)
ctx = dv.dv_create(0)
log = torch.empty(LAYER // 2, dtype=torch.int16, pin_memory=True)
fl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
ep = dv.endpoint_of(log, fl)
reg = dv.region(7, 8, 0, B, P, P + 1)
plan = dv.dv_dplan_scatter(ctx, cache, reg, ep, 0, 0, flag_slot=0, seq=1, max_step=0)
for i in range(3):
    dv.dvt_fill_rows(cache, 5, reg, None, 0)
    dv.dv_scatter(ctx, cache, reg, ep, 0, flag_slot=0, seq=10 + i, xfer=dv.DV_XFER_FUSED)
torch.cuda.synchronize()
plan.seq = 100
for i in range(3):
    dv.dvt_fill_rows(cache, 5, reg, plan, 0)
torch.cuda.synchronize()
dv.dv_dplan_free(ctx, plan)
print("ok")
