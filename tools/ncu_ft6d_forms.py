"""ncu driver: the C2 FT6D prompt layer (163.8 MB) packed and unpacked once with the register
transpose and once with the TMA-row form (dvt_tune("DV_TMA")), two launches each (warm-up,
measured). Run under: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
-k regex:"k_transpose" python tools/ncu_ft6d_forms.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 3, 40, 128, 8, 1000, 2048
k6 = torch.empty((L, B, H, D // 8, S, 8), dtype=torch.int16, device="cuda")
v6 = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
c6 = dv.cache(k6, v6)
wire = torch.empty(2 * B * H * P * D, dtype=torch.int16, device="cuda")
ep = dv.endpoint_of(wire)
ctx = dv.dv_create(0)
for tma in (0, 1):
    dv.dvt_tune("DV_TMA", tma)
    for rep in range(2):
        dv.dv_scatter(ctx, c6, dv.region(rep, rep + 1, 0, B, 0, P), ep, 0)
    for rep in range(2):
        dv.dv_gather(ctx, ep, 0, c6, dv.region(rep, rep + 1, 0, B, 0, P))
    torch.cuda.synchronize()
dv.dvt_tune("DV_TMA", dv.TMA_DEFAULT)
print("ok")
