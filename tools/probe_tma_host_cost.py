"""Host time per dv_scatter call of a C2 FT6D prompt layer with the register transpose and with the
TMA-row form (tensor-map encode + occupancy query per call), the GPU kept busy by a spin so the
host time is not hidden: is the TMA form host-bound back to back? (profiles/r02f_tma_host_cost.jsonl)"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_01876_b200 as dv
L, H, D, B, P, S = 4, 40, 128, 8, 1000, 2048
k6 = torch.empty((L, B, H, D // 8, S, 8), dtype=torch.int16, device="cuda")
v6 = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
c6 = dv.cache(k6, v6)
nb = 2 * B * H * P * D * 2
wire = torch.empty(nb // 2, dtype=torch.int16, device="cuda")
ep = dv.endpoint_of(wire)
ctx = dv.dv_create(0)
for tma in (0, 1):
    dv.dvt_tune("DV_TMA", tma)
    for _ in range(3):
        dv.dv_scatter(ctx, c6, dv.region(1, 2, 0, B, 0, P), ep, 0)
    torch.cuda.synchronize()
    dv.dvt_spin(50_000_000, 1)
    t0 = time.perf_counter()
    for _ in range(20):
        dv.dv_scatter(ctx, c6, dv.region(1, 2, 0, B, 0, P), ep, 0)
    host_us = (time.perf_counter() - t0) / 20 * 1e6
    torch.cuda.synchronize()
    print(json.dumps({"tma": tma, "host_us_per_call": round(host_us, 1)}))
