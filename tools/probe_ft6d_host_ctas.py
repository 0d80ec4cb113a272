import torch, sys
sys.path.insert(0, '.')
import paper_2403_01876_b200 as dv
L, H, D, B, P, S = 4, 40, 128, 8, 1000, 2048
k6 = torch.empty((L, B, H, D // 8, S, 8), dtype=torch.int16, device="cuda")
v = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
k5 = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
nb = 2 * B * H * P * D * 2
hp = torch.empty(nb // 2, dtype=torch.int16, pin_memory=True)
st = torch.cuda.current_stream()
for hc in (16,):
    ctx = dv.dv_create(0, host_ctas=hc)
    for name, c in (("ft6d", dv.cache(k6, v)), ("kv5d", dv.cache(k5, v))):
        for P2 in (1000, 64):
            nbb = 2 * B * H * P2 * D * 2
            f = lambda: dv.dv_scatter(ctx, c, (1, 2, 0, B, 0, P2), dv.endpoint_of(hp), 0, xfer=dv.DV_XFER_FUSED)
            f(); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(5): f()
            b.record(st); torch.cuda.synchronize()
            us = a.elapsed_time(b) / 5 * 1e3
            print(f"host_ctas={hc} {name} positions={P2} {nbb/us/1e3:.1f} GB/s")
    ctx.close()
