"""C2 token step (one position, all 40 layers, 6.55 MB) packed into HBM, FT6D keys (16-byte K
runs) vs KV5D, back to back behind a spin head start: device us per launch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
v = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
k5 = torch.empty_like(v)
k6 = torch.empty((L, B, H, D // 8, S, 8), dtype=torch.int16, device="cuda")
ctx = dv.dv_create(0)
nb = 2 * L * B * H * D * 2
buf = torch.empty(nb * 8 // 2, dtype=torch.int16, device="cuda")
ep = dv.endpoint_of(buf)
st = torch.cuda.current_stream()
for name, c in (("kv5d", dv.cache(k5, v)), ("ft6d", dv.cache(k6, v))):
    cnt = [0]

    def one():
        cnt[0] += 1
        q = P + cnt[0] % 1000
        dv.dv_scatter(ctx, c, (0, L, 0, B, q, q + 1), ep, (cnt[0] % 8) * nb)
    res = []
    for _ in range(7):
        for _ in range(3):
            one()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dv.dvt_spin(4_000_000, 1)
        a.record(st)
        for _ in range(200):
            one()
        b.record(st)
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / 200 * 1e3)
    print(name, "token pack us", round(sorted(res)[3], 2))
