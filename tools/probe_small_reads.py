"""Small reads from pinned host (dv_gather of a wire chunk into the cache): copy engine (STAGED:
H2D DMA into staging + unpack kernel) vs SM zero-copy loads (FUSED), back to back, device time per
call (spin head start hides the host enqueue), for chunk sizes from one C2 token-layer (160 KiB)
to a C2 token step (6.55 MB)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, S = 40, 40, 128, 8, 2048
k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
c = dv.cache(k, v)
ctx = dv.dv_create(0)
host = torch.zeros(64 << 20, dtype=torch.int16, pin_memory=True)
ep = dv.endpoint_of(host)
st = torch.cuda.current_stream()

for nl, npos in ((1, 1), (1, 8), (4, 1), (8, 4), (40, 1)):
    reg = dv.region(0, nl, 0, B, 100, 100 + npos)
    nbytes = 2 * nl * B * H * npos * D * 2
    row = {"bytes": nbytes}
    for name, xf in (("staged", dv.DV_XFER_STAGED), ("fused", dv.DV_XFER_FUSED)):
        for _ in range(3):
            dv.dv_gather(ctx, ep, 0, c, reg, xfer=xf)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 200
        dv.dvt_spin(n * 40_000, 1)
        a.record(st)
        for _ in range(n):
            dv.dv_gather(ctx, ep, 0, c, reg, xfer=xf)
        b.record(st)
        torch.cuda.synchronize()
        row[name + "_us"] = round(a.elapsed_time(b) / n * 1e3, 2)
    print(json.dumps(row), flush=True)
