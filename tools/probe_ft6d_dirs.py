"""FT6D register transpose in both directions (C2 prompt layer, 163.8 MB, median of 7 x 20, layer
cycled): pack FT6D -> wire (DIR 0), unpack wire -> FT6D (DIR 1), remap FT6D -> KV5D (DIR 0),
remap KV5D -> FT6D (DIR 1); KV5D pack/unpack beside them. frac = 2R / us / 6534.8 GB/s."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 12, 40, 128, 8, 1000, 2048
k6 = torch.empty((L, B, H, D // 8, S, 8), dtype=torch.int16, device="cuda")
v6 = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
k5 = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
v5 = torch.empty_like(k5)
c6, c5 = dv.cache(k6, v6), dv.cache(k5, v5)
nb = 2 * B * H * P * D * 2
wire = torch.empty(nb // 2, dtype=torch.int16, device="cuda")
ep = dv.endpoint_of(wire)
ctx = dv.dv_create(0)
st = torch.cuda.current_stream()


def med(fn, n=20, reps=7):
    out = []
    for _ in range(reps):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(n):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / n * 1e3)
    return sorted(out)[reps // 2]


lay = [0]


def nxt():
    lay[0] = (lay[0] + 5) % (L - 1)
    return lay[0]


ops = {
    "pack_ft6d": lambda: dv.dv_scatter(ctx, c6, dv.region(nxt(), lay[0] + 1, 0, B, 0, P), ep, 0),
    "unpack_ft6d": lambda: dv.dv_gather(ctx, ep, 0, c6, dv.region(nxt(), lay[0] + 1, 0, B, 0, P)),
    "remap_ft6d_to_kv5d": lambda: dv.dv_remap(ctx, c6, c5, dv.region(nxt(), lay[0] + 1, 0, B, 0, P)),
    "remap_kv5d_to_ft6d": lambda: dv.dv_remap(ctx, c5, c6, dv.region(nxt(), lay[0] + 1, 0, B, 0, P)),
    "pack_kv5d": lambda: dv.dv_scatter(ctx, c5, dv.region(nxt(), lay[0] + 1, 0, B, 0, P), ep, 0),
    "unpack_kv5d": lambda: dv.dv_gather(ctx, ep, 0, c5, dv.region(nxt(), lay[0] + 1, 0, B, 0, P)),
}
for name, fn in ops.items():
    us = med(fn)
    print(json.dumps({"op": name, "pk_cap": os.environ.get("DV_PK", "16"), "us": round(us, 2),
                      "frac_2R": round(2 * nb / us / 1e3 / 6534.8, 4)}), flush=True)
