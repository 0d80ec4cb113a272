"""Grid-size sweep (dv_config.max_ctas) for the large HBM copies: the C2 KV5D prompt-layer pack
(163.8 MB) and a 16-layer C3 direct remap (4.72 GB), median of 7 x 20 launches, cold-ish (the
source layer cycles)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
c = dv.cache(k, v)
nb = 2 * B * H * P * D * 2
dbuf = torch.empty(nb // 2, dtype=torch.int16, device="cuda")
ep = dv.endpoint_of(dbuf)
st = torch.cuda.current_stream()


def med(fn, n=20, reps=7):
    out = []
    for _ in range(reps):
        for _ in range(2):
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


for ctas in [int(x) for x in os.environ.get("CTAS", "592,740,888,1000,1036,1184,1332,1480").split(",")]:
    ctx = dv.dv_create(0, max_ctas=ctas)
    lay = [0]

    def prm():
        lay[0] = (lay[0] + 7) % L
        dv.dv_scatter(ctx, c, dv.region(lay[0], lay[0] + 1, 0, B, 0, P), ep, 0)
    us = med(prm)
    print(json.dumps({"max_ctas": ctas, "op": "C2 prompt layer pack (163.8 MB)", "us": round(us, 2),
                      "frac_2R": round(2 * nb / us / 1e3 / 6534.8, 4)}), flush=True)
    ctx.close()
