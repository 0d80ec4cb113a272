"""Where the C2 token-step pack's 4 us go: device time per launch (back to back, PDL, launches queued
behind a spin head start so host enqueue is hidden) of

  * the token step at 1/2/4/8/16/40 layers (25,600 * L/40 runs of 256 B, 512 KiB apart): the
    slope of time vs bytes is the kernel's marginal rate, the intercept its fixed cost per launch;
  * a near-contiguous copy of the same 6.55 MB (positions [0,320) of one layer and request: 80 runs
    of 80 KiB) and torch's cudaMemcpyAsync D2D of 6.55 MB from a >L2 ring;
  * the smallest launch (one position of one head: 2 runs of 256 B).

One JSON line per case. Launch-shape knobs come from the environment (DV_U, DV_VEC, ...)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P = 40, 40, 128, 8, 1000
S = 2048
k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
c = dv.cache(k, v)
ctx = dv.dv_create(0)
step_b = 2 * L * B * H * D * 2
buf = torch.empty(step_b * 8 // 2, dtype=torch.int16, device="cuda")
ep = dv.endpoint_of(buf)
st = torch.cuda.current_stream()
HBM = 6544.0


def timed(fn, n=200, reps=7):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    out = []
    for r in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dv.dvt_spin(4_000_000, 1)
        a.record(st)
        for i in range(n):
            fn(r * n + i)
        b.record(st)
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / n * 1e3)
    return sorted(out)[reps // 2]


def token(nl):
    def f(i):
        q = (P + i % 1000) % S
        dv.dv_scatter(ctx, c, dv.region(0, nl, 0, B, q, q + 1), ep, (i % 8) * step_b)
    return f


tag = {x: os.environ[x] for x in ("DV_U", "DV_VEC", "DV_PDL", "DV_SMALL") if x in os.environ}
rows = []
for nl in (1, 2, 4, 8, 16, 40):
    us = timed(token(nl))
    nb = step_b * nl // L
    rows.append((nb, us))
    print(json.dumps({"case": "token_step", "layers": nl, "bytes": nb, "us": round(us, 3),
                      "frac_2R": round(2 * nb / us / 1e3 / HBM, 3), "frac_R": round(nb / us / 1e3 / HBM, 3), **tag}))
# least-squares line through (bytes, us): marginal rate and fixed cost
n = len(rows)
mx = sum(r[0] for r in rows) / n
my = sum(r[1] for r in rows) / n
slope = sum((r[0] - mx) * (r[1] - my) for r in rows) / sum((r[0] - mx) ** 2 for r in rows)
icpt = my - slope * mx
print(json.dumps({"case": "token_step_fit", "fixed_us": round(icpt, 3), "marginal_gbs_read": round(1e-3 / slope, 1),
                  "marginal_frac_R": round(1e-3 / slope / HBM, 3), **tag}))


def contiguous(i):
    layer = i % L
    bb = (i // L) % B
    dv.dv_scatter(ctx, c, dv.region(layer, layer + 1, bb, bb + 1, 0, 320), ep, (i % 8) * step_b)


us = timed(contiguous)
print(json.dumps({"case": "near_contiguous_6.55MB", "runs": 80, "us": round(us, 3),
                  "frac_2R": round(2 * step_b / us / 1e3 / HBM, 3), **tag}))

ring = torch.empty(64 * step_b // 2, dtype=torch.int16, device="cuda")   # 419 MB > L2
dstb = torch.empty(step_b // 2, dtype=torch.int16, device="cuda")


def memcpy(i):
    o = (i % 64) * (step_b // 2)
    dstb.copy_(ring[o:o + step_b // 2])


us = timed(memcpy)
print(json.dumps({"case": "torch_d2d_6.55MB", "us": round(us, 3), "frac_2R": round(2 * step_b / us / 1e3 / HBM, 3)}))


def tiny(i):
    q = (P + i % 1000) % S
    dv.dv_scatter(ctx, c, dv.region(0, 1, 0, 1, q, q + 1, 0, 1), ep, (i % 8) * 1024)


us = timed(tiny)
print(json.dumps({"case": "tiny_512B", "us": round(us, 3), **tag}))
