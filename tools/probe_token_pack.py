"""Device time (host enqueue hidden behind a spin head start) of a C2 token step (25,600 runs of 256 B, 6.55 MB) packed into an HBM buffer: time per launch
(median of 7 x 200), for the DV_U / DV_SMALL variants given in the environment."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P = 40, 40, 128, 8, 1000
S = int(os.environ.get("PROBE_S", "2048"))   # max_seq of the cache (TLB reach experiments)
k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
c = dv.cache(k, v)
ctx = dv.dv_create(0)
nb = 2 * L * B * H * D * 2
buf = torch.empty(nb * 8 // 2, dtype=torch.int16, device="cuda")
ep = dv.endpoint_of(buf)
st = torch.cuda.current_stream()
cnt = [0]


def one():
    cnt[0] += 1
    q = (P + cnt[0] % 1000) % S
    dv.dv_scatter(ctx, c, dv.region(0, L, 0, B, q, q + 1), ep, (cnt[0] % 8) * nb)


def t1(n=200):
    for _ in range(3):
        one()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dv.dvt_spin(4_000_000, 1)   # 4 ms head start: the launches queue up, timing sees device time
    a.record(st)
    for _ in range(n):
        one()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


us = sorted(t1() for _ in range(7))[3]
print(f"S={S} U={os.environ.get('DV_U', 'auto')} SMALL={os.environ.get('DV_SMALL', 'default')} "
      f"us={us:.2f} frac_2R={2 * nb / us / 1e3 / 6534.8:.3f}")
