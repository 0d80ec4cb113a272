"""Trace of bench.py's e2e loop (C2 token step: dv_gather from pinned host -> cache on an input
stream, then dv_scatter cache -> pinned-host log): per-step completion stamps of the input side
(H2D + unpack) and of the output side, for xfer = staged (D2H on the caller's stream, so an event
after it marks the DMA's end) and decoupled (event marks the pack's end only)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
STEP = 2 * L * B * H * D * 2
RING = 64
k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
cache = dv.cache(k, v)
ctx = dv.dv_create(0)
log = torch.empty(RING * STEP // 2, dtype=torch.int16, pin_memory=True)
fl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
ep = dv.endpoint_of(log, fl)
delta = torch.empty(RING * STEP // 2, dtype=torch.int16, pin_memory=True)
dep = dv.endpoint_of(delta)
main = torch.cuda.current_stream()
s_ins = [torch.cuda.Stream(), torch.cuda.Stream()]
n_in = int(os.environ.get("N_IN", "2"))


def loop(xfer, n=120, seq0=0):
    t0 = torch.cuda.Event(enable_timing=True)
    ein = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    eout = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    torch.cuda.synchronize()
    dv.dvt_spin(3_000_000, 1, stream=main.cuda_stream)
    t0.record(main)
    for s in s_ins:
        s.wait_event(t0)
    for t in range(1, n + 1):
        q = P + t
        s_in = s_ins[t % n_in]
        dv.dv_gather(ctx, dep, ((t - 1) % RING) * STEP, cache, dv.region(0, L, 0, B, q, q + 1), stream=s_in)
        ein[t - 1].record(s_in)
        main.wait_event(ein[t - 1])
        dv.dv_scatter(ctx, cache, dv.region(0, L, 0, B, q, q + 1), ep, (t % RING) * STEP, flag_slot=0,
                      seq=seq0 + t, xfer=xfer, stream=main)
        eout[t - 1].record(main)
    dv.dv_wait(ctx, ep, 0, seq0 + n, stream=main)
    end = torch.cuda.Event(enable_timing=True)
    end.record(main)
    torch.cuda.synchronize()
    us = lambda e: round(t0.elapsed_time(e) * 1e3, 1)  # noqa: E731
    rows = [(us(ein[i]), us(eout[i])) for i in range(n)]
    total = us(end)
    return {"xfer": xfer, "n_in": n_in, "us_per_step": round(total / n, 1), "gbs_per_dir": round(STEP * n / total / 1e3, 2),
            "steady_in_end_deltas": [round(rows[i][0] - rows[i - 1][0], 1) for i in range(min(60, n - 10), min(70, n))],
            "steady_out_end_deltas": [round(rows[i][1] - rows[i - 1][1], 1) for i in range(min(60, n - 10), min(70, n))],
            "out_minus_in_lag": [round(rows[i][1] - rows[i][0], 1) for i in range(min(60, n - 10), min(70, n))]}


def loop3(xfer, n=120, seq0=0, slots=8):
    """dv_fetch (H2D into a device wire slot) on s_h2d, dv_gather (unpack from that slot) on s_unp,
    dv_scatter on main: the H2Ds run back to back, independent of the unpack kernels."""
    s_h2d, s_unp = torch.cuda.Stream(), torch.cuda.Stream()
    wire = torch.empty(slots * STEP // 2, dtype=torch.int16, device="cuda")
    wep = dv.endpoint_of(wire)
    t0 = torch.cuda.Event(enable_timing=True)
    eh = [torch.cuda.Event() for _ in range(n)]
    eu = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    torch.cuda.synchronize()
    dv.dvt_spin(3_000_000, 1, stream=main.cuda_stream)
    t0.record(main)
    s_h2d.wait_event(t0)
    s_unp.wait_event(t0)
    for t in range(1, n + 1):
        q = P + t
        j = (t - 1) % slots
        if t > slots:
            s_h2d.wait_event(eu[t - 1 - slots])          # slot j free: its unpack is done
        lag = int(os.environ.get("LAG", "0"))
        if lag and t > lag:                               # bounded run-ahead: step t's H2D after
            dv.dv_wait(ctx, ep, 0, seq0 + t - lag, stream=s_h2d)   # step t-lag's D2H landed
        dv.dv_fetch(ctx, dep, ((t - 1) % RING) * STEP, wire.data_ptr() + j * STEP, STEP, stream=s_h2d)
        eh[t - 1].record(s_h2d)
        s_unp.wait_event(eh[t - 1])
        dv.dv_gather(ctx, wep, j * STEP, cache, dv.region(0, L, 0, B, q, q + 1), stream=s_unp)
        eu[t - 1].record(s_unp)
        main.wait_event(eu[t - 1])
        dv.dv_scatter(ctx, cache, dv.region(0, L, 0, B, q, q + 1), ep, (t % RING) * STEP, flag_slot=0,
                      seq=seq0 + t, xfer=xfer, stream=main)
    dv.dv_wait(ctx, ep, 0, seq0 + n, stream=main)
    end = torch.cuda.Event(enable_timing=True)
    end.record(main)
    torch.cuda.synchronize()
    total = t0.elapsed_time(end) * 1e3
    return {"xfer": xfer, "form": "fetch|gather|scatter on 3 streams", "us_per_step": round(total / n, 1),
            "gbs_per_dir": round(STEP * n / total / 1e3, 2)}


if os.environ.get("FORM") == "3":
    for name, xf in (("staged", dv.DV_XFER_STAGED), ("decoupled", dv.DV_XFER_DECOUPLED)):
        loop3(xf, 20, 40_000)
        for n in (120, 500):
            r = loop3(xf, n, 50_000 + n * 10 + (0 if name == "staged" else 100_000))
            r["xfer"] = name
            r["n"] = n
            r["lag"] = os.environ.get("LAG", "0")
            print(json.dumps(r), flush=True)
    sys.exit(0)

for name, xf in (("staged", dv.DV_XFER_STAGED), ("decoupled", dv.DV_XFER_DECOUPLED)):
    loop(xf, 20, 10_000)
    r = loop(xf, 120, 20_000 if name == "staged" else 30_000)
    r["xfer"] = name
    print(json.dumps(r), flush=True)
