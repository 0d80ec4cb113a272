"""bench.py's e2e loop (C2 token step: dv_gather of step t's K/V from pinned host into the cache on
an input stream, then dv_stream_out of step t into the pinned-host ring on the main stream) under
different HOST submission orders and stream priorities -- does the order in which the H2D of step
t+1 and the D2H of step t reach the copy engines decide how well the two PCIe directions overlap?

  order 0: gather(t), stream_out(t)                       (bench.py today)
  order k: gather(t+k) enqueued before stream_out(t)      (input k steps ahead, bounded by the ring)
Prints GB/s per direction per variant (device time, 300 steps after 20 warm-up)."""
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
dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=5)
ctx = dv.dv_create(0)
log = torch.empty(RING * STEP // 2, dtype=torch.int16, pin_memory=True)
fl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
ep = dv.endpoint_of(log, fl)
ring = dv.endpoint_array([dv.endpoint_of(log, fl, n_slots=RING, slot_bytes=STEP)])
stage = dv.Setup([0, L], [0, B], S)
delta = torch.empty(RING * STEP // 2, dtype=torch.int16, pin_memory=True)
dep = dv.endpoint_of(delta)
seq = [0]


def pos(t):
    return P + (t - 1) % (S - P)


def run(order, prio_in, prio_main, xfer_in, n=300, warm=20):
    main = torch.cuda.Stream(priority=prio_main)
    s_in = torch.cuda.Stream(priority=prio_in)
    evs = {}

    def gather(t):
        q = pos(t)
        dv.dv_gather(ctx, dep, ((t - 1) % RING) * STEP, cache, dv.region(0, L, 0, B, q, q + 1), xfer=xfer_in,
                     stream=s_in.cuda_stream)
        e = torch.cuda.Event()
        e.record(s_in)
        evs[t] = e

    def out(t):
        q = pos(t)
        main.wait_event(evs.pop(t))
        seq[0] += 1
        dv.dv_stream_out(ctx, cache, (0, L, 0, B, q, q + 1), stage, 0, 0, stage, ring, seq=seq[0],
                         xfer=dv.DV_XFER_DECOUPLED, stream=main.cuda_stream)

    def loop(t0, m):
        for t in range(t0, t0 + order):
            gather(t)
        for t in range(t0, t0 + m):
            if t + order not in evs and order:
                gather(t + order)
            if not order:
                gather(t)
            out(t)
        for t in list(evs):   # drain look-ahead gathers that were not streamed out
            main.wait_event(evs.pop(t))
    torch.cuda.synchronize()
    loop(1, warm)
    dv.dv_wait(ctx, ep, 0, seq[0], stream=main.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    s_in.wait_event(a)
    loop(warm + 1 + order, n)
    dv.dv_wait(ctx, ep, 0, seq[0], stream=main.cuda_stream)
    b.record(main)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / n
    return {"order": order, "prio_in": prio_in, "prio_main": prio_main,
            "xfer_in": {dv.DV_XFER_STAGED: "staged", dv.DV_XFER_AUTO: "auto"}[xfer_in],
            "us_per_step": round(us, 1), "gbs_per_dir": round(STEP / us / 1e3, 2)}


lo, hi = torch.cuda.Stream.priority_range()  # (low, high) numbers: high priority is the lower number
for rep in range(2):
    for order in (0, 1, 2, 4):
        for pin, pmain in ((0, 0), (hi, 0), (0, hi)):
            print(json.dumps(run(order, pin, pmain, dv.DV_XFER_STAGED)), flush=True)
