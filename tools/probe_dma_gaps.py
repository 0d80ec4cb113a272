"""Where do the per-step gaps of a decoupled staged token step come from? Back-to-back 6.55 MB
D2H copies on one stream, with (a) nothing else, (b) a flag stream-op after each, (c) an event
hand-off from a second stream before each, (d) both, (e) two DMA streams alternating."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

N = 6_553_600
K = 300
ctx = dv.dv_create(0)
src = torch.empty(64 * N // 2, dtype=torch.int16, device="cuda")
dst = torch.empty(64 * N // 2, dtype=torch.int16, pin_memory=True)
fl = torch.zeros(4, dtype=torch.int64, pin_memory=True)
ep = dv.endpoint_of(dst, fl)
s0, s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def run(mode):
    seq = [0]

    def one(i):
        j = i % 64
        s = s0
        if mode == "alt":
            s = s0 if i % 2 == 0 else s2
        if mode in ("event", "both"):
            e = torch.cuda.Event()
            e.record(s1)
            s.wait_event(e)
        s.wait_stream(s) if False else None
        with torch.cuda.stream(s):
            dst[j * N // 2:(j + 1) * N // 2].copy_(src[j * N // 2:(j + 1) * N // 2], non_blocking=True)
        if mode in ("flag", "both"):
            seq[0] += 1
            dv.dv_signal(ctx, ep, 0, seq[0], stream=s.cuda_stream)
    for i in range(10):
        one(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s0)
    s2.wait_stream(s0)
    for i in range(K):
        one(i)
    s0.wait_stream(s2)
    b.record(s0)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / K
    return {"mode": mode, "us": us, "gbs": N / us / 1e3}


for m in ("plain", "flag", "event", "both", "alt"):
    print(json.dumps(run(m)))
