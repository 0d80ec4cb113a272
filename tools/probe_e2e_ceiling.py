"""Ceiling of the bench's e2e loop: 6.55 MB H2D on one stream and 6.55 MB D2H on another, per
step, (a) independent, (b) with the e2e dependency (D2H of step t after H2D of step t), (c) (b)
plus a small HBM kernel between them, as dv_gather(staged) -> dv_scatter(decoupled) does."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

# pinned buffers on the GPU's NUMA node, as bench.py's e2e loop has them (first touch after binding)
AFFINITY = bench._bind_gpu_local_cpus(0)

N = 6_553_600
K = 300
hsrc = torch.empty(64 * N // 2, dtype=torch.int16, pin_memory=True)
hdst = torch.empty(64 * N // 2, dtype=torch.int16, pin_memory=True)
d1 = torch.empty(64 * N // 2, dtype=torch.int16, device="cuda")
d2 = torch.empty(64 * N // 2, dtype=torch.int16, device="cuda")
s_in, s_out, s_k = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def sl(t, i):
    j = i % 64
    return t[j * N // 2:(j + 1) * N // 2]


def run(mode):
    def one(i):
        with torch.cuda.stream(s_in):
            sl(d1, i).copy_(sl(hsrc, i), non_blocking=True)
        if mode != "independent":
            e = torch.cuda.Event()
            e.record(s_in)
            if mode == "kernel":
                s_k.wait_event(e)
                with torch.cuda.stream(s_k):
                    sl(d2, i).copy_(sl(d1, i))
                e = torch.cuda.Event()
                e.record(s_k)
            s_out.wait_event(e)
        with torch.cuda.stream(s_out):
            sl(hdst, i).copy_(sl(d2 if mode == "kernel" else d1, i), non_blocking=True)
    for i in range(10):
        one(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s_out)
    s_in.wait_stream(s_out)
    for i in range(K):
        one(i)
    s_out.wait_stream(s_in)
    b.record(s_out)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / K
    return {"mode": mode, "us_per_step": us, "gbs_per_dir": N / us / 1e3}


if __name__ == "__main__" and len(sys.argv) == 1:
    for m in ("independent", "chained", "kernel"):
        print(json.dumps(dict(run(m), cpu_affinity=AFFINITY)))


def trace(mode="kernel", n=60):
    """Per-step event stamps (ms since the first): when each H2D, kernel and D2H ended."""
    ev = {k: [torch.cuda.Event(enable_timing=True) for _ in range(n)] for k in ("h", "k", "d")}
    t0 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(s_in)
    s_out.wait_stream(s_in)
    s_k.wait_stream(s_in)
    for i in range(n):
        with torch.cuda.stream(s_in):
            sl(d1, i).copy_(sl(hsrc, i), non_blocking=True)
        ev["h"][i].record(s_in)
        src = d1
        if mode == "kernel":
            s_k.wait_event(ev["h"][i])
            with torch.cuda.stream(s_k):
                sl(d2, i).copy_(sl(d1, i))
            ev["k"][i].record(s_k)
            s_out.wait_event(ev["k"][i])
            src = d2
        else:
            s_out.wait_event(ev["h"][i])
        with torch.cuda.stream(s_out):
            sl(hdst, i).copy_(sl(src, i), non_blocking=True)
        ev["d"][i].record(s_out)
    torch.cuda.synchronize()
    rows = []
    for i in range(n):
        rows.append({k: round(t0.elapsed_time(ev[k][i]) * 1e3, 1) for k in ("h", "k", "d") if mode == "kernel" or k != "k"})
    return rows


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "trace":
    for m in ("chained", "kernel"):
        r = trace(m)
        print(m, json.dumps(r[20:30]))
