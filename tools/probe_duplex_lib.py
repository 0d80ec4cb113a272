"""The e2e ceiling on THIS box through the library's own copy-engine path: per step a 6.55 MB
H2D (dv_fetch, staged) on one stream and a 6.55 MB D2H (dv_flush, staged) on another, independent
(no dependency between the directions), then the same with the e2e dependency (step t's D2H after
step t's H2D), next to bench.py's e2e loop on the same box. GB/s per direction."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2403_01876_b200 as dv  # noqa: E402

AFF = bench._bind_gpu_local_cpus(0)
N = bench.STEP_BYTES
R = 64
ctx = dv.dv_create(0)
hsrc = torch.empty(R * N // 2, dtype=torch.int16, pin_memory=True)
hdst = torch.empty(R * N // 2, dtype=torch.int16, pin_memory=True)
d1 = torch.empty(R * N // 2, dtype=torch.int16, device="cuda")
d2 = torch.empty(R * N // 2, dtype=torch.int16, device="cuda")
hs_ep, hd_ep = dv.endpoint_of(hsrc), dv.endpoint_of(hdst)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
K = 200


def run(mode):
    evs = [torch.cuda.Event() for _ in range(R)]

    def one(i):
        j = i % R
        dv.dv_fetch(ctx, hs_ep, j * N, d1.data_ptr() + j * N, N, xfer=dv.DV_XFER_STAGED, stream=s_in.cuda_stream)
        if mode == "chained":
            evs[j].record(s_in)
            s_out.wait_event(evs[j])
        src = d1 if mode == "chained" else d2
        dv.dv_flush(ctx, src.data_ptr() + j * N, N, hd_ep, j * N, xfer=dv.DV_XFER_STAGED, stream=s_out.cuda_stream)
    for i in range(10):
        one(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s_out)
    s_in.wait_event(a)
    for i in range(K):
        one(i)
    s_out.wait_stream(s_in)
    b.record(s_out)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / K
    return {"mode": mode, "us_per_step": round(us, 1), "gbs_per_dir": round(N / us / 1e3, 2), "cpu_affinity": AFF}


for rep in range(2):
    for m in ("independent", "chained"):
        print(json.dumps(dict(run(m), rep=rep)), flush=True)
