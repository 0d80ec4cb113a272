"""Does the way the pinned host buffer was allocated change SM zero-copy read speed? Token-step
(40 layers x 1 position, 6.55 MB) and prompt-layer (163.8 MB) fused gathers from (a) torch.empty(
pin_memory=True), (b) tensor.pin_memory() of a pageable tensor, (c) dv_host_alloc (cudaHostAlloc
portable|mapped), (d) dv_host_alloc_near; back-to-back device time per call."""
import ctypes
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
ctx = dv.dv_create(0, host_ctas=int(os.environ.get("DV_HOST_CTAS", "16")))
st = torch.cuda.current_stream()
N = 90_000_000
bufs = {}
bufs["torch_empty_pinned"] = torch.empty(N, dtype=torch.int16, pin_memory=True)
bufs["pin_memory_copy"] = torch.zeros(N, dtype=torch.int16).pin_memory()
p = dv.dv_host_alloc(2 * N)
bufs["dv_host_alloc"] = p
p2 = dv.dv_host_alloc_near(0, 2 * N)
bufs["dv_host_alloc_near"] = p2[0] if isinstance(p2, tuple) else p2
for name, b in bufs.items():
    ep = dv.endpoint_of(b) if isinstance(b, torch.Tensor) else dv.endpoint(dv.DV_EP_HOST, b, 2 * N)
    for sname, nl, npos in (("token step 6.55 MB", 40, 1), ("prompt layer 163.8 MB", 1, 1000), ("token-layer 160 KiB", 1, 1)):
        reg = dv.region(0, nl, 0, B, 100, 100 + npos)
        nbytes = 2 * nl * B * H * npos * D * 2
        reps = 10 if nbytes > 50e6 else 100
        for _ in range(3):
            dv.dv_gather(ctx, ep, 0, c, reg, xfer=dv.DV_XFER_FUSED)
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dv.dvt_spin(int(min(reps * nbytes / 40e3, 50e6)) + 2_000_000, 1)
        a.record(st)
        for _ in range(reps):
            dv.dv_gather(ctx, ep, 0, c, reg, xfer=dv.DV_XFER_FUSED)
        e.record(st)
        torch.cuda.synchronize()
        us = a.elapsed_time(e) / reps * 1e3
        print(json.dumps({"alloc": name, "shape": sname, "us": round(us, 2), "gbs": round(nbytes / us / 1e3, 2),
                          "rdbulk": os.environ.get("DV_RDBULK", "0"), "host_ctas": os.environ.get("DV_HOST_CTAS", "16")}),
              flush=True)
