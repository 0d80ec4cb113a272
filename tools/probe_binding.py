"""Host cost per call of the Python binding: dv_scatter of one C2 token-layer (fused, flag in HBM)
and one C5 dv_stream_out_direct, through the CPython fast path and through ctypes (DV_NO_FAST=1 in
a second process). Calls are queued behind a spin so the host time is the binding + library."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

ctx = dv.dv_create(0)
k = torch.empty((40, 8, 40, 2048, 128), dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
c = dv.cache(k, v)
buf = torch.empty(1 << 20, dtype=torch.int16, device="cuda")
fl = torch.zeros(1, dtype=torch.int64, device="cuda")
ep = dv.endpoint_of(buf, fl)
k2 = torch.empty((8, 16, 72, 2048, 128), dtype=torch.int16, device="cuda")
v2 = torch.empty_like(k2)
own, rep = dv.cache(k2, v2), dv.cache(torch.empty_like(k2), torch.empty_like(v2))
setup = dv.Setup([0, 8], [0, 16], 2048)
dst_arr, sig_arr = dv.cache_array([rep]), dv.endpoint_array([ep])
sp = torch.cuda.current_stream().cuda_stream
out = {"fast": dv.fast() is not None}
for name, fn in (
        ("dv_scatter_us", lambda i: dv.dv_scatter(ctx, c, dv.region(i % 40, i % 40 + 1, 0, 8, 1000, 1001), ep, 0,
                                                  flag_slot=0, seq=i + 1, stream=sp)),
        ("dv_scatter_tuple_region_us", lambda i: dv.dv_scatter(ctx, c, (i % 40, i % 40 + 1, 0, 8, 1000, 1001), ep, 0,
                                                               flag_slot=0, seq=10 ** 5 + i, stream=sp)),
        ("dv_stream_out_direct_us", lambda i: dv.dv_stream_out_direct(
            ctx, own, dv.region(0, 8, 0, 16, 1000, 1001), setup, 0, 0, setup, dst_arr, sig_arr, seq=10 ** 6 + i,
            stream=sp))):
    for i in range(50):
        fn(i)
    torch.cuda.synchronize()
    n = 400   # well inside the launch queue, so no call blocks on a full queue
    dv.dvt_spin(n * 30_000, 1, stream=sp)
    t0 = time.perf_counter()
    for i in range(n):
        fn(100 + i)
    out[name] = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    best = out[name]
    for _ in range(4):   # best of 5 batches
        dv.dvt_spin(n * 30_000, 1, stream=sp)
        t0 = time.perf_counter()
        for i in range(n):
            fn(100 + i)
        best = min(best, (time.perf_counter() - t0) / n * 1e6)
        torch.cuda.synchronize()
    out[name] = best
print(json.dumps(out))
