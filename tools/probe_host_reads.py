"""Zero-copy reads from pinned host (dv_gather of a wire chunk into the cache, FUSED): per-thread
32-byte loads (k_run_copy) vs bulk asynchronous copies into shared memory (k_unpack_bulk, TMA
`cp.async.bulk`), selected by the environment of this process (DV_RDBULK=0/1, DV_RDCH bytes per
bulk read, DV_RDST reads in flight per CTA). Prints one JSON line per chunk size:
device time per call back to back (spin head start hides the host enqueue), the latency of one
call on an idle stream (event-bracketed), and a bit-exact check of the unpacked region (packed back
on the device and compared with the host wire).

  DV_RDBULK=1 DV_RDCH=8192 DV_RDST=4 python tools/probe_host_reads.py [--ncu]

--ncu: two calls per size only (for `ncu --metrics pcie__read_bytes.sum,...`)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, S = 40, 40, 128, 8, 2048
NCU = "--ncu" in sys.argv
k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
c = dv.cache(k, v)
ctx = dv.dv_create(0, host_ctas=int(os.environ.get("DV_HOST_CTAS", "16")))
host = torch.randint(-32768, 32767, (90_000_000,), dtype=torch.int16).pin_memory()
ep = dv.endpoint_of(host)
st = torch.cuda.current_stream()
form = {"rdbulk": os.environ.get("DV_RDBULK", "0"), "rdch": os.environ.get("DV_RDCH", "8192"),
        "rdst": os.environ.get("DV_RDST", "4"), "host_ctas": os.environ.get("DV_HOST_CTAS", "16")}

SHAPES = (("token-layer 160 KiB", 1, 1), ("8 layers x 4 pos 1.3 MB", 8, 4), ("token step 6.55 MB", 40, 1),
          ("9 layers x 16 pos 11.8 MB", 9, 16), ("prompt layer 163.8 MB", 1, 1000))
for name, nl, npos in SHAPES:
    reg = dv.region(0, nl, 0, B, 100, 100 + npos)
    nbytes = 2 * nl * B * H * npos * D * 2
    row = {"shape": name, "bytes": nbytes, **form}
    reps = 2 if NCU else (20 if nbytes > 50e6 else 200)
    for _ in range(2 if NCU else 3):
        dv.dv_gather(ctx, ep, 0, c, reg, xfer=dv.DV_XFER_FUSED)
    torch.cuda.synchronize()
    if not NCU:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dv.dvt_spin(int(min(reps * nbytes / 40e3, 50e6)) + 2_000_000, 1)
        a.record(st)
        for _ in range(reps):
            dv.dv_gather(ctx, ep, 0, c, reg, xfer=dv.DV_XFER_FUSED)
        b.record(st)
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / reps * 1e3
        row["back_to_back_us"] = round(us, 2)
        row["gbs"] = round(nbytes / us / 1e3, 2)
        one = []
        for _ in range(30 if nbytes < 50e6 else 3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            dv.dv_gather(ctx, ep, 0, c, reg, xfer=dv.DV_XFER_FUSED)
            b.record(st)
            torch.cuda.synchronize()
            one.append(a.elapsed_time(b) * 1e3)
        one.sort()
        row["single_call_us_p50"] = round(one[len(one) // 2], 2)
    # parity: pack the region back into device memory and compare with the host wire
    back = torch.empty(nbytes // 2, dtype=torch.int16, device="cuda")
    dv.dv_scatter(ctx, c, reg, dv.endpoint_of(back), 0)
    torch.cuda.synchronize()
    row["bit_exact"] = bool(torch.equal(back.cpu(), host[:nbytes // 2]))
    print(json.dumps(row), flush=True)
    assert row["bit_exact"], row
ctx.close()
