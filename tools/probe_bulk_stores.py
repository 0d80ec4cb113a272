"""TMA bulk stores (k_pack_bulk: gather into shared memory, one cp.async.bulk shared->global per
CTA chunk, SASS UBLKCP.G.S) vs per-thread STG.256 (k_run_copy) for the dense-destination packs,
selected by the environment of this process (DV_BULK=0/1). Back-to-back device time per call (spin
head start) and a bit-exact check of every wire against the device verifier (dvt_verify):
  C2 token step (6.55 MB, 25,600 runs of 256 B) -> pinned host (fused) and -> HBM;
  C2 prompt layer (163.8 MB, 640 runs of 256 KB) -> pinned host (fused) and -> HBM.
  DV_BULK=1 python tools/probe_bulk_stores.py [--ncu]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
NCU = "--ncu" in sys.argv
k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
c = dv.cache(k, v)
seed = 11
dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=seed)
ctx = dv.dv_create(0)
st = torch.cuda.current_stream()
host = torch.empty(90_000_000, dtype=torch.int16, pin_memory=True)
dbuf = torch.empty(90_000_000, dtype=torch.int16, device="cuda")
for shape, nl, npos in (("token step 6.55 MB", 40, 1), ("prompt layer 163.8 MB", 1, 1000)):
    nbytes = 2 * nl * B * H * npos * D * 2
    for dst, buf in (("pinned host", host), ("HBM", dbuf)):
        ep = dv.endpoint_of(buf)
        reps = 2 if NCU else (10 if nbytes > 50e6 else 200)
        pos = [P]

        def call():
            q = pos[0]
            dv.dv_scatter(ctx, c, (0, nl, 0, B, q, q + npos) if npos == 1 else (0, nl, 0, B, 0, npos), ep, 0,
                          xfer=dv.DV_XFER_FUSED)
            pos[0] = P + (pos[0] - P + 1) % 900
        for _ in range(2 if NCU else 3):
            call()
        torch.cuda.synchronize()
        row = {"shape": shape, "dst": dst, "bytes": nbytes, "bulk": os.environ.get("DV_BULK", "0")}
        if not NCU:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dv.dvt_spin(int(min(reps * nbytes / 30e3, 60e6)) + 2_000_000, 1)
            a.record(st)
            for _ in range(reps):
                call()
            b.record(st)
            torch.cuda.synchronize()
            us = a.elapsed_time(b) / reps * 1e3
            row.update(us=round(us, 2), gbs=round(nbytes / us / 1e3, 2))
        # parity of the last wire
        q = P + (pos[0] - P - 1) % 900
        reg = dv.region(0, nl, 0, B, q, q + 1) if npos == 1 else dv.region(0, nl, 0, B, 0, npos)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        dv.dvt_verify(c, cnt.data_ptr(), seed=seed, reg=reg, wire_ptr=buf.data_ptr())
        torch.cuda.synchronize()
        row["mismatches"] = int(cnt.item())
        print(json.dumps(row), flush=True)
        assert row["mismatches"] == 0
ctx.close()
