"""Per-layer token latency with the stream-out FUSED INTO THE PRODUCER (device plans, include/dv.h
dv_dplan_*) against the separate stream-out kernel (dv_scatter behind the producer with PDL), C2
layer of 160 KiB (40 heads, 8 requests, one position), to pinned host and into HBM.

Both arms use the same vectorised producer (dvt_fill_rows). Stamps (%globaltimer): the producer's
first CTA start (t_start), its last CTA's stores done (t_end), the flag release (library trace /
the plan's trace). Reported per arm: start -> flag (the whole "write the layer's K/V and make it
visible at the destination") and, for the separate arm, end -> flag (the usual writer-end metric).
LOADED=1: a bf16 GEMM loop on a low-priority stream, producer + stream-out on a high-priority one;
PART=k: the producer and the stream-out on a k-SM partition (dv_partition_create), the GEMM on the
rest."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
LAYER = 2 * B * H * D * 2
k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
cache = dv.cache(k, v)
ctx = dv.dv_create(0)
SEED = 20240305
N = 1040
LOADED = os.environ.get("LOADED") == "1"
lo_pr, hi_pr = torch.cuda.Stream.priority_range()
PART = int(os.environ.get("PART", "0"))   # PART=k: producer + stream-out on a k-SM partition, GEMM on the rest
if PART:
    part = dv.dv_partition_create(0, PART, hi_pr)
    st, gst = torch.cuda.ExternalStream(part.streaming), torch.cuda.ExternalStream(part.compute)
else:
    st = torch.cuda.Stream(priority=hi_pr)
    gst = torch.cuda.Stream(priority=lo_pr)
sp = st.cuda_stream
if LOADED:
    ga = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    gb = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)


def pct(x):
    x = sorted(x[L:])
    return round(x[len(x) // 2], 3), round(x[int(len(x) * 0.99)], 3)


def run(dst_host):
    dev = "cpu" if dst_host else "cuda"
    log = torch.empty(L * LAYER // 2, dtype=torch.int16, device=dev, pin_memory=dst_host)
    fl = torch.zeros(L, dtype=torch.int64, device=dev, pin_memory=dst_host)
    ep = dv.endpoint_of(log, fl)
    plans = [dv.dv_dplan_scatter(ctx, cache, dv.region(l, l + 1, 0, B, P, P + 1), ep, l * LAYER, 0, flag_slot=l,
                                 seq=1, max_step=S - P - 1) for l in range(L)]
    out = {}
    for arm in ("fused", "separate"):
        t0 = torch.full((N,), 2 ** 63 - 1, dtype=torch.int64, device="cuda")
        te = torch.zeros(N, dtype=torch.int64, device="cuda")
        ts = torch.zeros((N, 4), dtype=torch.int64, device="cuda")
        ts[:, 1:3] = 2 ** 63 - 1
        seq = [10 ** 6]

        def one(i):
            layer, step = i % L, i // L
            q = P + step
            reg = dv.region(layer, layer + 1, 0, B, q, q + 1)
            if arm == "fused":
                pl = plans[layer]
                pl.trace = ts[i].data_ptr()
                dv.dvt_fill_rows(cache, SEED, reg, pl, step, t_start_ptr=t0[i].data_ptr(), t_end_ptr=te[i].data_ptr(),
                                 stream=sp)
            else:
                dv.dvt_fill_rows(cache, SEED, reg, None, 0, t_start_ptr=t0[i].data_ptr(), t_end_ptr=te[i].data_ptr(),
                                 stream=sp)
                dv.dvt_trace(ctx, ts[i].data_ptr())
                seq[0] += 1
                dv.dv_scatter(ctx, cache, reg, ep, layer * LAYER, flag_slot=layer, seq=seq[0], xfer=dv.DV_XFER_FUSED,
                              stream=sp)
        for i in range(2 * L):   # warm-up
            one(i % L)
        dv.dvt_trace(ctx, 0)
        torch.cuda.synchronize()
        if LOADED:
            with torch.cuda.stream(gst):
                for _ in range(60):
                    torch.matmul(ga, gb)
        dv.dvt_spin(20_000_000, 1, stream=sp)
        for i in range(N):
            one(i)
        dv.dvt_trace(ctx, 0)
        torch.cuda.synchronize()
        a = pct(((ts[:, 0] - t0).double() / 1e3).tolist())
        r = {"start_to_flag_p50_us": a[0], "start_to_flag_p99_us": a[1]}
        if arm == "separate":
            b = pct(((ts[:, 0] - te).double() / 1e3).tolist())
            r.update({"writer_end_to_flag_p50_us": b[0], "writer_end_to_flag_p99_us": b[1]})
        c = pct(((te - t0).double() / 1e3).tolist())
        r.update({"producer_p50_us": c[0]})
        out[arm] = r
    return out


for rep in range(2):
    for host in (True, False):
        print(json.dumps({"rep": rep, "dst": "host" if host else "hbm", "loaded": LOADED, "sm_partition": PART or None,
                          **run(host)}), flush=True)
