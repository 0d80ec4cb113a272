"""Link and peak probe: copy-engine and SM-store GB/s per GPU pair and for
all pairs at once, and pinned-host D2H/H2D GB/s per GPU and for every GPU at once, in ONE process
that sees every GPU (single-process P2P via dv_peer_enable). On a one-GPU box the peer rows are
the loopback (same-GPU) copies and the "all" rows equal the single ones.

  python tools/probe_links.py [--mib 256] > gpurun_out/links.jsonl

SM-store rows use dv_flush(DV_XFER_FUSED) (the library's run-copy kernel storing into the peer's
memory), copy-engine rows use cudaMemcpyAsync through torch."""
import argparse
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402


def timed(dev, fn, reps):
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream()
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    n = args.mib << 20
    G = torch.cuda.device_count()
    bufs = [torch.empty(n, dtype=torch.uint8, device=f"cuda:{g}") for g in range(G)]
    dsts = [torch.empty(n, dtype=torch.uint8, device=f"cuda:{g}") for g in range(G)]
    ctxs = [dv.dv_create(g) for g in range(G)]
    for a in range(G):
        for b in range(G):
            dv.dv_peer_enable(a, b)
    out = lambda **kw: print(json.dumps(kw), flush=True)  # noqa: E731
    out(probe="topology", gpus=G, names=[torch.cuda.get_device_name(g) for g in range(G)])

    # per pair: copy engine and SM stores, src GPU a -> dst GPU b (b == a: loopback in HBM)
    for a in range(G):
        for b in range(G):
            if G > 1 and a == b:
                continue
            ms = timed(a, lambda: dsts[b].copy_(bufs[a], non_blocking=True), args.reps)
            ep = dv.endpoint(dv.DV_EP_PEER if a != b else dv.DV_EP_DEVICE, dsts[b].data_ptr(), n, device=b)
            ms2 = timed(a, lambda: dv.dv_flush(ctxs[a], bufs[a].data_ptr(), n, ep, 0, xfer=dv.DV_XFER_FUSED,
                                               stream=torch.cuda.current_stream(a)), args.reps)
            out(probe="pair", src=a, dst=b, bytes=n, ce_gbs=n / ms / 1e6, sm_store_gbs=n / ms2 / 1e6)

    # all pairs at once (ring shift g -> g+1), one host thread per source GPU
    def ring(kind):
        res = [0.0] * G

        def run(g):
            b = (g + 1) % G
            if kind == "ce":
                res[g] = timed(g, lambda: dsts[b].copy_(bufs[g], non_blocking=True), args.reps)
            else:
                ep = dv.endpoint(dv.DV_EP_PEER if b != g else dv.DV_EP_DEVICE, dsts[b].data_ptr(), n, device=b)
                res[g] = timed(g, lambda: dv.dv_flush(ctxs[g], bufs[g].data_ptr(), n, ep, 0,
                                                      xfer=dv.DV_XFER_FUSED, stream=torch.cuda.current_stream(g)),
                               args.reps)
        th = [threading.Thread(target=run, args=(g,)) for g in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        return [n / ms / 1e6 for ms in res]
    for kind in ("ce", "sm_store"):
        r = ring(kind)
        out(probe="ring_all", kind=kind, per_gpu_gbs=r, min_gbs=min(r), sum_gbs=sum(r))

    # pinned host D2H / H2D per GPU, then every GPU at once
    hosts = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(G)]
    for g in range(G):
        d2h = n / timed(g, lambda: hosts[g].copy_(bufs[g], non_blocking=True), args.reps) / 1e6
        h2d = n / timed(g, lambda: bufs[g].copy_(hosts[g], non_blocking=True), args.reps) / 1e6
        out(probe="host_single", gpu=g, d2h_gbs=d2h, h2d_gbs=h2d)
    for name, fn in (("d2h", lambda g: hosts[g].copy_(bufs[g], non_blocking=True)),
                     ("h2d", lambda g: bufs[g].copy_(hosts[g], non_blocking=True))):
        res = [0.0] * G

        def run(g):
            res[g] = n / timed(g, lambda: fn(g), args.reps) / 1e6
        th = [threading.Thread(target=run, args=(g,)) for g in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        out(probe="host_all", dir=name, per_gpu_gbs=res, sum_gbs=sum(res))
    for c in ctxs:
        c.close()


if __name__ == "__main__":
    main()
