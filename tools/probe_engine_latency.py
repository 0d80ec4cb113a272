"""Per-layer token latency (writer end -> seq flag released), C2 layer (160 KiB) to pinned host
(system-scope release) or into HBM (gpu scope), idle and while a bf16 GEMM loop saturates the SMs
on a low-priority stream. Paths compared:
  launch   dv_scatter per layer on a high-priority stream right behind the writer (PDL), as in
           round 1 (profiles/r01g_latency_loaded.jsonl);
  engine   the persistent engine (dv_engine_*): a plan per layer, kicked by a stream memory write
           after the writer (dv_engine_kick);
  ring     the same plans, rung by the writer kernel's last CTA itself (dvt_fill_ring).
Stamps: %globaltimer of the writer's end (max over its CTAs) and of the flag release (the copy
kernel's dvt_trace stamp, or the engine's per-job stamp).
  python tools/probe_engine_latency.py [--n 400] [--ctas 8]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
LAYER = 2 * B * H * D * 2


def pct(xs):
    xs = sorted(xs)
    return {"p50_us": round(xs[len(xs) // 2], 3), "p99_us": round(xs[int(len(xs) * 0.99)], 3),
            "min_us": round(xs[0], 3), "n": len(xs)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=400)
    ap.add_argument("--ctas", type=int, default=8)
    args = ap.parse_args()
    n = args.n
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    cache = dv.cache(k, v)
    ctx = dv.dv_create(0)
    lo, hi = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    bm = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    runs = 4                                       # engine / ring x idle / loaded
    T = runs * (n // L) + 2
    te = torch.zeros(n, dtype=torch.int64, device="cuda")
    ts = torch.zeros((n, 4), dtype=torch.int64, device="cuda")
    NST = 4096
    stamps = torch.zeros((NST, 5), dtype=torch.int64, device="cuda")
    ticket = torch.zeros(1, dtype=torch.int32, device="cuda")
    dummy = torch.zeros(1, dtype=torch.int64, device="cuda")
    import time
    for dst in ("host", "hbm"):
        host = dst == "host"
        log = torch.empty(LAYER // 2 * L * T, dtype=torch.int16, device="cpu" if host else "cuda", pin_memory=host)
        fl = torch.zeros(L, dtype=torch.int64, device="cpu" if host else "cuda", pin_memory=host)
        ep = dv.endpoint_of(log, fl)
        eng = dv.Engine(ctx, args.ctas)
        plans = [eng.plan_scatter(cache, (l, l + 1, 0, B, P, P + 1), ep, l * LAYER, L * LAYER, flag_slot=l, seq=1,
                                  max_step=T - 1) for l in range(L)]
        dbs = [eng.doorbell(pl) for pl in plans]
        eng.park()
        eng.trace(stamps.data_ptr(), NST)
        # warm every kernel first (lazy loading); the ring goes to a dummy word, not the engine
        torch.matmul(a, bm)
        for l in range(L):
            reg = (l, l + 1, 0, B, P, P + 1)
            dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=1, reg=reg, stream=hi)
            dv.dvt_fill_ring(cache, 1, reg, dummy.data_ptr(), 0, ticket.data_ptr(), stream=hi)
            dv.dv_scatter(ctx, cache, reg, ep, l * LAYER, flag_slot=l, seq=10 ** 6, stream=hi)
        torch.cuda.synchronize()
        eng_step = 0
        for mode in ("launch", "engine", "ring"):
            for loaded in (False, True):
                te.zero_()
                ts.zero_()
                ts[:, 1:3] = 2 ** 63 - 1
                torch.cuda.synchronize()
                if mode != "launch":
                    eng.resume()
                if loaded:
                    with torch.cuda.stream(lo):
                        for _ in range(60 if n <= 400 else 150):
                            torch.matmul(a, bm)
                dv.dvt_spin(20_000_000, 1, stream=hi)
                for i in range(n):
                    layer = i % L
                    t = eng_step + i // L
                    reg = (layer, layer + 1, 0, B, P + t, P + t + 1)
                    if mode == "ring":
                        dv.dvt_fill_ring(cache, 1, reg, dbs[layer], t, ticket.data_ptr(), t_end_ptr=te[i].data_ptr(),
                                         stream=hi)
                    else:
                        dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=1, reg=reg, stream=hi, t_end_ptr=te[i].data_ptr())
                    if mode == "engine":
                        eng.kick(plans[layer], t, stream=hi)
                    elif mode == "launch":
                        dv.dvt_trace(ctx, ts[i].data_ptr())
                        dv.dv_scatter(ctx, cache, reg, ep, layer * LAYER, flag_slot=layer, seq=10 ** 7 + i, stream=hi)
                dv.dvt_trace(ctx, 0)
                hi.synchronize()
                lo.synchronize()
                if mode != "launch":
                    t0 = time.time()
                    while eng.done(plans[L - 1]) < eng_step + n // L:
                        assert time.time() - t0 < 20, eng.done(plans[L - 1])
                    eng.park()
                    rows = stamps[[((eng_step + i // L) * L + i % L) % NST for i in range(n)]]
                    fin = rows[:, 0]
                    phases = {name: pct(((rows[:, j] - te).double() / 1e3).tolist()[L:])["p50_us"]
                              for j, name in ((1, "found"), (2, "past_b1"), (3, "copy_issued"), (4, "past_b2"))}
                    eng_step += n // L
                else:
                    fin = ts[:, 0]
                    phases = {"resident": pct(((ts[:, 1] - te).double() / 1e3).tolist()[L:])["p50_us"],
                              "past_wait": pct(((ts[:, 2] - te).double() / 1e3).tolist()[L:])["p50_us"],
                              "stores_issued": pct(((ts[:, 3] - te).double() / 1e3).tolist()[L:])["p50_us"]}
                torch.cuda.synchronize()
                r = pct(((fin - te).double() / 1e3).tolist()[L:])
                row = {"dst": dst, "mode": mode, "loaded": loaded, "ctas": args.ctas, **r, "phase_p50_us": phases}
                print(json.dumps(row), flush=True)
        eng.close()
    ctx.close()


if __name__ == "__main__":
    main()
