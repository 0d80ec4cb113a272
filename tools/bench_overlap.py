"""NEXT-2: streaming overlapped with compute (PAPER.md:123-135 Opt 2/3; §5.1 "streaming slowdown is
within 2%"; the overhead factor m of Eq. 3-6).

Synthetic compute stands in for the model (torch ops = plumbing, not the product): a bf16 GEMM
(compute-bound, prefill-like) or a large device copy (HBM-bound, decode-like), launched per token
step on a compute stream. On a second stream dvstream streams the previous step's new K/V (C2:
6.55 MB, all 40 layers) to pinned host. We report the compute time alone, with concurrent
streaming (fused SM kernel, fused with a CTA budget, or staged = pack + copy engine), and the
slowdown. Writes one JSON line per variant.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
STEP = 2 * L * B * H * D * 2


def main():
    dev = torch.device("cuda", 0)
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device=dev)
    v = torch.empty_like(k)
    cache = dv.cache(k, v)
    dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=1)
    log = torch.empty(STEP * 8 // 2, dtype=torch.int16, pin_memory=True)
    fl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    ep = dv.endpoint_of(log, fl)
    comp = torch.cuda.Stream()
    strm_lo = torch.cuda.Stream()
    strm_hi = torch.cuda.Stream(priority=-1)   # highest priority: streaming CTAs scheduled first
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    big_src = torch.empty(2 << 30, dtype=torch.uint8, device=dev)
    big_dst = torch.empty_like(big_src)

    computes = {
        "gemm_bf16_8192x2": lambda: (torch.matmul(a, b), torch.matmul(a, b)),
        "hbm_copy_2GiB": lambda: big_dst.copy_(big_src),
    }
    ctxs = {"fused": dv.dv_create(0), "fused_16ctas": dv.dv_create(0, max_ctas=16),
            "fused_64ctas": dv.dv_create(0, max_ctas=64), "staged": dv.dv_create(0),
            "decoupled": dv.dv_create(0)}
    xfers = {"fused": dv.DV_XFER_FUSED, "fused_16ctas": dv.DV_XFER_FUSED, "fused_64ctas": dv.DV_XFER_FUSED,
             "staged": dv.DV_XFER_STAGED, "decoupled": dv.DV_XFER_DECOUPLED}
    seq0 = [0]
    n = 30
    for (cname, cfn), strm_name in [(kv, sn) for kv in computes.items() for sn in ("normal", "high")]:
        strm = strm_hi if strm_name == "high" else strm_lo

        def run(variant):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
            sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(comp)
            strm.wait_event(t0)
            for i in range(n):
                with torch.cuda.stream(comp):
                    ev[i][0].record(comp)
                    cfn()
                    ev[i][1].record(comp)
                if variant is not None:
                    q = P + i
                    sev[i][0].record(strm)
                    # the previous step's K/V (the cache is resident; its position is fresh)
                    dv.dv_scatter(ctxs[variant], cache, dv.region(0, L, 0, B, q, q + 1), ep, (i % 8) * STEP,
                                  flag_slot=0, seq=seq0[0] + i + 1, xfer=xfers[variant], stream=strm)
                    sev[i][1].record(strm)
            comp.wait_stream(strm)
            if variant is not None:
                # the step ends when the last chunk's flag is visible (decoupled: DMA + flag run on the
                # library's streams, not on strm)
                dv.dv_wait(ctxs[variant], ep, 0, seq0[0] + n, stream=comp)
                seq0[0] += n
            t1.record(comp)
            torch.cuda.synchronize()
            c_ms = sorted(x.elapsed_time(y) for x, y in ev)[n // 2]
            s_ms = sorted(x.elapsed_time(y) for x, y in sev)[n // 2] if variant else None
            return c_ms, s_ms, t0.elapsed_time(t1) / n
        for _ in range(2):
            run(None)
        base_c, _, base_tot = run(None)
        print(json.dumps({"compute": cname, "stream_priority": strm_name, "variant": "none",
                          "compute_ms_p50": base_c, "step_ms": base_tot}), flush=True)
        for var in ctxs:
            run(var)
            c, sm, tot = run(var)
            print(json.dumps({"compute": cname, "stream_priority": strm_name, "variant": var,
                              "compute_ms_p50": c, "stream_ms_p50": sm,
                              "step_ms": tot, "compute_slowdown_pct": 100 * (c - base_c) / base_c,
                              "step_slowdown_pct": 100 * (tot - base_tot) / base_tot,
                              "stream_gbs_under_load": (STEP / (sm * 1e-3) / 1e9 if sm and var != "decoupled"
                                                        else None),
                              "m_factor": tot / base_tot}), flush=True)


if __name__ == "__main__":
    main()
