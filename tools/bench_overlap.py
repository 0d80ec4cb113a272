"""NEXT-2: token streaming overlapped with the model's compute (PAPER.md:123-135 Opt 2/3; §5.1
"streaming slowdown is within 2%"; the overhead factor m of Eq. 3-6).

A synthetic model step stands in for the model (torch ops are plumbing here, not the product):
  * "gemm"  -- two bf16 8192^3 GEMMs (compute-bound, prefill-like, ~1.4 ms);
  * "hbm"   -- a 1 GiB device copy (HBM-bound, decode-like: a decode step reads weights + KV).
Step t's compute runs on a compute stream; the K/V the model produced in step t-1 (one new
position of every layer: a C2 token step, 6.55 MB) is streamed to pinned host on a high-priority
stream with dvstream (DV_XFER_DECOUPLED, the headline form), ordered after step t-1's compute --
i.e. streaming overlaps step t's compute exactly as Opt 3 describes.

Measurement (paired, interleaved, so clock / power drift cancels): trials of K steps alternate
without / with streaming in an ABBA order; a trial's time runs from its first compute launch to
the point where its compute AND every flag of its streamed steps are done. The slowdown of each
adjacent (without, with) pair is one sample; we report its mean and a 95 % confidence interval
(Student t), the compute kernels' own slowdown (their event-bracketed durations), and m. The
streamed words are verified on the device (dvt_verify against the generator) for every step of
the last trial.
"""
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
STEP = 2 * L * B * H * D * 2
# two-sided 95 % Student t quantiles by degrees of freedom (n - 1)
_T95 = {1: 12.706, 2: 4.303, 3: 3.182, 4: 2.776, 5: 2.571, 6: 2.447, 7: 2.365, 8: 2.306, 9: 2.262,
        10: 2.228, 11: 2.201, 12: 2.179, 13: 2.160, 14: 2.145, 15: 2.131, 16: 2.120, 17: 2.110,
        18: 2.101, 19: 2.093, 20: 2.086, 24: 2.064, 29: 2.045, 39: 2.023}


def t95(df):
    keys = sorted(_T95)
    for k in keys:
        if df <= k:
            return _T95[k]
    return 1.96


def ci(xs):
    m = statistics.fmean(xs)
    if len(xs) < 2:
        return m, None
    return m, t95(len(xs) - 1) * statistics.stdev(xs) / math.sqrt(len(xs))


def measure(ctx, cache, seed, pos0=P, steps=20, pairs=24, kinds=("gemm", "hbm"), xfer=None):
    """Returns {kind: {...}} for the synthetic model steps in `kinds`."""
    dev = torch.device("cuda", torch.cuda.current_device())
    xfer = dv.DV_XFER_DECOUPLED if xfer is None else xfer
    comp = torch.cuda.Stream()
    strm = torch.cuda.Stream(priority=-1)       # highest priority: streaming CTAs scheduled first
    log = torch.empty(STEP * steps // 2, dtype=torch.int16, pin_memory=True)
    fl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    ring = dv.endpoint_array([dv.endpoint_of(log, fl, n_slots=steps, slot_bytes=STEP)])
    stage = dv.Setup([0, L], [0, B], S)
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    big_src = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    big_dst = torch.empty_like(big_src)
    fns = {"gemm": lambda: (torch.matmul(a, b), torch.matmul(a, b)), "hbm": lambda: big_dst.copy_(big_src)}
    seq = [int(fl[0])]
    out = {}

    def trial(fn, stream_on):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(comp)
        for i in range(steps):
            with torch.cuda.stream(comp):
                ev[i][0].record(comp)
                fn()
                ev[i][1].record(comp)
            if stream_on:
                # step i-1's new K/V (position pos0 + i) streams while step i computes: ordered
                # after the compute that "wrote" it (event of the previous step), on `strm`
                if i > 0:
                    strm.wait_event(ev[i - 1][1])
                q = pos0 + i
                seq[0] += 1
                dv.dv_stream_out(ctx, cache, (0, L, 0, B, q, q + 1), stage, 0, 0, stage, ring, seq=seq[0],
                                 xfer=xfer, stream=strm)
        comp.wait_stream(strm)
        if stream_on:
            dv.dv_wait(ctx, ring[0], 0, seq[0], stream=comp)   # the trial ends when its last flag is visible
        t1.record(comp)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1), [x.elapsed_time(y) for x, y in ev]

    for kind in kinds:
        fn = fns[kind]
        for _ in range(2):
            trial(fn, False)
            trial(fn, True)
        base, with_, slow, cbase, cwith = [], [], [], [], []
        for pr in range(pairs):
            order = (False, True) if pr % 2 == 0 else (True, False)   # ABBA
            r = {}
            for on in order:
                r[on] = trial(fn, on)
            base.append(r[False][0] / steps)
            with_.append(r[True][0] / steps)
            slow.append(100.0 * (r[True][0] - r[False][0]) / r[False][0])
            cbase += r[False][1]
            cwith += r[True][1]
        m_slow, hw = ci(slow)
        cb, cw = statistics.median(cbase), statistics.median(cwith)
        out[kind] = {
            "step_ms_without": statistics.fmean(base), "step_ms_with": statistics.fmean(with_),
            "step_slowdown_pct": m_slow, "step_slowdown_ci95_pct": hw,
            "m_factor": statistics.fmean(with_) / statistics.fmean(base),
            "compute_ms_p50_without": cb, "compute_ms_p50_with": cw,
            "compute_slowdown_pct": 100.0 * (cw - cb) / cb,
            "pairs": pairs, "steps_per_trial": steps, "steps_per_variant": pairs * steps,
            "stream_bytes_per_step": STEP,
            "resolved": (hw is not None and abs(m_slow) > hw),
        }
    # every word of every step of the last streaming trial, on the device
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    last = seq[0]
    for s in range(last - steps + 1, last + 1):
        i = (s - (last - steps + 1))
        q = pos0 + i
        w = log[(s % steps) * STEP // 2:(s % steps + 1) * STEP // 2]
        dv.dvt_verify(cache, cnt.data_ptr(), seed=seed, reg=dv.region(0, L, 0, B, q, q + 1), wire_ptr=w.data_ptr())
    torch.cuda.synchronize()
    out["parity"] = {"steps_verified": steps, "words": steps * STEP // 2, "mismatches": int(cnt.item()),
                     "how": "dvt_verify of the last streaming trial's ring slots vs the generator"}
    out["how"] = ("trials of K steps alternate without/with streaming (ABBA); slowdown per adjacent pair; "
                  "mean with a Student-t 95% CI; streaming = dv_stream_out DECOUPLED on a high-priority stream "
                  "after the previous step's compute")
    return out


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=24)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--xfer", default="decoupled", choices=["decoupled", "fused"])
    args = ap.parse_args()
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    cache = dv.cache(k, v)
    seed = 20240305
    dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=seed)
    ctx = dv.dv_create(0)
    xf = {"decoupled": dv.DV_XFER_DECOUPLED, "fused": dv.DV_XFER_FUSED}[args.xfer]
    r = measure(ctx, cache, seed, steps=args.steps, pairs=args.pairs, xfer=xf)
    r["xfer"] = args.xfer
    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
