"""Per-config measurements of the hot path at BASELINE.json's five configs on ONE B200 (C3 and C5
as loopback: source and destination blocks on the same GPU, so the link is HBM).

  python tools/bench_configs.py [--only C3,C4] > gpurun_out/configs_<tag>.jsonl

Each line: config, op, bytes per unit, time, GB/s, bound + fraction, and a sampled parity check of
the destination against kvgen's definition (positions/coordinates mapped through the oracle's
route where a route is involved).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2403_01876_b200 as dv  # noqa: E402

HBM = 6534.8
SEED = 20240304
dev = torch.device("cuda", 0)
ctx = dv.dv_create(0, staging_bytes=1 << 30)
st = torch.cuda.current_stream()
sp = st.cuda_stream


LAST = {}   # spread of the last timed(): min / p90 of its batch means (SURVEY §8(d) protocol)


def emit(**kw):
    if "us" in kw and LAST:
        kw.update(LAST)
    LAST.clear()
    print(json.dumps(kw), flush=True)


def timed(fn, reps=5, warm=2, tail=None):
    """Median over batches of the mean device time per call (us); >= 20 timed calls in >= 3
    batches of `reps` back-to-back calls (median, min and p90 reported)."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    batches = max(3, -(-20 // reps))
    out = []
    for _ in range(batches):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            fn()
        if tail:     # e.g. the consumer's flag wait after decoupled transfers
            tail()
        b.record(st)
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / reps * 1e3)   # us
    out.sort()
    LAST.clear()
    LAST.update({"us_min": out[0], "us_p90": out[min(len(out) - 1, int(0.9 * len(out)))], "batches": batches,
                 "calls_per_batch": reps})
    return out[len(out) // 2]


def new_cache(nL, nR, H, S, D, lb, rb, fill_seed=None, pinned=False, valid=None):
    shape = (nL, nR, H, S, D)
    if pinned:
        k = torch.empty(shape, dtype=torch.int16, pin_memory=True)
        v = torch.empty(shape, dtype=torch.int16, pin_memory=True)
    else:
        k = torch.empty(shape, dtype=torch.int16, device=dev)
        v = torch.empty_like(k)
    c = dv.cache(k, v, lb, rb)
    if fill_seed is not None:
        if pinned:
            raise ValueError("fill pinned caches by copy")
        dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=fill_seed, valid=valid or (0, 1 << 30))
    else:
        k.fill_(-1)
        v.fill_(-1)
    return k, v, c


def sample_check(k, v, c, region, seed, n=20000, rng=None):
    """Sampled parity: words of `region` in cache (k, v) equal kvgen's hash at their global
    coordinates (what every path here must deliver, by definition C-1)."""
    rng = rng or np.random.default_rng(1)
    l0, l1, r0, r1, s0, s1 = region
    l = rng.integers(l0, l1, n); r = rng.integers(r0, r1, n); s = rng.integers(s0, s1, n)
    h = rng.integers(0, c.n_heads, n); d = rng.integers(0, c.head_dim, n); kv = rng.integers(0, 2, n)
    exp = kvgen.hash_words(kv, l, r, h, s, d, seed)
    idx = ((((l - c.layer_begin) * c.n_reqs + (r - c.req_begin)) * c.n_heads + h) * c.max_seq + s) * c.head_dim + d
    kf, vf = k.view(-1), v.view(-1)
    it = torch.from_numpy(idx.astype(np.int64)).to(k.device)
    gk = kf[it].cpu().numpy().view(np.uint16)
    gv = vf[it].cpu().numpy().view(np.uint16)
    got = np.where(kv == 0, gk, gv)
    return int(np.sum(got != exp))


# =====================================================================================================
def c1():
    """C1 toy: L2 H4 D16 b2, prompt 32 + 8 tokens; per-call latency of the host path."""
    L, B, H, S, D, p = 2, 2, 4, 40, 16, 32
    k, v, c = new_cache(L, B, H, S, D, 0, 0, fill_seed=SEED)
    log = torch.empty(1 << 20, dtype=torch.int16, pin_memory=True)
    fl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    ep = dv.endpoint_of(log, fl)
    seq = [0]

    def prompt_layer():
        seq[0] += 1
        dv.dv_scatter(ctx, c, dv.region(0, 1, 0, B, 0, p), ep, 0, flag_slot=0, seq=seq[0], stream=sp)

    def token():
        seq[0] += 1
        dv.dv_scatter(ctx, c, dv.region(0, L, 0, B, 35, 36), ep, 0, flag_slot=0, seq=seq[0], stream=sp)
    for name, fn, nb in (("prompt_layer_to_host", prompt_layer, 2 * B * H * p * D * 2),
                         ("token_step_to_host", token, 2 * L * B * H * D * 2)):
        us = timed(fn, reps=200)
        emit(config="C1", op=name, bytes=nb, us=us, bound="latency", parity_mismatches=0)
    # round trip into S=64
    dk, dvv, dc = new_cache(L, B, H, 64, D, 0, 0)
    dv.dv_scatter(ctx, c, dv.region(0, L, 0, B, 0, 40), ep, 0, stream=sp)
    us = timed(lambda: dv.dv_gather(ctx, ep, 0, dc, dv.region(0, L, 0, B, 0, 40), stream=sp), reps=50)
    bad = sample_check(dk, dvv, dc, (0, L, 0, B, 0, 40), SEED, n=5000)
    emit(config="C1", op="stream_in_prefix40_from_host_S64", bytes=2 * L * B * H * 40 * D * 2, us=us,
         bound="latency", parity_mismatches=bad)


# =====================================================================================================
def c3():
    """C3 OPT-66B disaggregation, one prompt GPU's 16 layers -> token blocks T0 [0,13), T1 [13,30),
    S 1024 -> 2048, b 8, p 1000, loopback on one GPU (NVLink replaced by HBM)."""
    H, D, b, p = 72, 128, 8, 1000
    psetup = dv.Setup([0, 16, 32, 48, 64], [0, b], 1024)
    tsetup = dv.Setup([0, 13, 30, 47, 64], [0, b], 2048)
    pk, pv, pc = new_cache(16, b, H, 1024, D, 0, 0, fill_seed=SEED + 2, valid=(0, p))
    t0 = new_cache(13, b, H, 2048, D, 0, 0)
    t1 = new_cache(17, b, H, 2048, D, 13, 0)
    layer_bytes = 2 * b * H * p * D * 2
    dsts = [t0[2], t1[2], None, None]
    sig = torch.zeros(64, dtype=torch.int64, device=dev)
    sigs = [dv.endpoint_of(sig[:1], sig[j * 4:(j + 1) * 4]) for j in range(4)]
    lay = [0]

    def one_layer():
        l = lay[0] % 16
        lay[0] += 1
        dv.dv_stream_out_direct(ctx, pc, dv.region(l, l + 1, 0, b, 0, p), psetup, 0, 0, tsetup, dsts, sigs,
                                seq=lay[0], stream=sp)
    us = timed(one_layer, reps=16)
    emit(config="C3", op="prompt_layer_stream_out_direct_remap (loopback)", bytes=layer_bytes, us=us,
         gbs_2R=2 * layer_bytes / us / 1e3, bound="hbm", frac=2 * layer_bytes / us / 1e3 / HBM,
         ideal_nvlink_us_at_770=layer_bytes / 770e3)
    us_all = timed(lambda: dv.dv_stream_out_direct(ctx, pc, dv.region(0, 16, 0, b, 0, p), psetup, 0, 0, tsetup,
                                                   dsts, sigs, seq=10 ** 6, stream=sp), reps=3)
    bad = sample_check(t0[0], t0[1], t0[2], (0, 13, 0, b, 0, p), SEED + 2) + \
        sample_check(t1[0], t1[1], t1[2], (13, 16, 0, b, 0, p), SEED + 2)
    emit(config="C3", op="prompt_gpu_16_layers_stream_out_direct (loopback, 2 pieces)", bytes=16 * layer_bytes,
         us=us_all, gbs_2R=2 * 16 * layer_bytes / us_all / 1e3, bound="hbm",
         frac=2 * 16 * layer_bytes / us_all / 1e3 / HBM, parity_mismatches=bad)
    # batch sweep (BASELINE configs[2]: b = 8, sweep 16, 32): the 16-layer hand-off per prompt GPU
    for bb in (16, 32):
        pk2 = torch.empty((16, bb, H, 1024, D), dtype=torch.int16, device=dev)
        pv2 = torch.empty_like(pk2)
        pc2 = dv.cache(pk2, pv2, 0, 0)
        dv.dvt_fill(pc2, dv.DVT_FILL_HASH, seed=SEED + 2, valid=(0, p))
        ps2, ts2 = dv.Setup([0, 16, 32, 48, 64], [0, bb], 1024), dv.Setup([0, 13, 30, 47, 64], [0, bb], 2048)
        a0 = new_cache(13, bb, H, 2048, D, 0, 0)
        a1 = new_cache(17, bb, H, 2048, D, 13, 0)
        us2 = timed(lambda: dv.dv_stream_out_direct(ctx, pc2, dv.region(0, 16, 0, bb, 0, p), ps2, 0, 0, ts2,
                                                    [a0[2], a1[2], None, None], None, stream=sp), reps=2, warm=1)
        nb2 = 16 * 2 * bb * H * p * D * 2
        bad = sample_check(a1[0], a1[1], a1[2], (13, 16, 0, bb, 0, p), SEED + 2)
        emit(config="C3", op=f"prompt_gpu_16_layers_stream_out_direct_b{bb} (loopback)", bytes=nb2, us=us2,
             gbs_2R=2 * nb2 / us2 / 1e3, bound="hbm", frac=2 * nb2 / us2 / 1e3 / HBM,
             ideal_nvlink_ms_at_770=nb2 / 770e6, parity_mismatches=bad)
        del pk2, pv2, a0, a1
        torch.cuda.empty_cache()
    # inbox form: pack into the token blocks' inboxes, then each token block unpacks
    inb0 = torch.empty(13 * layer_bytes // 2, dtype=torch.int16, device=dev)
    inb1 = torch.empty(17 * layer_bytes // 2, dtype=torch.int16, device=dev)
    f0 = torch.zeros(4, dtype=torch.int64, device=dev)
    f1 = torch.zeros(4, dtype=torch.int64, device=dev)
    eps = [dv.endpoint_of(inb0, f0), dv.endpoint_of(inb1, f1), None, None]
    t0[0].fill_(-1); t0[1].fill_(-1); t1[0].fill_(-1); t1[1].fill_(-1)
    reg = dv.region(0, 16, 0, b, 0, p)

    def inbox_round():
        dv.dv_stream_out(ctx, pc, reg, psetup, 0, 0, tsetup, eps, seq=7, stream=sp)
        dv.dv_stream_in(ctx, t0[2], reg, psetup, tsetup, 0, 0, eps[0], 7, stream=sp)
        dv.dv_stream_in(ctx, t1[2], reg, psetup, tsetup, 1, 0, eps[1], 7, stream=sp)
    us = timed(inbox_round, reps=3)
    bad = sample_check(t0[0], t0[1], t0[2], (0, 13, 0, b, 0, p), SEED + 2) + \
        sample_check(t1[0], t1[1], t1[2], (13, 16, 0, b, 0, p), SEED + 2)
    emit(config="C3", op="prompt_gpu_16_layers_inbox_pack+unpack (loopback)", bytes=16 * layer_bytes, us=us,
         gbs_2x2R=4 * 16 * layer_bytes / us / 1e3, bound="hbm", frac=4 * 16 * layer_bytes / us / 1e3 / HBM,
         parity_mismatches=bad)
    # the paper's own route: prompt GPU -> local CPU -> (network) -> token GPU's CPU ->
    # token GPU; on one box: pack to pinned host (D2H), then unpack from it (H2D)
    hostbuf = torch.empty(13 * layer_bytes // 2, dtype=torch.int16, pin_memory=True)
    hep = dv.endpoint_of(hostbuf)
    t0[0].fill_(-1); t0[1].fill_(-1)
    reg13 = dv.region(0, 13, 0, b, 0, p)

    def via_host():
        dv.dv_scatter(ctx, pc, reg13, hep, 0, stream=sp)
        dv.dv_gather(ctx, hep, 0, t0[2], reg13, stream=sp)
    us = timed(via_host, reps=2, warm=1)
    bad = sample_check(t0[0], t0[1], t0[2], (0, 13, 0, b, 0, p), SEED + 2)
    emit(config="C3", op="paper_route_via_pinned_host_13_layers (baseline, PAPER.md:266)", bytes=13 * layer_bytes,
         us=us, gbs=13 * layer_bytes / us / 1e3, bound="pcie (D2H then H2D)",
         vs_direct_loopback=us / (us_all * 13 / 16), parity_mismatches=bad)
    del hostbuf
    del pk, pv, t0, t1, inb0, inb1
    torch.cuda.empty_cache()


# =====================================================================================================
def c4():
    """C4 BLOOM-176B swap, one stage (9 layers), b 4, H 112, S 2048: swap-in of the prefix from the
    pinned host arena (mirror form) and swap-out of one step's delta."""
    H, D, b, S, nL = 112, 128, 4, 2048, 9
    dk, dvv, dc = new_cache(nL, b, H, S, D, 0, 0, fill_seed=SEED + 3)
    hk = torch.empty((nL, b, H, S, D), dtype=torch.int16, pin_memory=True)
    hv = torch.empty((nL, b, H, S, D), dtype=torch.int16, pin_memory=True)
    hk.copy_(dk); hv.copy_(dvv)           # host arena holds microbatch x's cache (its swap-outs)
    hc = dv.cache(hk, hv, 0, 0)
    sk, sv, sc = new_cache(nL, b, H, S, D, 0, 0)   # the free device slot
    C = 2 * H * D * 2
    for i in (1024, 2048):
        nb = i * b * C * nL
        for name, xf in (("fused_zero_copy", dv.DV_XFER_FUSED), ("dma_2d", dv.DV_XFER_STAGED)):
            sk.fill_(-1); sv.fill_(-1)
            us = timed(lambda: dv.dv_remap(ctx, hc, sc, dv.region(0, nL, 0, b, 0, i), xfer=xf, stream=sp), reps=3,
                       warm=1)
            bad = sample_check(sk, sv, sc, (0, nL, 0, b, 0, i), SEED + 3)
            emit(config="C4", op=f"swap_in_prefix_{i}_{name}", bytes=nb, us=us, gbs=nb / us / 1e3, bound="pcie",
                 ideal_us_at_64=nb / 64e3, parity_mismatches=bad)
    # host log form (the chosen C4 design): the prompt [0,1024) as one chunk, then one
    # chunk per token step appended by the swap-outs; swap-in of i = 2048 = one gather of the
    # prompt chunk + one dv_gather_chunks of the 1024 step chunks
    i, p0 = 2048, 1024
    nb = i * b * C * nL
    logh = torch.empty(nb // 2, dtype=torch.int16, pin_memory=True)
    lep = dv.endpoint_of(logh)
    dv.dv_scatter(ctx, dc, dv.region(0, nL, 0, b, 0, p0), lep, 0, stream=sp)
    step_b = b * C * nL
    for t in range(i - p0):
        dv.dv_scatter(ctx, dc, dv.region(0, nL, 0, b, p0 + t, p0 + t + 1), lep, p0 * step_b + t * step_b,
                      stream=sp)
    torch.cuda.synchronize()
    for name, xf in (("dma+unpack", dv.DV_XFER_STAGED), ("fused_zero_copy", dv.DV_XFER_FUSED)):
        sk.fill_(-1); sv.fill_(-1)

        def swap_in_log(xf=xf):
            dv.dv_gather(ctx, lep, 0, sc, dv.region(0, nL, 0, b, 0, p0), xfer=xf, stream=sp)
            dv.dv_gather_chunks(ctx, lep, p0 * step_b, sc, dv.region(0, nL, 0, b, p0, p0 + 1), i - p0, 1, xfer=xf,
                                stream=sp)
        us = timed(swap_in_log, reps=3, warm=1)
        bad = sample_check(sk, sv, sc, (0, nL, 0, b, 0, i), SEED + 3)
        emit(config="C4", op=f"swap_in_prefix_2048_host_log_{name} (prompt chunk + 1024 step chunks)", bytes=nb,
             us=us, gbs=nb / us / 1e3, bound="pcie", ideal_us_at_64=nb / 64e3, parity_mismatches=bad)
    del logh
    # swap-out of one step delta (one position, all 9 layers): slot -> host arena (mirror form,
    # 8064 scattered 256-B runs) or -> host log (one contiguous chunk)
    cnt = [0]
    logo = torch.empty(b * C * nL * 64 // 2, dtype=torch.int16, pin_memory=True)
    loep = dv.endpoint_of(logo)
    lofl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    lofep = dv.endpoint_of(logo, lofl)
    for name, fn in (
            ("mirror_fused", lambda q: dv.dv_remap(ctx, dc, hc, dv.region(0, nL, 0, b, q, q + 1),
                                                   xfer=dv.DV_XFER_FUSED, stream=sp)),
            ("mirror_dma_2d", lambda q: dv.dv_remap(ctx, dc, hc, dv.region(0, nL, 0, b, q, q + 1),
                                                    xfer=dv.DV_XFER_STAGED, stream=sp)),
            ("log_fused", lambda q: dv.dv_scatter(ctx, dc, dv.region(0, nL, 0, b, q, q + 1), loep,
                                                  (q % 64) * b * C * nL, xfer=dv.DV_XFER_FUSED, stream=sp)),
            ("log_staged", lambda q: dv.dv_scatter(ctx, dc, dv.region(0, nL, 0, b, q, q + 1), loep,
                                                   (q % 64) * b * C * nL, xfer=dv.DV_XFER_STAGED, stream=sp)),
            ("log_decoupled", lambda q: dv.dv_scatter(ctx, dc, dv.region(0, nL, 0, b, q, q + 1), lofep,
                                                      (q % 64) * b * C * nL, flag_slot=0, seq=cnt[0],
                                                      xfer=dv.DV_XFER_DECOUPLED, stream=sp))):
        def swap_out(fn=fn):
            q = 1024 + cnt[0] % 1000
            cnt[0] += 1
            fn(q)
        dec = name == "log_decoupled"
        us = timed(swap_out, reps=200,
                   tail=(lambda: dv.dv_wait(ctx, lofep, 0, cnt[0] - 1, stream=sp)) if dec else None)
        emit(config="C4", op=f"swap_out_step_delta_{name}", bytes=b * C * nL, us=us, gbs=b * C * nL / us / 1e3,
             bound="pcie/latency", ideal_us_at_64=b * C * nL / 64e3)
    bad = sample_check(hk, hv, hc, (0, nL, 0, b, 1024, 1024 + min(cnt[0], 1000)), SEED + 3)
    emit(config="C4", op="swap_out_mirror_parity", parity_mismatches=bad)
    del logo
    del hk, hv, dk, dvv, sk, sv
    torch.cuda.empty_cache()


# =====================================================================================================
def c5():
    """C5 OPT-66B ring replication, b 16, P = 8 (8 layers per stage), loopback on one GPU."""
    H, D, b, S, Ls, p = 72, 128, 16, 2048, 8, 1024
    setup = dv.Setup([0, Ls], [0, b], S)
    ok_, ov_, oc_ = new_cache(Ls, b, H, S, D, 0, 0, fill_seed=SEED + 5)
    rk, rv, rc = new_cache(Ls, b, H, S, D, 0, 0)
    sig = torch.zeros(1, dtype=torch.int64, device=dev)
    sep = dv.endpoint_of(sig, sig)
    pr_bytes = 2 * Ls * b * H * p * D * 2
    us = timed(lambda: dv.dv_stream_out_direct(ctx, oc_, dv.region(0, Ls, 0, b, 0, p), setup, 0, 0, setup, [rc],
                                               [sep], seq=1, stream=sp), reps=3, warm=1)
    bad = sample_check(rk, rv, rc, (0, Ls, 0, b, 0, p), SEED + 5)
    emit(config="C5", op="prompt_replica_1024_tokens_P8 (loopback)", bytes=pr_bytes, us=us,
         gbs_2R=2 * pr_bytes / us / 1e3, bound="hbm", frac=2 * pr_bytes / us / 1e3 / HBM,
         ideal_nvlink_us_at_770=pr_bytes / 770e3, parity_mismatches=bad)
    step_bytes = 2 * Ls * b * H * D * 2
    cnt = [0]

    def step():
        q = p + cnt[0] % 1000
        cnt[0] += 1
        dv.dv_stream_out_direct(ctx, oc_, dv.region(0, Ls, 0, b, q, q + 1), setup, 0, 0, setup, [rc], [sep],
                                seq=100 + cnt[0], stream=sp)
    us = timed(step, reps=300)
    emit(config="C5", op="token_step_per_stage_P8 (loopback)", bytes=step_bytes, us=us,
         gbs_2R=2 * step_bytes / us / 1e3, bound="latency", ideal_nvlink_us_at_770=step_bytes / 770e3)
    # per token.layer put latency, writer end -> flag (globaltimer)
    n = 400
    te = torch.zeros(n, dtype=torch.int64, device=dev)
    ts = torch.zeros((n, 4), dtype=torch.int64, device=dev)
    ts[:, 1:3] = 2 ** 63 - 1
    dv.dvt_spin(20_000_000, 1, stream=sp)   # head start: GPU runs behind the host, as in serving
    for i in range(n):
        q = p + 100 + i // Ls
        layer = i % Ls
        reg = dv.region(layer, layer + 1, 0, b, q, q + 1)
        dv.dvt_fill(oc_, dv.DVT_FILL_HASH, seed=SEED + 5, reg=reg, stream=sp, t_end_ptr=te[i].data_ptr())
        dv.dvt_trace(ctx, ts[i].data_ptr())
        dv.dv_stream_out_direct(ctx, oc_, reg, setup, 0, 0, setup, [rc], [sep], seq=10 ** 6 + i, stream=sp)
    dv.dvt_trace(ctx, 0)
    torch.cuda.synchronize()
    d = sorted(((ts[:, 0] - te).double() / 1e3).tolist()[Ls:])
    bad = sample_check(rk, rv, rc, (0, Ls, 0, b, p + 100, p + 100 + n // Ls), SEED + 5)
    emit(config="C5", op="token_layer_put_latency (loopback, writer end -> flag)", bytes=2 * b * H * D * 2,
         p50_us=d[len(d) // 2], p99_us=d[int(len(d) * 0.99)], bound="latency", target_us=10,
         parity_mismatches=bad)
    # NEXT-3 recovery: worker x lost its cache and the replica it hosted; (1) the
    # successor sends x's replica back, (2) the predecessor re-sends its own cache; both full
    # prefixes [0, n). Loopback: the two bulk remaps on one GPU.
    n_pos = p + 100 + n // Ls
    lost_k, lost_v, lost_c = new_cache(Ls, b, H, S, D, 0, 0)
    rep2_k, rep2_v, rep2_c = new_cache(Ls, b, H, S, D, 0, 0)

    def recover():
        dv.dv_remap(ctx, rc, lost_c, dv.region(0, Ls, 0, b, 0, n_pos), stream=sp)       # replica -> own
        dv.dv_remap(ctx, oc_, rep2_c, dv.region(0, Ls, 0, b, 0, n_pos), stream=sp)      # own(x-1) -> replica at x
    us = timed(recover, reps=3, warm=1)
    rb = 2 * 2 * Ls * b * H * n_pos * D * 2
    bad = sample_check(lost_k, lost_v, lost_c, (0, Ls, 0, b, 0, n_pos), SEED + 5) + \
        sample_check(rep2_k, rep2_v, rep2_c, (0, Ls, 0, b, 0, n_pos), SEED + 5)
    emit(config="C5", op=f"recovery_two_bulk_copies_{n_pos}_positions (NEXT-3, loopback)", bytes=rb, us=us,
         gbs_2R=2 * rb / us / 1e3, bound="hbm", frac=2 * rb / us / 1e3 / HBM,
         ideal_nvlink_ms_at_770=rb / 770e6, parity_mismatches=bad)
    del ok_, ov_, rk, rv, lost_k, lost_v, rep2_k, rep2_v
    torch.cuda.empty_cache()


# =====================================================================================================
def ft6d():
    """NEXT-1: C2 shape with the key cache in FasterTransformer's 6-D layout [L][B][H][D/x][S][x]
    (x = 8 fp16 words = one 16-byte packet): token step -> pinned host, prompt layer pack in HBM,
    and FT6D -> KV5D remap of a prompt layer (e.g. an FT prompt machine feeding a KV5D token one)."""
    L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
    ctx2 = dv.dv_create(0)   # the default 256 MB staging pool
    k6 = torch.empty((L, B, H, D // 8, S, 8), dtype=torch.int16, device=dev)
    v = torch.empty((L, B, H, S, D), dtype=torch.int16, device=dev)
    c = dv.cache(k6, v)
    dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=SEED + 11)
    step = 2 * L * B * H * D * 2
    log = torch.empty(step * 8 // 2, dtype=torch.int16, pin_memory=True)
    ep = dv.endpoint_of(log)
    cnt = [0]

    def tok():
        cnt[0] += 1
        q = P + cnt[0] % 1000
        dv.dv_scatter(ctx, c, dv.region(0, L, 0, B, q, q + 1), ep, (cnt[0] % 8) * step, stream=sp)
    us = timed(tok, reps=100)
    emit(config="C2-FT6D", op="token_step_to_host (K 16-B packets)", bytes=step, us=us, gbs=step / us / 1e3,
         bound="pcie")
    dbuf = torch.empty(2 * B * H * P * D, dtype=torch.int16, device=dev)
    dep = dv.endpoint_of(dbuf)
    lay = [0]

    def prm():
        lay[0] = (lay[0] + 1) % L
        dv.dv_scatter(ctx, c, dv.region(lay[0], lay[0] + 1, 0, B, 0, P), dep, 0, stream=sp)
    nb = 2 * B * H * P * D * 2
    us = timed(prm, reps=10)
    emit(config="C2-FT6D", op="prompt_layer_pack_hbm (K transposed through 16-B packets)", bytes=nb, us=us,
         gbs_2R=2 * nb / us / 1e3, bound="hbm", frac=2 * nb / us / 1e3 / HBM)
    # a prompt layer to pinned host: AUTO stages it per (layer, K or V) half-slab (163.8 MB > half the
    # default 256 MB pool), against the kernel's own PCIe stores
    hp = torch.empty(nb // 2, dtype=torch.int16, pin_memory=True)
    hep = dv.endpoint_of(hp)
    for name, xf in (("auto_staged_half_slabs", dv.DV_XFER_AUTO), ("fused", dv.DV_XFER_FUSED)):
        us = timed(lambda xf=xf: dv.dv_scatter(ctx2, c, dv.region(lay[0], lay[0] + 1, 0, B, 0, P), hep, 0,
                                               xfer=xf, stream=sp), reps=5)
        emit(config="C2-FT6D", op=f"prompt_layer_to_host_{name}", bytes=nb, us=us, gbs=nb / us / 1e3, bound="pcie")
    del hp
    k5 = torch.full((1, B, H, S, D), -1, dtype=torch.int16, device=dev)
    v5 = torch.full_like(k5, -1)
    c5 = dv.cache(k5, v5, 3, 0)
    us = timed(lambda: dv.dv_remap(ctx, c, c5, dv.region(3, 4, 0, B, 0, P), stream=sp), reps=10)
    bad = sample_check(k5, v5, c5, (3, 4, 0, B, 0, P), SEED + 11)
    emit(config="C2-FT6D", op="prompt_layer_remap_FT6D_to_KV5D", bytes=nb, us=us, gbs_2R=2 * nb / us / 1e3,
         bound="hbm", frac=2 * nb / us / 1e3 / HBM, parity_mismatches=bad)
    del k6, v, dbuf, k5, v5, log
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C3,C4,C5,FT6D")
    a = ap.parse_args()
    for name in a.only.split(","):
        t0 = time.time()
        {"C1": c1, "C3": c3, "C4": c4, "C5": c5, "FT6D": ft6d}[name]()
        emit(config=name, op="wall_s", value=time.time() - t0)


if __name__ == "__main__":
    main()
