"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact.

Inputs come from kvgen only (numpy on the host side; the device fill kernel is itself pinned to
kvgen here). Expected values come from oracle/ only.
"""
import os
import random

import numpy as np
import pytest
import torch

import kvgen
import paper_2403_01876_b200 as dv
from oracle import kvstream as ok
from oracle import scenarios

from gpu_util import ctx, flags, pinned_u16, sentinel_like, to_dev, to_np, to_pinned

pytestmark = pytest.mark.gpu

XFERS = [dv.DV_XFER_FUSED, dv.DV_XFER_STAGED]


def dev_cache(K, V, lb, rb, pinned=False):
    k = to_pinned(K) if pinned else to_dev(K)
    v = to_pinned(V) if pinned else to_dev(V)
    return k, v, dv.cache(k, v, lb, rb)


def oc(K, V, lb, rb, S):
    return ok.Cache(K, V, lb, rb, K.shape[2], S, K.shape[4])


# ------------------------------------------------------------------------------------------------
def test_device_fill_matches_kvgen():
    """The device-side writer (dvt_fill) implements kvgen's generator bit-exactly."""
    L, B, H, S, D = 3, 2, 5, 24, 16
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    c = dv.cache(k, v, 7, 3)
    dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=kvgen.config_seed(1), valid=(2, 20))
    torch.cuda.synchronize()
    K, V = kvgen.kv5d_cache("hash", 7, L, 3, B, H, S, D, seed=kvgen.config_seed(1), valid_pos=(2, 20))
    assert np.array_equal(to_np(k), K) and np.array_equal(to_np(v), V)
    L, B, H, S, D = 2, 2, 2, 16, 16
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    c = dv.cache(k, v, 2, 1)
    box = (4, 3, H, S, D)
    dv.dvt_fill(c, dv.DVT_FILL_UID, box=box)
    torch.cuda.synchronize()
    K, V = kvgen.kv5d_cache("uid", 2, L, 1, B, H, S, D, box=box)
    assert np.array_equal(to_np(k), K) and np.array_equal(to_np(v), V)


# ------------------------------------------------------------------------------------------------
def _rand_case(rng):
    H = rng.choice([1, 3, 4, 8])
    D = rng.choice([8, 16, 64, 128])          # D*e in {16, 32, 128, 256} bytes
    nL, nR = rng.randint(1, 5), rng.randint(1, 4)
    S = rng.randint(2, 70)
    lb, rb = rng.randint(0, 9), rng.randint(0, 9)
    l0 = lb + rng.randint(0, nL - 1); l1 = rng.randint(l0 + 1, lb + nL)
    r0 = rb + rng.randint(0, nR - 1); r1 = rng.randint(r0 + 1, rb + nR)
    s0 = rng.randint(0, S - 1); s1 = rng.randint(s0 + 1, S)
    return H, D, nL, nR, S, lb, rb, (l0, l1, r0, r1, s0, s1)


@pytest.mark.parametrize("seed", range(24))
@pytest.mark.parametrize("xfer", XFERS)
@pytest.mark.parametrize("host", [False, True])
def test_scatter_gather_random_shapes(seed, xfer, host):
    """pack into a device/host endpoint == oracle.pack; unpack from it into a sentinel cache with
    another max_seq == oracle.unpack; bytes around the chunk in the endpoint stay untouched."""
    rng = random.Random(seed)
    H, D, nL, nR, S, lb, rb, reg = _rand_case(rng)
    K, V = kvgen.kv5d_cache("hash", lb, nL, rb, nR, H, S, D, seed=seed)
    k, v, c = dev_cache(K, V, lb, rb)
    wire_words = ok.region_bytes(*reg, H, D, 2) // 2
    pad = 64
    buf = pinned_u16(wire_words + 2 * pad) if host else sentinel_like((wire_words + 2 * pad,))
    ep = dv.endpoint_of(buf)
    ctx_ = ctx()
    dv.dv_scatter(ctx_, c, dv.region(*reg), ep, dst_off=pad * 2, xfer=xfer)
    torch.cuda.synchronize()
    got = to_np(buf)
    exp = ok.pack(oc(K, V, lb, rb, S), reg)
    assert np.array_equal(got[pad:pad + wire_words], exp)
    assert np.all(got[:pad] == kvgen.SENTINEL) and np.all(got[pad + wire_words:] == kvgen.SENTINEL)
    # gather into a destination with a different max_seq
    S2 = max(reg[5], S + rng.randint(-3, 9))
    dk = sentinel_like((nL, nR, H, S2, D))
    dvv = sentinel_like((nL, nR, H, S2, D))
    dc = dv.cache(dk, dvv, lb, rb)
    dv.dv_gather(ctx_, ep, pad * 2, dc, dv.region(*reg), xfer=xfer)
    torch.cuda.synchronize()
    o = oc(*kvgen.sentinel_cache(nL, nR, H, S2, D), lb, rb, S2)
    ok.unpack(o, reg, exp)
    assert np.array_equal(to_np(dk), o.K) and np.array_equal(to_np(dvv), o.V)


@pytest.mark.parametrize("seed", range(16))
@pytest.mark.parametrize("mode", ["dev-dev", "dev-host", "host-dev-fused", "host-dev-staged"])
def test_remap_random_shapes(seed, mode):
    """Direct layout-to-layout copy (different S, layer and request offsets) == oracle.remap."""
    rng = random.Random(100 + seed)
    H, D, nL, nR, S, lb, rb, reg = _rand_case(rng)
    K, V = kvgen.kv5d_cache("hash", lb, nL, rb, nR, H, S, D, seed=seed)
    src_host = mode.startswith("host")
    dst_host = mode == "dev-host"
    k, v, c = dev_cache(K, V, lb, rb, pinned=src_host)
    # destination holds a superset of the region's layers/requests at other offsets
    dlb, drb = reg[0] - rng.randint(0, 2), reg[2] - rng.randint(0, 2)
    dlb, drb = max(dlb, 0), max(drb, 0)
    dnL, dnR = reg[1] - dlb + rng.randint(0, 2), reg[3] - drb + rng.randint(0, 2)
    S2 = reg[5] + rng.randint(0, 20)
    dk = sentinel_like((dnL, dnR, H, S2, D), pinned=dst_host)
    dvv = sentinel_like((dnL, dnR, H, S2, D), pinned=dst_host)
    dc = dv.cache(dk, dvv, dlb, drb)
    xfer = dv.DV_XFER_STAGED if mode.endswith("staged") else dv.DV_XFER_FUSED
    dv.dv_remap(ctx(), c, dc, dv.region(*reg), xfer=xfer)
    torch.cuda.synchronize()
    o = oc(*kvgen.sentinel_cache(dnL, dnR, H, S2, D), dlb, drb, S2)
    ok.remap(oc(K, V, lb, rb, S), o, reg)
    assert np.array_equal(to_np(dk), o.K) and np.array_equal(to_np(dvv), o.V)
    assert np.array_equal(to_np(k), K) and np.array_equal(to_np(v), V)   # source untouched


# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("xfer", XFERS)
def test_c1_toy_round_trip_through_host(xfer):
    """C1 (BASELINE.json configs[0]): L2 H4 D16 b2, prompt 32 + 8 tokens, fp16. Prompt streamed out
    layer by layer to a pinned-host log, then 8 token steps; stream_in of [0,40) into a sentinel
    cache with S=64. uid fill: every word decodes to its coordinate; poison never crosses."""
    L, B, H, S, D, p, T = 2, 2, 4, 40, 16, 32, 8
    box = (L, B, H, S, D)
    K, V = kvgen.kv5d_cache("uid", 0, L, 0, B, H, S, D, box=box)
    k, v, c = dev_cache(K, V, 0, 0)
    one = dv.Setup([0, L], [0, B], S)
    big = dv.Setup([0, L], [0, B], 64)
    C = 2 * H * D * 2  # bytes per layer.token.request
    log = pinned_u16(L * B * (p + T) * C // 2)
    fl = flags(1, pinned=True)
    cx = ctx()
    # prompt, layer by layer (Opt 2): each layer's chunk appended to the log
    off = 0
    regions = [(l, l + 1, 0, B, 0, p) for l in range(L)] + \
              [(0, L, 0, B, ok.token_position(p, t), ok.token_position(p, t) + 1) for t in range(1, T + 1)]
    offs = []
    seq = 0
    for reg in regions:
        seq += 1
        ep = dv.endpoint_of(log, fl)
        dv.dv_scatter(cx, c, dv.region(*reg), ep, dst_off=off, flag_slot=0, seq=seq, xfer=xfer)
        offs.append(off)
        off += ok.region_bytes(*reg, H, D, 2)
    torch.cuda.synchronize()
    assert int(fl[0]) == seq and dv.dv_query(cx, dv.endpoint_of(log, fl), 0, seq)
    # oracle: the same sequence of chunks
    osrc = oc(K, V, 0, 0, S)
    exp_log = np.concatenate([ok.pack(osrc, reg) for reg in regions])
    assert np.array_equal(to_np(log)[:exp_log.size], exp_log)
    # stream back in (each chunk at its offset) into S=64
    dk = sentinel_like((L, B, H, 64, D)); dvv = sentinel_like((L, B, H, 64, D))
    dc = dv.cache(dk, dvv, 0, 0)
    for reg, o in zip(regions, offs):
        dv.dv_gather(cx, dv.endpoint_of(log, fl), o, dc, dv.region(*reg), flag_slot=0, wait_seq=seq, xfer=xfer)
    torch.cuda.synchronize()
    odst = oc(*kvgen.sentinel_cache(L, B, H, 64, D), 0, 0, 64)
    for reg, o in zip(regions, offs):
        ok.unpack(odst, reg, exp_log[o // 2:(o + ok.region_bytes(*reg, H, D, 2)) // 2])
    assert np.array_equal(to_np(dk), odst.K) and np.array_equal(to_np(dvv), odst.V)
    # independent of the oracle: every word decodes to its own coordinate (definition C-1)
    g = to_np(dk)[:, :, :, :40]
    kv_, l_, r_, h_, s_, d_ = kvgen.uid_decode(g, box)
    ll, rr, hh, ss, dd = np.meshgrid(*[np.arange(n) for n in g.shape], indexing="ij")
    assert np.all(kv_ == 0) and np.all(l_ == ll) and np.all(r_ == rr) and np.all(s_ == ss) and np.all(d_ == dd)
    assert np.all(to_np(dk)[:, :, :, 40:] == kvgen.SENTINEL)
    # level 1 form on the same data: stream_out -> host inbox, stream_in -> S=64 cache
    inbox = pinned_u16(L * B * (p + T) * C // 2)
    ifl = flags(1, pinned=True)
    iep = dv.endpoint_of(inbox, ifl)
    dv.dv_stream_out(cx, c, dv.region(0, L, 0, B, 0, p + T), one, 0, 0, big, [iep], seq=5, xfer=xfer)
    dk2 = sentinel_like((L, B, H, 64, D)); dv2 = sentinel_like((L, B, H, 64, D))
    dv.dv_stream_in(cx, dv.cache(dk2, dv2), dv.region(0, L, 0, B, 0, p + T), one, big, 0, 0, iep, 5, xfer=xfer)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(dk2), odst.K) and np.array_equal(to_np(dv2), odst.V)


def test_flag_orders_consumer_after_producer():
    """A5: the consumer's stream waits on the producer's seq flag. The producer is delayed by a
    2 ms spin on another stream; without the wait the gather would read the sentinel."""
    L, B, H, S, D = 2, 2, 4, 16, 16
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=5)
    k, v, c = dev_cache(K, V, 0, 0)
    reg = (0, L, 0, B, 0, S)
    nbytes = ok.region_bytes(*reg, H, D, 2)
    for host in (False, True):
        inbox = pinned_u16(nbytes // 2) if host else sentinel_like((nbytes // 2,))
        fl = flags(4, pinned=host)
        ep = dv.endpoint_of(inbox, fl)
        prod, cons = torch.cuda.Stream(), torch.cuda.Stream()
        cx = ctx()
        dk = sentinel_like((L, B, H, S, D)); dvv = sentinel_like((L, B, H, S, D))
        torch.cuda.synchronize()
        dv.dvt_spin(2_000_000, 1, stream=prod)
        dv.dv_scatter(cx, c, dv.region(*reg), ep, 0, flag_slot=2, seq=7, xfer=dv.DV_XFER_FUSED, stream=prod)
        dv.dv_gather(cx, ep, 0, dv.cache(dk, dvv), dv.region(*reg), flag_slot=2, wait_seq=7, stream=cons)
        torch.cuda.synchronize()
        assert np.array_equal(to_np(dk), K) and np.array_equal(to_np(dvv), V)
        assert int(fl[2]) == 7


def test_release_scope_follows_memory():
    """A5 publish protocol: gpu-scope release only when the flag AND the payload are
    this GPU's own HBM; pinned host on either side -> system scope. (Memory mapped from another
    process is checked in tests/mp_worker.py.)"""
    cx = ctx()
    d = torch.zeros(64, dtype=torch.int64, device="cuda")
    h = torch.zeros(64, dtype=torch.int64, pin_memory=True)
    raw = dv.dv_device_alloc(0, 4096)
    try:
        assert dv.dvt_release_scope(cx, d.data_ptr(), d.data_ptr() + 64)
        assert dv.dvt_release_scope(cx, raw, raw + 256)
        assert dv.dvt_release_scope(cx, d.data_ptr())            # flag only (empty payload)
        assert not dv.dvt_release_scope(cx, h.data_ptr(), d.data_ptr())
        assert not dv.dvt_release_scope(cx, d.data_ptr(), h.data_ptr())
        assert not dv.dvt_release_scope(cx, h.data_ptr(), h.data_ptr())
    finally:
        dv.dv_device_free(raw)


def test_staged_publish_and_fetch_flush():
    L, B, H, S, D = 1, 1, 2, 8, 16
    cx = ctx()
    src = torch.arange(4096, dtype=torch.int16, device="cuda")
    host = pinned_u16(4096 + 64)
    fl = flags(2, pinned=True)
    ep = dv.endpoint_of(host, fl)
    for xfer in XFERS:
        host.fill_(-1)
        dv.dv_flush(cx, src.data_ptr(), 8192, ep, dst_off=64, flag_slot=1, seq=3 + xfer, xfer=xfer)
        torch.cuda.synchronize()
        assert int(fl[1]) == 3 + xfer
        assert np.array_equal(to_np(host)[32:32 + 4096], np.arange(4096, dtype=np.uint16))
        back = torch.zeros(4096, dtype=torch.int16, device="cuda")
        dv.dv_fetch(cx, ep, 64, back.data_ptr(), 8192, flag_slot=1, wait_seq=3 + xfer, xfer=xfer)
        torch.cuda.synchronize()
        assert torch.equal(back, src)


# ------------------------------------------------------------------------------------------------
def _blocks(setup: ok.Setup):
    for i in range(setup.n_stages):
        for u in range(setup.n_micro):
            yield i, u, setup.layer_bounds[i], setup.layer_bounds[i + 1], setup.req_bounds[u], setup.req_bounds[u + 1]


@pytest.mark.parametrize("form", ["inbox-fused", "inbox-staged-host", "direct"])
@pytest.mark.parametrize("psplit,tsplit,preq,treq", [
    ([0, 16, 32, 48, 64], [0, 13, 30, 47, 64], [0, 4], [0, 4]),        # C3 partitions (7 pieces)
    ([0, 16, 32, 48, 64], [0, 13, 30, 47, 64], [0, 4], [0, 2, 4]),     # + batch split (14 pieces)
    ([0, 9, 18, 27, 36, 45, 54, 62, 70], [0, 35, 70], [0, 2, 4], [0, 4]),  # merge
])
def test_disaggregation_stream_out_in(form, psplit, tsplit, preq, treq):
    """C3 shape shrunk (H=3, D=16, p=12, S 16 -> 24), all blocks on one GPU: every prompt block
    calls dv_stream_out, every token block dv_stream_in; token caches == oracle.disaggregate."""
    H, D, p, Sp, St, seed = 3, 16, 12, 16, 24, 21
    ps, ts = ok.Setup(psplit, preq, Sp), ok.Setup(tsplit, treq, St)
    dps, dts = dv.Setup(psplit, preq, Sp), dv.Setup(tsplit, treq, St)
    prompt, oprompt = {}, {}
    for i, u, a, b, c0, c1 in _blocks(ps):
        K, V = kvgen.kv5d_cache("hash", a, b - a, c0, c1 - c0, H, Sp, D, seed=seed, valid_pos=(0, p))
        prompt[(i, u)] = dev_cache(K, V, a, c0)
        oprompt[(i, u)] = oc(K, V, a, c0, Sp)
    token, otoken = {}, {}
    for j, w, a, b, c0, c1 in _blocks(ts):
        k = sentinel_like((b - a, c1 - c0, H, St, D)); v = sentinel_like((b - a, c1 - c0, H, St, D))
        token[(j, w)] = (k, v, dv.cache(k, v, a, c0))
        otoken[(j, w)] = oc(*kvgen.sentinel_cache(b - a, c1 - c0, H, St, D), a, c0, St)
    reg = dv.region(psplit[0], psplit[-1], preq[0], preq[-1], 0, p)
    cx = ctx()
    nblk_t = ts.n_stages * ts.n_micro
    if form == "direct":
        dcs = [token[(j, w)][2] for j, w, *_ in _blocks(ts)]
        nblk_p = ps.n_stages * ps.n_micro
        sigf = flags(nblk_t * nblk_p)
        sig = [dv.endpoint_of(sigf[:1], sigf[k * nblk_p:(k + 1) * nblk_p]) for k in range(nblk_t)]
        for (i, u), (_, _, c) in prompt.items():
            dv.dv_stream_out_direct(cx, c, reg, dps, i, u, dts, dcs, sig, seq=1)
    else:
        host = form.endswith("host")
        xfer = dv.DV_XFER_STAGED if "staged" in form else dv.DV_XFER_FUSED
        inb, eps = {}, []
        for j, w, a, b, c0, c1 in _blocks(ts):
            words = (b - a) * (c1 - c0) * H * p * D * 2
            buf = pinned_u16(words) if host else sentinel_like((words,))
            fl = flags(ps.n_stages * ps.n_micro, pinned=host)
            inb[(j, w)] = (buf, fl)
            eps.append(dv.endpoint_of(buf, fl))
        for (i, u), (_, _, c) in prompt.items():
            dv.dv_stream_out(cx, c, reg, dps, i, u, dts, eps, seq=1, xfer=xfer)
        for k_, (j, w, *_r) in enumerate(_blocks(ts)):
            dv.dv_stream_in(cx, token[(j, w)][2], reg, dps, dts, j, w, eps[k_], 1, xfer=xfer)
    torch.cuda.synchronize()
    scenarios.disaggregate(oprompt, ps, otoken, ts, p)
    for key, (k, v, _) in token.items():
        assert np.array_equal(to_np(k), otoken[key].K) and np.array_equal(to_np(v), otoken[key].V), key


def test_validation_has_no_partial_effect():
    """An invalid piece anywhere in a stream_out rejects the whole call before anything is
    enqueued (DESIGN.md conventions): the first inbox stays untouched."""
    H, D, p, S = 2, 16, 4, 8
    K, V = kvgen.kv5d_cache("hash", 0, 4, 0, 2, H, S, D, seed=3)
    k, v, c = dev_cache(K, V, 0, 0)
    src_s, dst_s = dv.Setup([0, 4], [0, 2], S), dv.Setup([0, 2, 4], [0, 2], S)
    good = sentinel_like((2 * 2 * H * p * D * 2,))
    small = sentinel_like((16,))
    eps = [dv.endpoint_of(good, flags(1)), dv.endpoint_of(small, flags(1))]
    with pytest.raises(dv.DVError) as ei:
        dv.dv_stream_out(ctx(), c, dv.region(0, 4, 0, 2, 0, p), src_s, 0, 0, dst_s, eps, seq=1)
    assert ei.value.status == dv.DV_EINVAL
    torch.cuda.synchronize()
    assert np.all(to_np(good) == kvgen.SENTINEL)
    with pytest.raises(dv.DVError) as ei:
        dv.dv_scatter(ctx(), c, dv.region(0, 4, 0, 2, 0, S + 1), eps[0])
    assert ei.value.status == dv.DV_ERANGE and "max_seq 8" in str(ei.value)
    with pytest.raises(dv.DVError) as ei:
        dv.dv_scatter(ctx(), c, dv.region(0, 5, 0, 2, 0, 2), eps[0])
    assert ei.value.status == dv.DV_EMAP
    bad = dv.cache(k, v, 0, 0)
    bad.head_dim = 12  # 24 bytes per row: not a multiple of 16
    with pytest.raises(dv.DVError) as ei:
        dv.dv_scatter(ctx(), bad, dv.region(0, 1, 0, 1, 0, 1), eps[0])
    assert ei.value.status == dv.DV_EALIGN


def test_empty_regions_are_noops_that_still_publish():
    H, D, S = 2, 16, 8
    K, V = kvgen.kv5d_cache("hash", 0, 2, 0, 2, H, S, D, seed=3)
    k, v, c = dev_cache(K, V, 0, 0)
    buf = sentinel_like((64,))
    fl = flags(1)
    dv.dv_scatter(ctx(), c, dv.region(0, 2, 0, 2, 3, 3), dv.endpoint_of(buf, fl), flag_slot=0, seq=9)
    torch.cuda.synchronize()
    assert int(fl[0]) == 9 and np.all(to_np(buf) == kvgen.SENTINEL)


# ------------------------------------------------------------------------------------------------
def _write_token_dev(c: dv.dv_cache, pos, seed):
    reg = dv.region(c.layer_begin, c.layer_begin + c.n_layers, c.req_begin, c.req_begin + c.n_reqs, pos, pos + 1)
    dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=seed, reg=reg)


@pytest.mark.parametrize("depth,rounds,xfer", [(3, 2, dv.DV_XFER_FUSED), (4, 2, dv.DV_XFER_STAGED), (5, 1, dv.DV_XFER_FUSED)])
def test_swap_rotation_matches_oracle(depth, rounds, xfer):
    """C4 shape shrunk: one stage, D microbatches with pinned-host mirror arenas, two device slots;
    rotation of PAPER.md:272 driven through dv_remap (swap-in: whole prefix host->slot; swap-out:
    the step's position slot->host). Final arenas and slots == oracle.swap_simulate."""
    L0, nL, b, H, S, D, p, seed = 9, 2, 2, 4, 24, 16, 6, 77
    host_np, host_t = {}, {}
    for x in range(depth):
        K, V = kvgen.kv5d_cache("hash", L0, nL, x * b, b, H, S, D, seed=seed, valid_pos=(0, p))
        K[:, :, :, p:] = kvgen.SENTINEL
        V[:, :, :, p:] = kvgen.SENTINEL
        host_np[x] = oc(K, V, L0, x * b, S)
        host_t[x] = (to_pinned(K), to_pinned(V))
    slots_t = [(sentinel_like((nL, b, H, S, D)), sentinel_like((nL, b, H, S, D))) for _ in range(2)]
    cx = ctx()

    def hc(x):
        return dv.cache(host_t[x][0], host_t[x][1], L0, x * b)

    def sc(s, x):
        return dv.cache(slots_t[s][0], slots_t[s][1], L0, x * b)

    # --- GPU driver of the rotation (independent of the oracle's loop) ---
    length = {x: p for x in range(depth)}
    slot_of = {0: 0}
    dv.dv_remap(cx, hc(0), sc(0, 0), dv.region(L0, L0 + nL, 0, b, 0, p), xfer=xfer)
    done = {x: 0 for x in range(depth)}
    for t in range(1, rounds + 1):
        for x in range(depth):
            xin, xout = (x + 1) % depth, (x - 1) % depth
            pos = p + t - 1
            _write_token_dev(sc(slot_of[x], x), pos, seed)
            done[x] += 1
            length[x] = p + done[x]
            if done[xout] > 0 and xout in slot_of:
                q = length[xout] - 1
                dv.dv_remap(cx, sc(slot_of[xout], xout), hc(xout),
                            dv.region(L0, L0 + nL, xout * b, xout * b + b, q, q + 1), xfer=xfer)
                free = slot_of.pop(xout)
            else:
                free = 1 - slot_of[x]
            if not (t == rounds and x == depth - 1):
                dv.dv_remap(cx, hc(xin), sc(free, xin), dv.region(L0, L0 + nL, xin * b, xin * b + b, 0, length[xin]),
                            xfer=xfer)
                slot_of[xin] = free
    last = depth - 1
    q = length[last] - 1
    dv.dv_remap(cx, sc(slot_of[last], last), hc(last), dv.region(L0, L0 + nL, last * b, last * b + b, q, q + 1), xfer=xfer)
    torch.cuda.synchronize()

    oslots = [oc(*kvgen.sentinel_cache(nL, b, H, S, D), L0, 0, S) for _ in range(2)]

    def write(cache, x, pos):
        for kv in (0, 1):
            blk = kvgen.logical_block("hash", kv, range(L0, L0 + nL), range(cache.req_begin, cache.req_begin + b),
                                      H, [pos], D, seed)
            cache.set_logical(kv, L0, L0 + nL, cache.req_begin, cache.req_begin + b, pos, pos + 1, blk)
    scenarios.swap_simulate(host_np, oslots, p, rounds, write)
    for x in range(depth):
        assert np.array_equal(to_np(host_t[x][0]), host_np[x].K) and np.array_equal(to_np(host_t[x][1]), host_np[x].V)
    for s in range(2):
        assert np.array_equal(to_np(slots_t[s][0]), oslots[s].K) and np.array_equal(to_np(slots_t[s][1]), oslots[s].V)


@pytest.mark.parametrize("P", [2, 4])
def test_ring_replication_and_recovery_loopback(P):
    """C5 shape shrunk, P stages on one GPU (loopback peers): prompt replica then per-token
    stream_out_direct into the replica store at (x+1)%P with seq flags; then recovery of stage 1.
    Replicas and restored caches == oracle (scenarios.ring_step / recover)."""
    Ls, b, H, S, D, p, T, seed = 2, 3, 4, 20, 16, 7, 4, 91
    L = Ls * P
    setup = dv.Setup([x * Ls for x in range(P + 1)], [0, b], S)
    own, rep, oown, orep = {}, {}, {}, {}
    for x in range(P):
        K, V = kvgen.kv5d_cache("hash", x * Ls, Ls, 0, b, H, S, D, seed=seed, valid_pos=(0, p))
        own[x] = dev_cache(K, V, x * Ls, 0)
        oown[x] = oc(K, V, x * Ls, 0, S)
        px = (x - 1) % P
        rk, rv = sentinel_like((Ls, b, H, S, D)), sentinel_like((Ls, b, H, S, D))
        rep[x] = (rk, rv, dv.cache(rk, rv, px * Ls, 0))
        orep[x] = oc(*kvgen.sentinel_cache(Ls, b, H, S, D), px * Ls, 0, S)
    sigf = flags(P * P)
    sig = [dv.endpoint_of(sigf[:1], sigf[y * P:(y + 1) * P]) for y in range(P)]
    cx = ctx()

    def replicate(reg_of, seq):
        for x in range(P):
            y = (x + 1) % P
            # destination "setup" of the replica store: replica[y] holds stage x's layers
            dcs = [None] * P
            dcs[x] = rep[y][2]
            dsig = [None] * P
            dsig[x] = sig[y]
            dv.dv_stream_out_direct(cx, own[x][2], dv.region(*reg_of(x)), setup, x, 0, setup, dcs, dsig, seq=seq)

    replicate(lambda x: (x * Ls, x * Ls + Ls, 0, b, 0, p), 1)
    scenarios.ring_step(oown, orep, lambda x: (x * Ls, x * Ls + Ls, 0, b, 0, p))
    for t in range(1, T + 1):
        q = p + t - 1
        for x in range(P):
            _write_token_dev(own[x][2], q, seed)
            blkK = kvgen.logical_block("hash", 0, range(x * Ls, x * Ls + Ls), range(b), H, [q], D, seed)
            blkV = kvgen.logical_block("hash", 1, range(x * Ls, x * Ls + Ls), range(b), H, [q], D, seed)
            oown[x].set_logical(0, x * Ls, x * Ls + Ls, 0, b, q, q + 1, blkK)
            oown[x].set_logical(1, x * Ls, x * Ls + Ls, 0, b, q, q + 1, blkV)
        replicate(lambda x: (x * Ls, x * Ls + Ls, 0, b, q, q + 1), 1 + t)
        scenarios.ring_step(oown, orep, lambda x: (x * Ls, x * Ls + Ls, 0, b, q, q + 1))
    torch.cuda.synchronize()
    for y in range(P):
        assert np.array_equal(to_np(rep[y][0]), orep[y].K) and np.array_equal(to_np(rep[y][1]), orep[y].V)
        x = (y - 1) % P
        assert int(sigf[y * P + x]) == 1 + T   # the seq plays the (x, j, t) ack role
    # failure of stage 1: wipe its cache and the replica it hosts, then the two recovery copies
    own[1][0].fill_(-1); own[1][1].fill_(-1); rep[1][0].fill_(-1); rep[1][1].fill_(-1)
    for a in (oown[1].K, oown[1].V, orep[1].K, orep[1].V):
        a[...] = kvgen.SENTINEL
    n = p + T
    a_, b_ = (1 + 1) % P, (1 - 1) % P
    dv.dv_remap(cx, rep[a_][2], own[1][2], dv.region(Ls, 2 * Ls, 0, b, 0, n))
    dv.dv_remap(cx, own[b_][2], rep[1][2], dv.region(b_ * Ls, b_ * Ls + Ls, 0, b, 0, n))
    torch.cuda.synchronize()
    scenarios.recover(1, oown, orep, n)
    assert np.array_equal(to_np(own[1][0]), oown[1].K) and np.array_equal(to_np(own[1][1]), oown[1].V)
    assert np.array_equal(to_np(rep[1][0]), orep[1].K) and np.array_equal(to_np(rep[1][1]), orep[1].V)


def test_paper_baselines_produce_the_wire():
    """The prior-art baselines (per-run copies, 2-D buffered copies) produce the same wire chunk."""
    H, D, nL, nR, S = 4, 16, 3, 2, 20
    K, V = kvgen.kv5d_cache("hash", 0, nL, 0, nR, H, S, D, seed=8)
    k, v, c = dev_cache(K, V, 0, 0)
    reg = (0, nL, 0, nR, 5, 11)
    exp = ok.pack(oc(K, V, 0, 0, S), reg)
    out = sentinel_like((exp.size,))
    calls = dv.dvb_per_run_copy(c, dv.region(*reg), out.data_ptr())
    torch.cuda.synchronize()
    assert calls == 2 * nL * nR * H and np.array_equal(to_np(out), exp)
    out.fill_(-1)
    stg = torch.empty(exp.size, dtype=torch.int16, device="cuda")
    calls = dv.dvb_buffered_copy(c, dv.region(*reg), stg.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    assert calls == 2 * nL * nR + 1 and np.array_equal(to_np(out), exp)


@pytest.mark.parametrize("xfer,npos", [(dv.DV_XFER_FUSED, 1), (dv.DV_XFER_FUSED | dv.DV_PUBLISH_STREAMOP, 1),
                                       (dv.DV_XFER_STAGED, 1), (dv.DV_XFER_DECOUPLED, 1),
                                       (dv.DV_XFER_FUSED, 24)])
def test_host_poller_never_sees_flag_before_payload(xfer, npos):
    """Release protocol (A5) observed from the CPU: a host thread spins on the pinned flag while
    the GPU streams 300 per-layer chunks; whenever it sees seq k it immediately compares chunk k
    with the oracle. A flag visible before its payload would show up as a mismatch. npos = 24:
    768 KiB chunks written by 192 CTAs, so the one system-scope release of the last CTA must
    cover every other CTA's PCIe stores (cumulativity, DESIGN.md §6 protocol 2)."""
    import threading
    L, B, H, S, D = 4, 8, 8, 64, 128
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=12)
    k, v, c = dev_cache(K, V, 0, 0)
    osrc = oc(K, V, 0, 0, S)
    n = 300
    regs = [(i % L, i % L + 1, 0, B, (i * npos) % (S - npos), (i * npos) % (S - npos) + npos) for i in range(n)]
    chunk = ok.region_bytes(*regs[0], H, D, 2)
    exp = [ok.pack(osrc, r) for r in regs]
    log = pinned_u16(n * chunk // 2)
    fl = flags(1, pinned=True)
    ep = dv.endpoint_of(log, fl)
    lnp = log.numpy().view(np.uint16)
    fnp = fl.numpy()
    bad, seen = [], []
    stop = threading.Event()

    def poll():
        last = 0
        while not stop.is_set() or last < n:
            cur = int(fnp[0])
            if cur > last:
                i = cur - 1
                if not np.array_equal(lnp[i * chunk // 2:(i + 1) * chunk // 2], exp[i]):
                    bad.append(i)
                seen.append(cur)
                last = cur
            if stop.is_set() and cur >= n:
                break
    th = threading.Thread(target=poll, daemon=True)   # daemon: a failing test must not hang pytest
    th.start()
    try:
        cx = ctx()
        for i, r in enumerate(regs):
            dv.dvt_spin(3000, 1)   # spread the chunks out so the poller samples many of them
            dv.dv_scatter(cx, c, dv.region(*r), ep, i * chunk, flag_slot=0, seq=i + 1, xfer=xfer)
        torch.cuda.synchronize()
    finally:
        stop.set()
        th.join(timeout=60)
    assert not th.is_alive(), "poller never saw the last flag"
    assert not bad, f"flag seen before payload for chunks {bad[:10]}"
    assert len(seen) > 10 and seen[-1] == n


@pytest.mark.parametrize("big", [False, True])
def test_decoupled_scatter_flag_is_completion_and_source_is_free(big):
    """DV_XFER_DECOUPLED (stream_out is non-blocking): the caller's stream is only
    ordered after the pack, so rewriting the source right after the call must not change what
    lands in the host log; the flag (waited on by a consumer stream) is the completion signal.
    big: a region >= 32 MB (pipelined chunks on the DMA stream)."""
    L, B, H, S, D = (4, 8, 16, 160, 128) if big else (4, 4, 8, 64, 128)
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=31)
    k, v, c = dev_cache(K, V, 0, 0)
    osrc = oc(K, V, 0, 0, S)
    regs = [(0, L, 0, B, 0, S)] if big else [(0, L, 0, B, q, q + 1) for q in range(12)] + [(1, 3, 1, 4, 20, 50)]
    sizes = [ok.region_bytes(*r, H, D, 2) for r in regs]
    offs = np.cumsum([0] + sizes)
    log = pinned_u16(int(offs[-1]) // 2 + 8)
    log.fill_(-1)
    fl = flags(1, pinned=True)
    ep = dv.endpoint_of(log, fl)
    cx = ctx()
    for i, r in enumerate(regs):
        dv.dv_scatter(cx, c, dv.region(*r), ep, int(offs[i]), flag_slot=0, seq=i + 1, xfer=dv.DV_XFER_DECOUPLED)
        # the caller's stream may rewrite the source at once (different seed)
        dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=1000 + i, reg=dv.region(*r))
    cons = torch.cuda.Stream()
    dv.dv_wait(cx, ep, 0, len(regs), stream=cons.cuda_stream)
    cons.synchronize()
    assert int(fl[0]) == len(regs)
    got = log.numpy().view(np.uint16)
    for i, r in enumerate(regs):
        assert np.array_equal(got[offs[i] // 2:offs[i + 1] // 2], ok.pack(osrc, r)), i
    torch.cuda.synchronize()
    with pytest.raises(dv.DVError) as e:   # the flag is the only completion signal: required
        dv.dv_scatter(cx, c, dv.region(*regs[0]), ep, 0, flag_slot=-1, xfer=dv.DV_XFER_DECOUPLED)
    assert e.value.status == dv.DV_EINVAL


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("xfer", XFERS)
@pytest.mark.parametrize("host", [False, True])
def test_gather_chunks_matches_oracle(seed, xfer, host):
    """dv_gather_chunks (log of chunks -> cache in one go) == oracle.unpack_chunks."""
    rng = random.Random(500 + seed)
    H, D, nL, nR, S, lb, rb, reg = _rand_case(rng)
    S = max(S, 8)
    n = rng.randint(1, 3)
    step = n + rng.randint(0, 2)
    n_chunks = max(1, (S - n) // step)
    first = (reg[0], reg[1], reg[2], reg[3], 0, n)
    K, V = kvgen.kv5d_cache("hash", lb, nL, rb, nR, H, S, D, seed=seed)
    osrc = oc(K, V, lb, rb, S)
    log_np = np.concatenate([ok.pack(osrc, ok.shifted(first, k * step)) for k in range(n_chunks)])
    log = to_pinned(log_np) if host else to_dev(log_np)
    dk = sentinel_like((nL, nR, H, S, D)); dvv = sentinel_like((nL, nR, H, S, D))
    dv.dv_gather_chunks(ctx(), dv.endpoint_of(log), 0, dv.cache(dk, dvv, lb, rb), dv.region(*first), n_chunks, step,
                        xfer=xfer)
    torch.cuda.synchronize()
    o = oc(*kvgen.sentinel_cache(nL, nR, H, S, D), lb, rb, S)
    ok.unpack_chunks(o, first, log_np, n_chunks, step)
    assert np.array_equal(to_np(dk), o.K) and np.array_equal(to_np(dvv), o.V)


def test_swap_log_form_round_trip():
    """C4 log form end to end: prompt chunk + per-token delta chunks appended to a pinned host
    log by dv_scatter (swap-out), then one dv_gather_chunks + one dv_gather (swap-in) rebuild the
    microbatch in an empty slot == the source on [0, p+T)."""
    L, b, H, S, D, p, T = 3, 4, 8, 64, 128, 20, 30
    K, V = kvgen.kv5d_cache("hash", 9, L, 8, b, H, S, D, seed=31)
    k, v, c = dev_cache(K, V, 9, 8)
    C = 2 * L * b * H * D * 2
    log = pinned_u16((p + T) * C // 2)
    fl = flags(1, pinned=True)
    ep = dv.endpoint_of(log, fl)
    cx = ctx()
    dv.dv_scatter(cx, c, dv.region(9, 9 + L, 8, 8 + b, 0, p), ep, 0, flag_slot=0, seq=1)
    for t in range(T):
        dv.dv_scatter(cx, c, dv.region(9, 9 + L, 8, 8 + b, p + t, p + t + 1), ep, (p + t) * C, flag_slot=0,
                      seq=2 + t)
    sk = sentinel_like((L, b, H, S, D)); sv = sentinel_like((L, b, H, S, D))
    sc = dv.cache(sk, sv, 9, 8)
    dv.dv_gather(cx, ep, 0, sc, dv.region(9, 9 + L, 8, 8 + b, 0, p), flag_slot=0, wait_seq=1 + T)
    dv.dv_gather_chunks(cx, ep, p * C, sc, dv.region(9, 9 + L, 8, 8 + b, p, p + 1), T, 1, flag_slot=0,
                        wait_seq=1 + T)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(sk)[:, :, :, :p + T], K[:, :, :, :p + T])
    assert np.array_equal(to_np(sv)[:, :, :, :p + T], V[:, :, :, :p + T])
    assert np.all(to_np(sk)[:, :, :, p + T:] == kvgen.SENTINEL)



# ------------------------------------------------------------------------------------------------
# NEXT-1: FasterTransformer 6-D key layout;  NEXT-4: tensor-parallel head re-split
# ------------------------------------------------------------------------------------------------
def _mk(K, V, lb, rb, layout, pinned=False, hb=0):
    """Device (or pinned) cache from logical K, V in the requested layout + its oracle twin."""
    S, D = K.shape[3], K.shape[4]
    Kp = kvgen.as_ft6d_key(K) if layout == ok.LAYOUT_FT6D else K
    k = to_pinned(Kp) if pinned else to_dev(Kp)
    v = to_pinned(V) if pinned else to_dev(V)
    o = ok.Cache(Kp.copy(), V.copy(), lb, rb, K.shape[2], S, D, layout, hb)
    return k, v, dv.cache(k, v, lb, rb, head_begin=hb), o


def test_device_fill_ft6d_with_head_offset():
    L, B, H, S, D, hb = 2, 3, 4, 12, 64, 5
    K, V = kvgen.kv5d_cache("hash", 3, L, 1, B, H, S, D, seed=17, head_begin=hb, valid_pos=(1, 10))
    k = torch.empty(kvgen.as_ft6d_key(K).shape, dtype=torch.int16, device="cuda")
    v = torch.empty(V.shape, dtype=torch.int16, device="cuda")
    dv.dvt_fill(dv.cache(k, v, 3, 1, head_begin=hb), dv.DVT_FILL_HASH, seed=17, valid=(1, 10))
    torch.cuda.synchronize()
    assert np.array_equal(to_np(k), kvgen.as_ft6d_key(K)) and np.array_equal(to_np(v), V)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("layouts", [(ok.LAYOUT_FT6D, ok.LAYOUT_KV5D), (ok.LAYOUT_KV5D, ok.LAYOUT_FT6D),
                                     (ok.LAYOUT_FT6D, ok.LAYOUT_FT6D)])
@pytest.mark.parametrize("xfer", XFERS)
def test_ft6d_pack_unpack_remap(seed, layouts, xfer):
    """Pack from a cache in one layout, unpack into a cache in the other (and remap directly),
    with head sub-ranges; == the oracle (whose FT6D offset function is pinned on CPU)."""
    rng = random.Random(900 + seed)
    H, D = rng.choice([2, 3, 5]), rng.choice([16, 64, 128])
    nL, nR, S = rng.randint(1, 3), rng.randint(1, 3), rng.randint(2, 40)
    hb = rng.randint(0, 4)
    s0 = rng.randint(0, S - 1); s1 = rng.randint(s0 + 1, S)
    h0 = hb + rng.randint(0, H - 1); h1 = rng.randint(h0 + 1, hb + H)
    reg = (0, nL, 0, nR, s0, s1, h0, h1)
    K, V = kvgen.kv5d_cache("hash", 0, nL, 0, nR, H, S, D, seed=seed, head_begin=hb)
    k, v, c, o = _mk(K, V, 0, 0, layouts[0], hb=hb)
    exp = ok.pack(o, reg)
    buf = sentinel_like((exp.size,), pinned=(xfer == dv.DV_XFER_STAGED))
    dv.dv_scatter(ctx(), c, dv.region(*reg), dv.endpoint_of(buf), xfer=xfer)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(buf), exp)
    S2 = s1 + rng.randint(0, 5)
    Ks, Vs = kvgen.sentinel_cache(nL, nR, H, S2, D)
    dk, dvv, dc, do = _mk(Ks, Vs, 0, 0, layouts[1], hb=hb)
    dv.dv_gather(ctx(), dv.endpoint_of(buf), 0, dc, dv.region(*reg), xfer=xfer)
    torch.cuda.synchronize()
    ok.unpack(do, reg, exp)
    assert np.array_equal(to_np(dk), do.K) and np.array_equal(to_np(dvv), do.V)
    ek, ev, ec, eo = _mk(Ks, Vs, 0, 0, layouts[1], hb=hb)
    dv.dv_remap(ctx(), c, ec, dv.region(*reg))
    torch.cuda.synchronize()
    ok.remap(o, eo, reg)
    assert np.array_equal(to_np(ek), eo.K) and np.array_equal(to_np(ev), eo.V)


@pytest.mark.parametrize("D", [8, 40, 80, 96, 128, 256])
@pytest.mark.parametrize("layouts", [(ok.LAYOUT_FT6D, ok.LAYOUT_KV5D), (ok.LAYOUT_KV5D, ok.LAYOUT_FT6D)])
def test_ft6d_transpose_every_packet_group(D, layouts):
    """The register packet transpose (taken for regions of >= 32 positions) at every packet-group
    size PK the head dim allows: D = 8 (1 packet), 40 (5: PK 1), 80 (10: PK 2), 96 (12: PK 4),
    128 (16: PK 16), 256 (32: two PK-16 groups); pack, unpack and remap == the oracle."""
    H, nL, nR, S, hb = 3, 2, 2, 70, 1
    reg = (0, nL, 0, nR, 3, 67, 0, 0)
    K, V = kvgen.kv5d_cache("hash", 0, nL, 0, nR, H, S, D, seed=D, head_begin=hb)
    k, v, c, o = _mk(K, V, 0, 0, layouts[0], hb=hb)
    exp = ok.pack(o, reg)
    buf = sentinel_like((exp.size,))
    dv.dv_scatter(ctx(), c, dv.region(*reg), dv.endpoint_of(buf))
    torch.cuda.synchronize()
    assert np.array_equal(to_np(buf), exp)
    Ks, Vs = kvgen.sentinel_cache(nL, nR, H, S + 3, D)
    dk, dvv, dc, do = _mk(Ks, Vs, 0, 0, layouts[1], hb=hb)
    dv.dv_gather(ctx(), dv.endpoint_of(buf), 0, dc, dv.region(*reg))
    torch.cuda.synchronize()
    ok.unpack(do, reg, exp)
    assert np.array_equal(to_np(dk), do.K) and np.array_equal(to_np(dvv), do.V)
    ek, ev, ec, eo = _mk(Ks, Vs, 0, 0, layouts[1], hb=hb)
    dv.dv_remap(ctx(), c, ec, dv.region(*reg))
    torch.cuda.synchronize()
    ok.remap(o, eo, reg)
    assert np.array_equal(to_np(ek), eo.K) and np.array_equal(to_np(ev), eo.V)


@pytest.mark.parametrize("sh,th", [([0, 6], [0, 3, 6]), ([0, 2, 4, 6], [0, 3, 6]), ([0, 3, 6], [0, 1, 2, 3, 4, 5, 6])])
@pytest.mark.parametrize("direct", [False, True])
def test_tp_resplit_stream_out_in(sh, th, direct):
    """NEXT-4: prompt and token pipelines with different TP degrees (and layer splits): every
    prompt block (stage, micro, tp) streams out, every token block streams in; == oracle.stream."""
    H, D, p, S, seed = 6, 16, 7, 12, 43
    ps, ts = ok.Setup([0, 2, 4], [0, 2], S, sh), ok.Setup([0, 3, 4], [0, 2], S, th)
    dps, dts = dv.Setup([0, 2, 4], [0, 2], S, sh), dv.Setup([0, 3, 4], [0, 2], S, th)
    prompt, oprompt, token, otoken = {}, {}, {}, {}
    for i in range(ps.n_stages):
        for t in range(ps.n_tp):
            a, b, h0, h1 = ps.layer_bounds[i], ps.layer_bounds[i + 1], sh[t], sh[t + 1]
            K, V = kvgen.kv5d_cache("hash", a, b - a, 0, 2, h1 - h0, S, D, seed=seed, head_begin=h0)
            k, v, c, o = _mk(K, V, a, 0, ok.LAYOUT_KV5D, hb=h0)
            prompt[(i, 0, t)] = (k, v, c)
            oprompt[(i, 0, t)] = o
    for j in range(ts.n_stages):
        for t in range(ts.n_tp):
            a, b, h0, h1 = ts.layer_bounds[j], ts.layer_bounds[j + 1], th[t], th[t + 1]
            Ks, Vs = kvgen.sentinel_cache(b - a, 2, h1 - h0, S, D)
            k, v, c, o = _mk(Ks, Vs, a, 0, ok.LAYOUT_KV5D, hb=h0)
            token[(j, 0, t)] = (k, v, c)
            otoken[(j, 0, t)] = o
    reg = dv.region(0, 4, 0, 2, 0, p)
    cx = ctx()
    keys_t = sorted(token, key=lambda x: dts.flat(*x))
    if direct:
        dcs = [token[kk][2] for kk in keys_t]
        for (i, u, t), (_, _, c) in prompt.items():
            dv.dv_stream_out_direct(cx, c, reg, dps, i, u, dts, dcs, None, seq=1, my_tp=t)
    else:
        eps, keep = [], []
        for kk in keys_t:
            c = token[kk][2]
            buf = sentinel_like((c.n_layers * 2 * c.n_heads * p * D * 2,))
            fl = flags(ps.n_stages * ps.n_micro * ps.n_tp)
            keep += [buf, fl]          # endpoints hold raw pointers: keep the tensors alive
            eps.append(dv.endpoint_of(buf, fl))
        for (i, u, t), (_, _, c) in prompt.items():
            dv.dv_stream_out(cx, c, reg, dps, i, u, dts, eps, seq=1, my_tp=t)
        for n_, kk in enumerate(keys_t):
            dv.dv_stream_in(cx, token[kk][2], reg, dps, dts, kk[0], kk[1], eps[n_], 1, my_tp=kk[2])
    torch.cuda.synchronize()
    ok.stream(oprompt, ps, otoken, ts, (0, 4, 0, 2, 0, p))
    for kk, (k, v, _) in token.items():
        assert np.array_equal(to_np(k), otoken[kk].K) and np.array_equal(to_np(v), otoken[kk].V), kk


# ------------------------------------------------------------------------------------------------
# CUDA graphs: capture the per-token stream-out once, replay it with a device-side step counter
# ------------------------------------------------------------------------------------------------
def test_scatter_dyn_graph_replay_matches_oracle():
    L, B, H, S, D, p, T = 3, 2, 4, 24, 64, 10, 8
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=61)
    k, v, c = dev_cache(K, V, 0, 0)
    osrc = oc(K, V, 0, 0, S)
    chunk = ok.region_bytes(0, L, 0, B, p, p + 1, H, D, 2)
    log = pinned_u16((T + 2) * chunk // 2)
    fl = flags(1, pinned=True)
    ep = dv.endpoint_of(log, fl)
    d_step = torch.zeros(1, dtype=torch.int32, device="cuda")
    cx = ctx()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            dv.dv_scatter_dyn(cx, c, dv.region(0, L, 0, B, p, p + 1), ep, chunk, chunk, d_step.data_ptr(), T - 1,
                              flag_slot=0, seq=100)
    torch.cuda.synchronize()
    for t in range(T):
        with torch.cuda.stream(s):
            d_step.fill_(t)
            g.replay()
        torch.cuda.synchronize()
        assert int(fl[0]) == 100 + t
    got = to_np(log)
    for t in range(T):
        exp = ok.pack(osrc, (0, L, 0, B, p + t, p + t + 1))
        assert np.array_equal(got[(1 + t) * chunk // 2:(2 + t) * chunk // 2], exp)
    assert np.all(got[:chunk // 2] == kvgen.SENTINEL)
    # a step outside [0, max_step] is a no-op: nothing moves, nothing is published
    with torch.cuda.stream(s):
        d_step.fill_(T)
        g.replay()
    torch.cuda.synchronize()
    assert int(fl[0]) == 100 + T - 1
    assert np.all(to_np(log)[(1 + T) * chunk // 2:] == kvgen.SENTINEL)
    with pytest.raises(dv.DVError) as ei:   # validated for every step up to max_step
        dv.dv_scatter_dyn(cx, c, dv.region(0, L, 0, B, p, p + 1), ep, chunk, chunk, d_step.data_ptr(), S - p)
    assert ei.value.status == dv.DV_ERANGE


@pytest.mark.parametrize("dst_layout", [ok.LAYOUT_KV5D, ok.LAYOUT_FT6D])
def test_remap_dyn_graph_ring_step(dst_layout):
    """Per-token ring replication (C5) as one captured graph: remap position p+k of every layer into
    the replica store (another layout allowed) and publish seq+k."""
    L, B, H, S, D, p, T = 2, 3, 2, 20, 16, 5, 6
    K, V = kvgen.kv5d_cache("hash", 4, L, 0, B, H, S, D, seed=62)
    k, v, c = dev_cache(K, V, 4, 0)
    Ks, Vs = kvgen.sentinel_cache(L, B, H, S, D)
    rk, rv, rc, ro = _mk(Ks, Vs, 4, 0, dst_layout)
    sig = flags(2)
    sep = dv.endpoint_of(sig[:1], sig)
    d_step = torch.zeros(1, dtype=torch.int32, device="cuda")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            dv.dv_remap_dyn(ctx(), c, rc, dv.region(4, 4 + L, 0, B, p, p + 1), d_step.data_ptr(), T - 1, sep,
                            flag_slot=1, seq=7)
    torch.cuda.synchronize()
    for t in range(T):
        with torch.cuda.stream(s):
            d_step.fill_(t)
            g.replay()
    torch.cuda.synchronize()
    assert int(sig[1]) == 7 + T - 1
    osrc = oc(K, V, 4, 0, S)
    ok.remap(osrc, ro, (4, 4 + L, 0, B, p, p + T))
    assert np.array_equal(to_np(rk), ro.K) and np.array_equal(to_np(rv), ro.V)


def test_inbox_credit_loop_reuses_one_inbox_without_overwrite():
    """A5 inbox credits composed from the ABI: the sender waits for the receiver's consumed-seq ack
    (dv_wait) before refilling the single inbox slot; the receiver waits for the data seq, unpacks,
    then acks (dv_signal). Sender and receiver run on different streams; the sender is slowed down
    at random, the receiver too; every round must land intact in its own destination positions."""
    L, B, H, S, D, R = 2, 2, 4, 64, 64, 24
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=71)
    k, v, c = dev_cache(K, V, 0, 0)
    chunk = ok.region_bytes(0, L, 0, B, 0, 1, H, D, 2)
    inbox = sentinel_like((chunk // 2,))
    data_f = flags(1)
    ack_f = flags(1)
    iep, aep = dv.endpoint_of(inbox, data_f), dv.endpoint_of(ack_f[:1], ack_f)
    dk, dvv = sentinel_like((L, B, H, S, D)), sentinel_like((L, B, H, S, D))
    dc = dv.cache(dk, dvv)
    snd, rcv = torch.cuda.Stream(), torch.cuda.Stream()
    cx = ctx()
    rng = random.Random(5)
    for t in range(1, R + 1):
        reg = dv.region(0, L, 0, B, t, t + 1)
        if t > 1:
            dv.dv_wait(cx, aep, 0, t - 1, stream=snd)          # credit: previous round consumed
        dv.dvt_spin(rng.randint(0, 30000), 1, stream=snd)
        dv.dv_scatter(cx, c, reg, iep, 0, flag_slot=0, seq=t, stream=snd)
        dv.dvt_spin(rng.randint(0, 30000), 1, stream=rcv)
        dv.dv_gather(cx, iep, 0, dc, reg, flag_slot=0, wait_seq=t, stream=rcv)
        dv.dv_signal(cx, aep, 0, t, stream=rcv)                # give the credit back
    torch.cuda.synchronize()
    assert int(ack_f[0]) == R and int(data_f[0]) == R
    got_k, got_v = to_np(dk), to_np(dvv)
    assert np.array_equal(got_k[:, :, :, 1:R + 1], K[:, :, :, 1:R + 1])
    assert np.array_equal(got_v[:, :, :, 1:R + 1], V[:, :, :, 1:R + 1])
    assert np.all(got_k[:, :, :, R + 1:] == kvgen.SENTINEL) and np.all(got_k[:, :, :, 0] == kvgen.SENTINEL)


def test_one_context_two_threads_two_streams_staged():
    """One dv_ctx shared by two host threads on two streams, both hammering the staged paths
    (shared staging pool with event-guarded reuse): every transfer lands intact."""
    import threading
    L, B, H, S, D = 2, 4, 8, 64, 128
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=81)
    k, v, c = dev_cache(K, V, 0, 0)
    osrc = oc(K, V, 0, 0, S)
    cx = dv.dv_create(0, staging_bytes=4 << 20)   # small pool: forces wrap-around and reuse waits
    errs = []

    def worker(wid):
        try:
            st = torch.cuda.Stream()
            for it in range(12):
                s0 = (wid * 7 + it * 3) % (S - 16)
                reg = (0, L, 0, B, s0, s0 + 16)
                n = ok.region_bytes(*reg, H, D, 2)
                host = torch.empty(n // 2, dtype=torch.int16, pin_memory=True)
                dk = torch.full((L, B, H, S, D), -1, dtype=torch.int16, device="cuda")
                dvv = torch.full_like(dk, -1)
                with torch.cuda.stream(st):
                    dv.dv_scatter(cx, c, dv.region(*reg), dv.endpoint_of(host), 0, xfer=dv.DV_XFER_STAGED, stream=st)
                    dv.dv_gather(cx, dv.endpoint_of(host), 0, dv.cache(dk, dvv), dv.region(*reg),
                                 xfer=dv.DV_XFER_STAGED, stream=st)
                st.synchronize()
                if not np.array_equal(to_np(host), ok.pack(osrc, reg)):
                    errs.append((wid, it, "wire"))
                if not np.array_equal(to_np(dk)[:, :, :, s0:s0 + 16], K[:, :, :, s0:s0 + 16]):
                    errs.append((wid, it, "cache"))
        except Exception as e:  # pragma: no cover
            errs.append((wid, repr(e)))
    ths = [threading.Thread(target=worker, args=(w,)) for w in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    cx.close()
    assert not errs, errs[:5]


def test_more_validation_errors():
    L, B, H, S, D = 2, 2, 2, 16, 16
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=82)
    k, v, c = dev_cache(K, V, 0, 0)
    buf = sentinel_like((4096,))
    fl = flags(2)
    cx = ctx()
    cases = [
        (lambda: dv.dv_scatter(cx, c, dv.region(0, 1, 0, 1, 0, 1), dv.endpoint_of(buf, fl), 0, flag_slot=5, seq=1),
         dv.DV_EINVAL),                                           # flag slot beyond n_flags
        (lambda: dv.dv_scatter(cx, c, dv.region(0, 1, 0, 1, 0, 1), dv.endpoint_of(buf), 8), dv.DV_EALIGN),
        (lambda: dv.dv_scatter(cx, c, dv.region(0, 1, 0, 1, 0, 1, 1, 3), dv.endpoint_of(buf)), dv.DV_EMAP),
        (lambda: dv.dv_gather_chunks(cx, dv.endpoint_of(buf), 0, c, dv.region(0, 1, 0, 1, 0, 2), 3, 1),
         dv.DV_EINVAL),                                           # pos_step < positions per chunk
        (lambda: dv.dv_gather_chunks(cx, dv.endpoint_of(buf), 0, c, dv.region(0, 1, 0, 1, 0, 1), 20, 1),
         dv.DV_ERANGE),                                           # last chunk beyond max_seq
        (lambda: dv.dv_ipc_open(b"\0" * 96), dv.DV_EPEER),        # malformed blob
        (lambda: dv.dv_remap(cx, c, dv.cache(k[:, :, :, :, :8].contiguous(), v[:, :, :, :, :8].contiguous()),
                             dv.region(0, 1, 0, 1, 0, 1)), dv.DV_EMAP),   # head_dim differs
    ]
    for fn, st in cases:
        with pytest.raises(dv.DVError) as ei:
            fn()
        assert ei.value.status == st, (ei.value, st)
    torch.cuda.synchronize()
    assert np.all(to_np(buf) == kvgen.SENTINEL)


@pytest.mark.parametrize("elem_bytes", [1, 4, 8])
def test_other_word_sizes_fp8_fp32_fp64(elem_bytes):
    """The kernels move opaque words of any size with D*e % 16 == 0: fp8 (e=1), fp32 (e=4) and
    fp64 (e=8) caches pack, unpack (other max_seq) and remap bit-exactly."""
    tdt = {1: torch.int8, 4: torch.int32, 8: torch.int64}[elem_bytes]
    ndt = {1: np.int8, 4: np.int32, 8: np.int64}[elem_bytes]
    L, B, H, S, D = 3, 2, 3, 20, 32
    K, V = kvgen.random_cache(L, B, H, S, D, elem_bytes, seed=90 + elem_bytes)
    k = torch.from_numpy(K.view(ndt)).cuda()
    v = torch.from_numpy(V.view(ndt)).cuda()
    c = dv.cache(k, v, 2, 1)
    o = ok.Cache(K, V, 2, 1, H, S, D)
    reg = (3, 5, 1, 3, 4, 17)
    exp = ok.pack(o, reg)
    buf = torch.zeros(exp.size, dtype=tdt, device="cuda")
    dv.dv_scatter(ctx(), c, dv.region(*reg), dv.endpoint_of(buf))
    torch.cuda.synchronize()
    assert np.array_equal(buf.cpu().numpy().view(exp.dtype), exp)
    S2 = 29
    dk = torch.zeros((L, B, H, S2, D), dtype=tdt, device="cuda")
    dvv = torch.zeros_like(dk)
    dv.dv_gather(ctx(), dv.endpoint_of(buf), 0, dv.cache(dk, dvv, 2, 1), dv.region(*reg))
    torch.cuda.synchronize()
    od = ok.Cache(np.zeros((L, B, H, S2, D), K.dtype), np.zeros((L, B, H, S2, D), K.dtype), 2, 1, H, S2, D)
    ok.unpack(od, reg, exp)
    assert np.array_equal(dk.cpu().numpy().view(K.dtype), od.K) and np.array_equal(dvv.cpu().numpy().view(K.dtype), od.V)
    rk = torch.zeros_like(dk)
    rv = torch.zeros_like(dk)
    dv.dv_remap(ctx(), c, dv.cache(rk, rv, 2, 1), dv.region(*reg))
    torch.cuda.synchronize()
    assert np.array_equal(rk.cpu().numpy().view(K.dtype), od.K) and np.array_equal(rv.cpu().numpy().view(K.dtype), od.V)


def test_peer_enable():
    dv.dv_peer_enable(0, 0)                       # self: always reachable
    n = torch.cuda.device_count()
    with pytest.raises(dv.DVError) as ei:
        dv.dv_peer_enable(0, n)                   # out of range
    assert ei.value.status == dv.DV_EINVAL
    for peer in range(1, n):                      # only on multi-GPU boxes
        dv.dv_peer_enable(0, peer)
        dv.dv_peer_enable(0, peer)                # idempotent


@pytest.mark.parametrize("near", [False, True])
def test_library_host_arena_stream_out_and_back(near):
    """Library-owned pinned arenas (dv_host_alloc, dv_host_alloc_near: NUMA-local to the GPU) as
    the host endpoint of a token-step stream-out (fused and decoupled, flags in the arena) and of
    the gather back into another cache; every word checked on the device (dvt_verify)."""
    L, B, H, S, D = 3, 2, 4, 32, 64
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    c = dv.cache(k, v)
    dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=77)
    step = ok.region_bytes(0, L, 0, B, 0, 1, H, D, 2)
    nbytes = 8 * step + 64
    if near:
        p, node = dv.dv_host_alloc_near(0, nbytes)
        assert node >= -1
    else:
        p = dv.dv_host_alloc(nbytes)
    try:
        ep = dv.endpoint(dv.DV_EP_HOST, p, 8 * step, flags_ptr=p + 8 * step, n_flags=1)
        torch.cuda.synchronize()
        import ctypes
        ctypes.memset(p + 8 * step, 0, 8)
        cx = ctx()
        for t in range(8):
            dv.dv_scatter(cx, c, dv.region(0, L, 0, B, t, t + 1), ep, t * step, flag_slot=0, seq=t + 1,
                          xfer=dv.DV_XFER_DECOUPLED if t % 2 else dv.DV_XFER_FUSED)
        dv.dv_wait(cx, ep, 0, 8)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        for t in range(8):
            dv.dvt_verify(c, cnt.data_ptr(), seed=77, reg=dv.region(0, L, 0, B, t, t + 1), wire_ptr=p + t * step)
        k2, v2 = torch.full_like(k, -1), torch.full_like(v, -1)
        c2 = dv.cache(k2, v2)
        dv.dv_gather_chunks(cx, ep, 0, c2, dv.region(0, L, 0, B, 0, 1), 8, 1)
        dv.dvt_verify(c2, cnt.data_ptr(), seed=77, reg=dv.region(0, L, 0, B, 0, 8))
        torch.cuda.synchronize()
        assert int(cnt.item()) == 0
        assert int(k2[:, :, :, 8:].ne(-1).sum()) == 0
    finally:
        torch.cuda.synchronize()
        dv.dv_host_free(p)


@pytest.mark.parametrize("pinned", [False, True])
def test_flag_watcher_sees_each_seq_in_order(pinned):
    """dvt_watch (the latency observer of bench.py): a GPU thread on its own stream stamps the
    first time it reads each seq of a flag (device or pinned host) written by stream signals."""
    cx = ctx()
    fl = flags(1, pinned=pinned)
    ep = dv.endpoint_of(pinned_u16(16) if pinned else torch.empty(16, dtype=torch.int16, device="cuda"), fl)
    tw = torch.zeros(3, dtype=torch.int64, device="cuda")
    main, ws = torch.cuda.current_stream(), torch.cuda.Stream()
    dv.dvt_spin(1000, 1, stream=main)                  # every kernel loaded before the watcher spins
    dv.dvt_watch(ep.flags, 0, 1, tw.data_ptr(), 1000, stream=ws)
    torch.cuda.synchronize()
    dv.dvt_watch(ep.flags, 1, 3, tw.data_ptr(), 2_000_000_000, stream=ws)
    for i in range(3):
        dv.dvt_spin(50_000, 1, stream=main)
        dv.dv_signal(cx, ep, 0, i + 1, stream=main)
    torch.cuda.synchronize()
    t = tw.tolist()
    assert all(x > 0 for x in t) and t[0] < t[1] < t[2] and t[2] - t[0] >= 80_000


def test_spinning_consumer_does_not_block_first_stream_out():
    """dv_create loads every library kernel: a consumer kernel that is already spinning on a flag
    (here the dvt_watch observer) cannot deadlock against the lazy loading of the stream-out
    kernel's first launch. Fresh process, so no earlier test has loaded anything."""
    import subprocess
    import sys
    code = r'''
import sys, time, torch
sys.path.insert(0, %r)
import paper_2403_01876_b200 as dv
ctx = dv.dv_create(0)
k = torch.zeros((2, 2, 4, 16, 64), dtype=torch.int16, device="cuda"); v = torch.zeros_like(k)
buf = torch.empty(2 * 2 * 2 * 4 * 64, dtype=torch.int16, device="cuda")
fl = torch.zeros(1, dtype=torch.int64, device="cuda")
tw = torch.zeros(1, dtype=torch.int64, device="cuda")
ws = torch.cuda.Stream()
torch.cuda.synchronize()
dv.dvt_watch(fl.data_ptr(), 1, 1, tw.data_ptr(), 3_000_000_000, stream=ws)
t0 = time.time()
dv.dv_scatter(ctx, dv.cache(k, v), dv.region(0, 2, 0, 2, 5, 6), dv.endpoint_of(buf, fl), 0, flag_slot=0, seq=1)
torch.cuda.synchronize()
dt = time.time() - t0
assert int(tw[0]) > 0 and dt < 1.5, (int(tw[0]), dt)
print("ok", dt)
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("host", [False, True])
@pytest.mark.parametrize("npos", [1, 24])
def test_in_kernel_consumer_acquires_released_payload(host, npos):
    """A5, consumer form 2 (include/dv_device.cuh): a kernel launched BEFORE the stream-out, on its
    own stream, spins with dv_flag_wait on the flag, then copies the wire. It must read exactly the
    oracle's packed bytes: the release (gpu-scope cluster/ticket for HBM, system scope for pinned
    host) orders every CTA's payload before the flag for a GPU-side acquirer too."""
    L, B, H, S, D = 2, 4, 8, 64, 128
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=41 + npos)
    k, v, c = dev_cache(K, V, 0, 0)
    reg = (0, L, 0, B, 5, 5 + npos)
    exp = ok.pack(oc(K, V, 0, 0, S), reg)
    wire = pinned_u16(exp.size) if host else sentinel_like((exp.size,))
    fl = flags(1, pinned=host)
    ep = dv.endpoint_of(wire, fl)
    out = torch.full((exp.size,), -1, dtype=torch.int16, device="cuda")
    okf = torch.ones(1, dtype=torch.int32, device="cuda")
    cx = ctx()
    prod, cons = torch.cuda.Stream(), torch.cuda.Stream()
    dv.dvt_spin(1000, 1, stream=prod)   # every kernel loaded before the consumer spins
    torch.cuda.synchronize()
    dv.dvt_consume(ep.flags, 9, wire.data_ptr(), out.data_ptr(), exp.size * 2, okf.data_ptr(), stream=cons)
    dv.dvt_spin(2_000_000, 1, stream=prod)
    dv.dv_scatter(cx, c, dv.region(*reg), ep, 0, flag_slot=0, seq=9, xfer=dv.DV_XFER_FUSED, stream=prod)
    torch.cuda.synchronize()
    assert int(okf[0]) == 1
    assert np.array_equal(to_np(out), exp)


def test_region_tuples_equal_region_structs():
    """The binding's fast path takes a region as a plain tuple (no ctypes structure per call):
    scatter, gather and remap with tuples give the same bytes as with dv_region structures."""
    L, B, H, S, D = 2, 3, 4, 20, 64
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=61)
    k, v, c = dev_cache(K, V, 0, 0)
    for reg in [(0, 2, 1, 3, 4, 17), (1, 2, 0, 3, 0, 20, 1, 3)]:
        exp = ok.pack(oc(K, V, 0, 0, S), reg)
        a, b = sentinel_like((exp.size,)), sentinel_like((exp.size,))
        dv.dv_scatter(ctx(), c, reg, dv.endpoint_of(a))
        dv.dv_scatter(ctx(), c, dv.region(*reg), dv.endpoint_of(b))
        torch.cuda.synchronize()
        assert np.array_equal(to_np(a), exp) and np.array_equal(to_np(b), exp)
        dk, dvv = sentinel_like((L, B, H, S, D)), sentinel_like((L, B, H, S, D))
        dv.dv_gather(ctx(), dv.endpoint_of(a), 0, dv.cache(dk, dvv), reg)
        ek, ev = sentinel_like((L, B, H, S, D)), sentinel_like((L, B, H, S, D))
        dv.dv_remap(ctx(), c, dv.cache(ek, ev), reg)
        torch.cuda.synchronize()
        assert torch.equal(dk, ek) and torch.equal(dvv, ev)
    with pytest.raises(ValueError):
        dv.dv_scatter(ctx(), c, (0, 1, 0, 1), dv.endpoint_of(a))


def test_enomem_and_epeer_have_no_partial_effect():
    """DV_ENOMEM: a staged transfer with K in the FT6D layout and V in KV5D (two plans: staged per
    layer slab, or per (layer, K or V) half-slab) whose half-slab exceeds half the staging pool is
    refused before anything is enqueued (the destination stays untouched); a single-plan copy
    would instead be chunked by runs. DV_EPEER: exporting pinned host memory over CUDA IPC."""
    L, B, H, S, D = 2, 4, 8, 128, 128         # one layer slab over [0, 128): 2 MiB; half-slab 1 MiB
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=71)
    k, v, c, o = _mk(K, V, 0, 0, ok.LAYOUT_FT6D)
    cx = dv.dv_create(0, staging_bytes=1 << 20)
    nbytes = ok.region_bytes(0, L, 0, B, 0, S, H, D, 2)
    host = pinned_u16(nbytes // 2)
    host.fill_(-1)
    with pytest.raises(dv.DVError) as ei:
        dv.dv_scatter(cx, c, dv.region(0, L, 0, B, 0, S), dv.endpoint_of(host), xfer=dv.DV_XFER_STAGED)
    assert ei.value.status == dv.DV_ENOMEM and "staging" in str(ei.value)
    torch.cuda.synchronize()
    assert bool((host == -1).all())
    # the same call fused (no staging) succeeds and matches the oracle
    dv.dv_scatter(cx, c, dv.region(0, L, 0, B, 0, S), dv.endpoint_of(host), xfer=dv.DV_XFER_FUSED)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(host), ok.pack(o, (0, L, 0, B, 0, S)))
    with pytest.raises(dv.DVError) as ei:
        dv.dv_ipc_export(host.data_ptr())
    assert ei.value.status == dv.DV_EPEER
    cx.close()


def test_auto_falls_back_to_kernel_copies_when_staging_cannot_hold_a_slab():
    """AUTO picks staging for large host transfers (writes >= 32 MB, reads >= 4 MiB); with an FT6D
    key (two plans, staged per layer slab) and a pool smaller than two slabs it must fall back to
    the kernel's own PCIe stores / loads instead of failing -- bytes == the oracle. An explicit
    STAGED request still reports DV_ENOMEM."""
    L, B, H, S, D = 4, 8, 32, 128, 128       # 67 MB region, 16.8 MB per layer slab
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=73)
    k, v, c, o = _mk(K, V, 0, 0, ok.LAYOUT_FT6D)
    cx = dv.dv_create(0, staging_bytes=8 << 20)
    reg = (0, L, 0, B, 0, S)
    exp = ok.pack(o, reg)
    host = pinned_u16(exp.size)
    host.fill_(-1)
    dv.dv_scatter(cx, c, dv.region(*reg), dv.endpoint_of(host))            # AUTO
    torch.cuda.synchronize()
    assert np.array_equal(to_np(host), exp)
    Ks, Vs = kvgen.sentinel_cache(L, B, H, S, D)
    dk, dvv, dc, do = _mk(Ks, Vs, 0, 0, ok.LAYOUT_FT6D)
    dv.dv_gather(cx, dv.endpoint_of(host), 0, dc, dv.region(*reg))           # AUTO read, 67 MB
    torch.cuda.synchronize()
    ok.unpack(do, reg, exp)
    assert np.array_equal(to_np(dk), do.K) and np.array_equal(to_np(dvv), do.V)
    for call in (lambda: dv.dv_scatter(cx, c, dv.region(*reg), dv.endpoint_of(host), xfer=dv.DV_XFER_STAGED),
                 lambda: dv.dv_gather(cx, dv.endpoint_of(host), 0, dc, dv.region(*reg), xfer=dv.DV_XFER_STAGED)):
        with pytest.raises(dv.DVError) as ei:
            call()
        assert ei.value.status == dv.DV_ENOMEM
    cx.close()



@pytest.mark.parametrize("pool_mib", [24, 64])
def test_staged_two_plan_copies_per_layer_or_per_half_slab(pool_mib):
    """Staged FT6D transfers (two plans) move whole layer slabs when a slab fits half the pool
    (64 MiB pool, 16.8 MB slab) and (layer, K or V) half-slabs when only a half fits (24 MiB pool):
    scatter to and gather from pinned host, explicit STAGED and AUTO, == the oracle."""
    L, B, H, S, D = 3, 8, 32, 128, 128
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=79)
    k, v, c, o = _mk(K, V, 0, 0, ok.LAYOUT_FT6D)
    cx = dv.dv_create(0, staging_bytes=pool_mib << 20)
    reg = (0, L, 0, B, 2, 126)
    exp = ok.pack(o, reg)
    for xf in (dv.DV_XFER_STAGED, dv.DV_XFER_AUTO):
        host = pinned_u16(exp.size)
        host.fill_(-1)
        dv.dv_scatter(cx, c, dv.region(*reg), dv.endpoint_of(host), xfer=xf)
        torch.cuda.synchronize()
        assert np.array_equal(to_np(host), exp)
        Ks, Vs = kvgen.sentinel_cache(L, B, H, S, D)
        dk, dvv, dc, do = _mk(Ks, Vs, 0, 0, ok.LAYOUT_FT6D)
        dv.dv_gather(cx, dv.endpoint_of(host), 0, dc, dv.region(*reg), xfer=xf)
        torch.cuda.synchronize()
        ok.unpack(do, reg, exp)
        assert np.array_equal(to_np(dk), do.K) and np.array_equal(to_np(dvv), do.V)
    cx.close()
