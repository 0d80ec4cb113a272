"""GPU parity of device plans (include/dv.h dv_dplan_*, include/dv_device.cuh): the stream-out
fused into the producer kernel. The producer is the test library's vectorised writer
(dvt_fill_rows): it writes kvgen's words into its cache and, through the plan, every row of the
plan's region straight to the destination, then releases the flag from its last CTA. Everything is
compared with the CPU oracle (pack / remap of the kvgen cache), and the destination bytes outside
the plan stay untouched."""
import numpy as np
import pytest
import torch

import kvgen
import paper_2403_01876_b200 as dv
from oracle import kvstream as ok
from oracle import scenarios

from gpu_util import ctx, flags, sentinel_like, to_dev, to_np

pytestmark = pytest.mark.gpu

SEED = 20240311


def _cache(L, B, H, S, D, lb=0, rb=0, hb=0):
    K, V = kvgen.kv5d_cache("hash", lb, L, rb, B, H, S, D, seed=SEED, head_begin=hb)
    k, v = to_dev(K), to_dev(V)
    return k, v, dv.cache(k, v, lb, rb, head_begin=hb), ok.Cache(K, V, lb, rb, H, S, D, ok.LAYOUT_KV5D, hb)


@pytest.mark.parametrize("host", [False, True])
def test_fused_producer_streams_a_token_step_per_step(host):
    """A plan over (layers 3..7, all requests, all heads) x one position, 6 steps into a log of 6
    slots (host or HBM): the producer writes position p + k at step k for ALL layers; each slot ==
    oracle.pack of the plan's region shifted by k, flags seq + k, the cache == kvgen's words."""
    L, B, H, S, D, p = 10, 3, 4, 64, 128, 20
    k, v, c, o = _cache(L, B, H, S, D)
    k.fill_(0)   # the producer must rewrite its region of the cache
    v.fill_(0)
    reg = (3, 8, 0, B, p, p + 1)
    slot = ok.region_bytes(*reg, H, D, 2)
    log = sentinel_like((6 * slot // 2,), pinned=host)
    fl = flags(1, pinned=host)
    ep = dv.endpoint_of(log, fl)
    plan = dv.dv_dplan_scatter(ctx(), c, dv.region(*reg), ep, 0, slot, flag_slot=0, seq=100, max_step=5)
    assert plan.sys_scope == (1 if host else 0)
    torch.cuda.synchronize()
    for step in range(6):
        dv.dvt_fill_rows(c, SEED, dv.region(0, L, 0, B, p + step, p + step + 1), plan, step)
    torch.cuda.synchronize()
    assert int(fl[0]) == 105
    got = to_np(log)
    for step in range(6):
        exp = ok.pack(o, ok.shifted(reg, step))
        assert np.array_equal(got[step * slot // 2:(step + 1) * slot // 2], exp), step
    kk = to_np(k)
    assert np.array_equal(kk[:, :, :, p:p + 6], o.K[:, :, :, p:p + 6])


def test_fused_producer_plan_subset_and_offsets():
    """Cache with layer / request / head offsets; the plan covers a sub-range of its heads and
    requests; the producer writes more rows than the plan: only the plan's rows reach the
    destination (dst_off inside a larger buffer), every other byte stays the sentinel."""
    L, B, H, S, D = 4, 4, 6, 48, 64
    lb, rb, hb = 7, 2, 3
    k, v, c, o = _cache(L, B, H, S, D, lb, rb, hb)
    reg = (lb + 1, lb + 3, rb + 1, rb + 3, 10, 14, hb + 2, hb + 5)
    nb = ok.region_bytes(*reg[:6], reg[7] - reg[6], D, 2)   # 3 of the cache's heads
    buf = sentinel_like((nb // 2 + 4096,))
    fl = flags(1)
    plan = dv.dv_dplan_scatter(ctx(), c, dv.region(*reg), dv.endpoint_of(buf, fl), 4096, flag_slot=0, seq=9)
    torch.cuda.synchronize()
    dv.dvt_fill_rows(c, SEED, dv.region(lb, lb + L, rb, rb + B, 8, 16), plan, 0)
    torch.cuda.synchronize()
    got = to_np(buf)
    assert np.all(got[:2048] == 0xFFFF)
    assert np.array_equal(got[2048:2048 + nb // 2], ok.pack(o, reg))
    assert np.all(got[2048 + nb // 2:] == 0xFFFF)
    assert int(fl[0]) == 9


def test_fused_producer_remap_into_a_cache_then_consumer_stream():
    """A remap plan into another KV5D cache (other max_seq, its own layer/request origin) releasing
    a device flag: a consumer stream waits for the flag and copies the destination cache -- it sees
    every row of the step (20 steps, each compared with oracle.remap)."""
    L, B, H, S, D = 3, 2, 4, 40, 128
    k, v, c, o = _cache(L, B, H, S, D, lb=2)
    Ks, Vs = kvgen.sentinel_cache(L, B, H, 64, D)
    dk, dvv = to_dev(Ks), to_dev(Vs)
    dc = dv.cache(dk, dvv, 2, 0)
    do = ok.Cache(Ks.copy(), Vs.copy(), 2, 0, H, 64, D)
    fl = flags(1)
    sig = dv.endpoint_of(torch.empty(64, dtype=torch.int16, device="cuda"), fl)
    reg = (2, 5, 0, B, 10, 11)
    plan = dv.dv_dplan_remap(ctx(), c, dc, dv.region(*reg), sig, flag_slot=0, seq=1, max_step=19)
    assert plan.sys_scope == 0
    cons = torch.cuda.Stream()
    snap = torch.empty_like(dk)
    torch.cuda.synchronize()
    for step in range(20):
        dv.dvt_fill_rows(c, SEED, dv.region(2, 5, 0, B, 10 + step, 11 + step), plan, step)
        dv.dv_wait(ctx(), sig, 0, 1 + step, stream=cons.cuda_stream)
        with torch.cuda.stream(cons):
            snap.copy_(dk)
        cons.synchronize()
        ok.remap(o, do, ok.shifted(reg, step))
        assert np.array_equal(to_np(snap), do.K), step
    torch.cuda.synchronize()
    assert np.array_equal(to_np(dvv), do.V)


def test_fused_producer_remap_into_an_ft6d_cache():
    """A remap plan into a FasterTransformer 6-D cache (the key's packets S*16 bytes apart; the
    producer stores packets through dv_dplan_packet) over 8 steps == oracle.remap into FT6D; the
    rest of the destination keeps the sentinel."""
    L, B, H, S, D = 2, 3, 4, 32, 64
    k, v, c, o = _cache(L, B, H, S, D)
    Ks, Vs = kvgen.sentinel_cache(L, B, H, 48, D)
    K6 = kvgen.as_ft6d_key(Ks)
    dk, dvv = to_dev(K6), to_dev(Vs)
    dc = dv.cache(dk, dvv)
    do = ok.Cache(K6.copy(), Vs.copy(), 0, 0, H, 48, D, ok.LAYOUT_FT6D, 0)
    fl = flags(1)
    sig = dv.endpoint_of(torch.empty(64, dtype=torch.int16, device="cuda"), fl)
    reg = (0, L, 1, B, 5, 7, 1, 3)
    plan = dv.dv_dplan_remap(ctx(), c, dc, dv.region(*reg), sig, flag_slot=0, seq=1, max_step=7)
    assert list(plan.st_u) == [48 * 16, 16] and list(plan.st_s) == [16, D * 2]
    torch.cuda.synchronize()
    for step in range(8):
        dv.dvt_fill_rows(c, SEED, dv.region(0, L, 0, B, 5 + step, 7 + step), plan, step)
        ok.remap(o, do, ok.shifted(reg, step))
    torch.cuda.synchronize()
    assert int(fl[0]) == 8
    assert np.array_equal(to_np(dk), do.K) and np.array_equal(to_np(dvv), do.V)


def test_fused_producer_with_an_ft6d_cache():
    """A producer whose own cache keeps FasterTransformer's 6-D key (packets S*16 bytes apart)
    streams a region to a device wire through a scatter plan: its cache == kvgen's words in FT6D,
    the wire == oracle.pack of that cache (position-major: the plan transposes nothing, the
    producer already holds each row)."""
    L, B, H, S, D = 2, 3, 4, 40, 64
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=SEED)
    K6 = kvgen.as_ft6d_key(K)
    k6 = torch.zeros(K6.shape, dtype=torch.int16, device="cuda")
    v = torch.zeros(V.shape, dtype=torch.int16, device="cuda")
    c6 = dv.cache(k6, v)
    o = ok.Cache(K6, V, 0, 0, H, S, D, ok.LAYOUT_FT6D, 0)
    reg = (0, L, 1, B, 7, 19, 1, 4)
    nb = ok.region_bytes(*reg[:6], reg[7] - reg[6], D, 2)
    buf = sentinel_like((nb // 2,))
    fl = flags(1)
    plan = dv.dv_dplan_scatter(ctx(), c6, dv.region(*reg), dv.endpoint_of(buf, fl), 0, flag_slot=0, seq=3)
    torch.cuda.synchronize()
    dv.dvt_fill_rows(c6, SEED, dv.region(0, L, 0, B, 0, S), plan, 0)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(k6), K6) and np.array_equal(to_np(v), V)
    assert np.array_equal(to_np(buf), ok.pack(o, reg)) and int(fl[0]) == 3
    dv.dv_dplan_free(ctx(), plan)


def _blocks(setup):
    for i in range(setup.n_stages):
        for u in range(setup.n_micro):
            yield i, u, setup.layer_bounds[i], setup.layer_bounds[i + 1], setup.req_bounds[u], setup.req_bounds[u + 1]


@pytest.mark.parametrize("psplit,tsplit,preq,treq", [
    ([0, 16, 32, 48, 64], [0, 13, 30, 47, 64], [0, 4], [0, 4]),        # C3 partitions (7 pieces)
    ([0, 16, 32, 48, 64], [0, 13, 30, 47, 64], [0, 4], [0, 2, 4]),     # + batch split (14 pieces)
    ([0, 9, 18, 27, 36, 45, 54, 62, 70], [0, 35, 70], [0, 2, 4], [0, 4]),  # merge
])
@pytest.mark.parametrize("form", ["direct", "inbox"])
def test_fused_producer_disaggregation(psplit, tsplit, preq, treq, form):
    """C3 through plan sets (dv_dplan_stream_out_direct): every prompt block's PRODUCER writes its
    prompt K/V (positions [0, p)) and, through one plan per route piece, straight into the token
    blocks' caches (other layer partition, max_seq, batch split) with one release per piece;
    token caches == oracle.disaggregate, every signal at seq."""
    H, D, p, Sp, St = 3, 16, 12, 16, 24
    ps, ts = ok.Setup(psplit, preq, Sp), ok.Setup(tsplit, treq, St)
    dps, dts = dv.Setup(psplit, preq, Sp), dv.Setup(tsplit, treq, St)
    prompt, oprompt = {}, {}
    for i, u, a, b, c0, c1 in _blocks(ps):
        K, V = kvgen.kv5d_cache("hash", a, b - a, c0, c1 - c0, H, Sp, D, seed=SEED, valid_pos=(0, p))
        k = torch.full((b - a, c1 - c0, H, Sp, D), -2, dtype=torch.int16, device="cuda")   # the producer writes [0, p)
        v = torch.full_like(k, -2)
        prompt[(i, u)] = (k, v, dv.cache(k, v, a, c0))
        oprompt[(i, u)] = ok.Cache(K, V, a, c0, H, Sp, D)
    token, otoken = {}, {}
    for j, w, a, b, c0, c1 in _blocks(ts):
        k = sentinel_like((b - a, c1 - c0, H, St, D))
        v = sentinel_like((b - a, c1 - c0, H, St, D))
        token[(j, w)] = (k, v, dv.cache(k, v, a, c0))
        otoken[(j, w)] = ok.Cache(*kvgen.sentinel_cache(b - a, c1 - c0, H, St, D), a, c0, H, St, D)
    reg = dv.region(psplit[0], psplit[-1], preq[0], preq[-1], 0, p)
    dcs = [token[(j, w)][2] for j, w, *_ in _blocks(ts)]
    nblk_p, nblk_t = ps.n_stages * ps.n_micro, ts.n_stages * ts.n_micro
    sigf = flags(nblk_t * nblk_p)
    sig = [dv.endpoint_of(sigf[:1], sigf[kk * nblk_p:(kk + 1) * nblk_p]) for kk in range(nblk_t)]
    torch.cuda.synchronize()
    n_pieces = 0
    if form == "inbox":   # the paper's mailbox form: plans into inboxes, receivers run dv_stream_in
        eps, keep = [], []
        for j, w, a, b, c0, c1 in _blocks(ts):
            keep.append((sentinel_like(((b - a) * (c1 - c0) * H * p * D * 2,)), flags(nblk_p)))
            eps.append(dv.endpoint_of(*keep[-1]))
        torch.cuda.synchronize()
    for i, u, a, b, c0, c1 in _blocks(ps):
        if form == "direct":
            pset = dv.dv_dplan_stream_out_direct(ctx(), prompt[(i, u)][2], reg, dps, i, u, dts, dcs, sig, seq=1)
        else:
            pset = dv.dv_dplan_stream_out(ctx(), prompt[(i, u)][2], reg, dps, i, u, dts, eps, seq=1)
        n_pieces += pset.n
        dv.dvt_fill_rows(prompt[(i, u)][2], SEED, dv.region(a, b, c0, c1, 0, p), pset, 0)
    if form == "inbox":
        for kk, (j, w, *_r) in enumerate(_blocks(ts)):
            dv.dv_stream_in(ctx(), token[(j, w)][2], reg, dps, dts, j, w, eps[kk], 1)
    torch.cuda.synchronize()
    assert n_pieces == len(ok.route(ps, ts, (psplit[0], psplit[-1], preq[0], preq[-1], 0, p), H, D, 2))
    scenarios.disaggregate(oprompt, ps, otoken, ts, p)
    for key, (k, v, _) in token.items():
        assert np.array_equal(to_np(k), otoken[key].K) and np.array_equal(to_np(v), otoken[key].V), key
    if form == "direct":   # every (token block, prompt block) pair that shares a piece got its release
        for pc in ok.route(ps, ts, (psplit[0], psplit[-1], preq[0], preq[-1], 0, p), H, D, 2):
            kk = pc.dst_stage * ts.n_micro + pc.dst_micro
            assert int(sigf[kk * nblk_p + pc.src_stage * ps.n_micro + pc.src_micro]) == 1


def test_dplan_validation():
    """Errors before anything is planned: a log too small for max_step, positions past the source
    max_seq at max_step, a ring inbox."""
    L, B, H, S, D = 2, 2, 2, 16, 64
    k, v, c, o = _cache(L, B, H, S, D)
    reg = dv.region(0, L, 0, B, 4, 5)
    nb = ok.region_bytes(0, L, 0, B, 4, 5, H, D, 2)
    buf = sentinel_like((nb // 2 * 2,))
    with pytest.raises(dv.DVError) as ei:
        dv.dv_dplan_scatter(ctx(), c, reg, dv.endpoint_of(buf), 0, nb, max_step=2)
    assert ei.value.status in (dv.DV_ERANGE, dv.DV_EINVAL)
    with pytest.raises(dv.DVError) as ei:
        dv.dv_dplan_scatter(ctx(), c, reg, dv.endpoint_of(buf), 0, 0, max_step=S)
    assert ei.value.status == dv.DV_ERANGE
    ring = dv.endpoint_of(buf, flags(1), n_slots=2, slot_bytes=nb)
    with pytest.raises(dv.DVError):
        dv.dv_dplan_scatter(ctx(), c, reg, ring, 0)


def test_dplan_free_returns_tickets():
    """dv_dplan_free hands the plan's ticket back: the next plan reuses it, 70,000 make / free cycles
    stay inside the context's 65,536 plan tickets, and a freed plan's producer releases nothing
    (its rows still land)."""
    L, B, H, S, D = 1, 1, 2, 16, 64
    k, v, c, o = _cache(L, B, H, S, D)
    reg = (0, 1, 0, 1, 3, 4)
    nb = ok.region_bytes(*reg, H, D, 2)
    buf = sentinel_like((nb // 2,))
    fl = flags(1)
    ep = dv.endpoint_of(buf, fl)
    p1 = dv.dv_dplan_scatter(ctx(), c, dv.region(*reg), ep, 0, flag_slot=0, seq=5)
    t1 = p1.ticket
    dv.dv_dplan_free(ctx(), p1)
    assert not p1.ticket and not p1.flag
    p2 = dv.dv_dplan_scatter(ctx(), c, dv.region(*reg), ep, 0, flag_slot=0, seq=5)
    assert p2.ticket == t1
    for _ in range(70_000):
        q = dv.dv_dplan_scatter(ctx(), c, dv.region(*reg), ep, 0, flag_slot=0, seq=5)
        dv.dv_dplan_free(ctx(), q)
    dv.dv_dplan_free(ctx(), p2)
    torch.cuda.synchronize()
    dv.dvt_fill_rows(c, SEED, dv.region(*reg), p2, 0)   # freed: rows land, no release
    torch.cuda.synchronize()
    assert np.array_equal(to_np(buf), ok.pack(o, reg)) and int(fl[0]) == 0
