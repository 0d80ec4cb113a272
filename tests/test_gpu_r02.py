"""GPU tests added in round 2: ordering fixes, the bulk-read form, and the forms the
round-2 paths add. Bit-exact against the oracle (or kvgen's definition) as everywhere else.
"""
import os
import subprocess
import sys
import time

import numpy as np
import pytest
import torch

import kvgen
import paper_2403_01876_b200 as dv
from oracle import kvstream as ok

from gpu_util import ctx, flags, pinned_u16, sentinel_like, to_dev, to_np

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _wait_or_unblock(stream, timeout_s, unblock):
    """Poll an event on `stream` for up to timeout_s; if it never completes, run unblock() (so the
    test process does not hang) and return False."""
    ev = torch.cuda.Event()
    ev.record(stream)
    t0 = time.time()
    while not ev.query():
        if time.time() - t0 > timeout_s:
            unblock()
            torch.cuda.synchronize()
            return False
        time.sleep(0.001)
    return True


def test_decoupled_empty_region_publish_waits_for_earlier_dma():
    """ADVICE r01 (api.cu:723): with DV_XFER_DECOUPLED the flag of a non-empty step is stored on the
    context's flag stream after its DMA. An EMPTY region on the same slot must not publish a later
    seq before that DMA lands: a host poller that sees seq 2 must already see step 1's bytes
    (a 163.8 MB C2 prompt layer, ~3 ms on PCIe -- ample time for an early publish to show)."""
    L, B, H, S, D, p = 1, 8, 40, 1024, 128, 1000
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    c = dv.cache(k, v)
    seed = kvgen.config_seed(1)
    dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=seed)
    nbytes = ok.region_bytes(0, L, 0, B, 0, p, H, D, 2)
    ref = torch.empty(nbytes // 2, dtype=torch.int16, device="cuda")
    cx = ctx()
    dv.dv_scatter(cx, c, dv.region(0, L, 0, B, 0, p), dv.endpoint_of(ref), 0)
    ref_h = ref.cpu()
    host = pinned_u16(nbytes // 2)
    fl = flags(1, pinned=True)
    ep = dv.endpoint_of(host, fl)
    torch.cuda.synchronize()
    for rep in range(3):
        host.fill_(-1)
        base = 10 * rep
        dv.dv_scatter(cx, c, dv.region(0, L, 0, B, 0, p), ep, 0, flag_slot=0, seq=base + 1,
                      xfer=dv.DV_XFER_DECOUPLED)
        dv.dv_scatter(cx, c, dv.region(0, L, 0, B, 5, 5), ep, 0, flag_slot=0, seq=base + 2,
                      xfer=dv.DV_XFER_DECOUPLED)
        t0 = time.time()
        while int(fl[0]) < base + 2:
            assert time.time() - t0 < 10, "flag never published"
        # the instant seq base+2 is visible, step base+1's payload must be complete
        assert torch.equal(host, ref_h), f"seq {base + 2} visible before the earlier DMA landed"
        torch.cuda.synchronize()


def test_mixed_modes_on_one_slot_keep_the_flag_monotone():
    """a FUSED publish to a pinned-host flag after DECOUPLED ones on the same slot is
    ordered after the decoupled flags (the slot's seq never drops back, and a waiter for the fused
    seq sees the decoupled payload too)."""
    L, B, H, S, D, p = 1, 8, 40, 1024, 128, 1000
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    c = dv.cache(k, v)
    dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=5)
    nbytes = ok.region_bytes(0, L, 0, B, 0, p, H, D, 2)
    ref = torch.empty(nbytes // 2, dtype=torch.int16, device="cuda")
    cx = ctx()
    dv.dv_scatter(cx, c, dv.region(0, L, 0, B, 0, p), dv.endpoint_of(ref), 0)
    ref_h = ref.cpu()
    small = ok.region_bytes(0, L, 0, B, 3, 4, H, D, 2)
    host = pinned_u16(nbytes // 2 + small // 2)
    host.fill_(-1)
    fl = flags(1, pinned=True)
    ep = dv.endpoint_of(host, fl)
    torch.cuda.synchronize()
    dv.dv_scatter(cx, c, dv.region(0, L, 0, B, 0, p), ep, 0, flag_slot=0, seq=1, xfer=dv.DV_XFER_DECOUPLED)
    dv.dv_scatter(cx, c, dv.region(0, L, 0, B, 3, 4), ep, nbytes, flag_slot=0, seq=2, xfer=dv.DV_XFER_FUSED)
    seen = []
    t0 = time.time()
    while int(fl[0]) < 2:
        seen.append(int(fl[0]))
        assert time.time() - t0 < 10
    assert torch.equal(host[:nbytes // 2], ref_h), "fused seq 2 visible before the decoupled step 1 landed"
    torch.cuda.synchronize()
    assert int(fl[0]) == 2 and seen == sorted(seen)


def test_gather_chunks_enomem_and_auto_fallback_have_no_partial_effect():
    """ADVICE r01 (api.cu:1293): dv_gather_chunks decides its transfer before enqueueing anything.
    An explicit STAGED request whose chunk cannot be staged (FT6D key: per layer slab / half-slab
    units larger than half the pool) fails with DV_ENOMEM WITHOUT enqueueing its flag wait (the
    flag here is never set: an enqueued wait would hang the stream); AUTO falls back to the
    kernel's own loads and matches the oracle."""
    L, B, H, S, D = 2, 4, 8, 512, 128
    n, step, n_chunks = 64, 64, 5     # 5 MiB: AUTO picks staging for a host read >= 4 MiB
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=77)
    osrc = ok.Cache(K, V, 0, 0, H, S, D)
    first = (0, L, 0, B, 0, n)
    log_np = np.concatenate([ok.pack(osrc, ok.shifted(first, kk * step)) for kk in range(n_chunks)])
    log = torch.from_numpy(log_np.view(np.int16)).pin_memory()
    fl = flags(1, pinned=True)   # stays 0; the host can release an (erroneous) wait on it
    ep = dv.endpoint_of(log, fl)
    Ks, Vs = kvgen.sentinel_cache(L, B, H, S, D)
    Kf = kvgen.as_ft6d_key(Ks)
    dk, dvv = to_dev(Kf), to_dev(Vs)
    dc = dv.cache(dk, dvv)   # 6-D key tensor: FT6D layout
    # chunk 1 MiB; one layer slab 512 KiB, its K or V half 256 KiB > half the 256 KiB pool
    assert ok.region_bytes(0, 1, 0, B, 0, n, H, D, 2) // 2 > (256 << 10) // 2
    cx = dv.dv_create(0, staging_bytes=256 << 10)
    st = torch.cuda.Stream()
    status = None
    try:
        dv.dv_gather_chunks(cx, ep, 0, dc, dv.region(*first), n_chunks, step, flag_slot=0, wait_seq=5,
                            xfer=dv.DV_XFER_STAGED, stream=st.cuda_stream)
    except dv.DVError as e:
        status = e.status

    def unblock():
        fl[0] = 5
    clean = _wait_or_unblock(st, 5.0, unblock)
    assert status == dv.DV_ENOMEM
    assert clean, "DV_ENOMEM call left a flag wait enqueued"
    assert bool((dk == -1).all()) and bool((dvv == -1).all())
    dv.dv_gather_chunks(cx, ep, 0, dc, dv.region(*first), n_chunks, step, xfer=dv.DV_XFER_AUTO)
    torch.cuda.synchronize()
    o = ok.Cache(Kf.copy(), Vs.copy(), 0, 0, H, S, D, ok.LAYOUT_FT6D)
    ok.unpack_chunks(o, first, log_np, n_chunks, step)
    assert np.array_equal(to_np(dk), o.K) and np.array_equal(to_np(dvv), o.V)
    cx.close()


def test_captured_publishes_take_dedicated_tickets():
    """ADVICE r01 (api.cu:352): a publishing launch captured into a CUDA graph keeps its ticket for
    every replay, so captured launches get tickets the round-robin never hands out. Replay a
    captured per-step scatter while > 65,536 eager publishing launches (the round-robin period)
    run on another stream; every replayed step's wire and flag must be right."""
    L, B, H, S, D, p = 2, 2, 4, 64, 16, 8
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=91)
    k, v = to_dev(K), to_dev(V)
    c = dv.cache(k, v)
    osrc = ok.Cache(K, V, 0, 0, H, S, D)
    cx = dv.dv_create(0)
    step_bytes = ok.region_bytes(0, L, 0, B, p, p + 1, H, D, 2)
    wire = torch.full((step_bytes // 2 * (S - p),), -1, dtype=torch.int16, device="cuda")
    gfl = flags(1)
    ep = dv.endpoint_of(wire, gfl)
    d_step = torch.zeros(1, dtype=torch.int32, device="cuda")
    g = torch.cuda.CUDAGraph()
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        with torch.cuda.graph(g, stream=gs):
            dv.dv_scatter_dyn(cx, c, dv.region(0, L, 0, B, p, p + 1), ep, 0, step_bytes, d_step.data_ptr(),
                              S - p - 1, flag_slot=0, seq=100, stream=gs.cuda_stream)
    torch.cuda.synchronize()
    # eager publishing launches on another stream, wrapping the round-robin ticket range
    es = torch.cuda.Stream()
    efl = flags(1)
    ebuf = torch.empty(64, dtype=torch.int16, device="cuda")
    eep = dv.endpoint_of(ebuf, efl)
    src = torch.empty(64, dtype=torch.int16, device="cuda")
    n_eager = 65_536 + 1_000
    steps = S - p
    per = n_eager // steps + 1
    j = 0
    for t in range(steps):
        with torch.cuda.stream(gs):
            d_step.fill_(t)
            g.replay()
        for _ in range(per):
            j += 1
            dv.dv_flush(cx, src.data_ptr(), 128, eep, 0, flag_slot=0, seq=j, xfer=dv.DV_XFER_FUSED,
                        stream=es.cuda_stream)
    torch.cuda.synchronize()
    assert j >= n_eager and int(efl[0]) == j
    assert int(gfl[0]) == 100 + steps - 1
    got = to_np(wire)
    for t in range(steps):
        exp = ok.pack(osrc, (0, L, 0, B, p + t, p + t + 1))
        assert np.array_equal(got[t * step_bytes // 2:(t + 1) * step_bytes // 2], exp), t
    cx.close()


BULK_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
import kvgen, paper_2403_01876_b200 as dv
from oracle import kvstream as ok
from gpu_util import to_dev, to_np, sentinel_like
cx = dv.dv_create(0)
for seed, (L, B, H, S, D, reg) in enumerate([(3, 4, 5, 40, 128, (0, 3, 0, 4, 7, 31)),
                                               (2, 2, 3, 64, 16, (0, 2, 1, 2, 0, 64)),
                                               (4, 8, 8, 130, 64, (1, 4, 0, 8, 2, 129))]):
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=seed)
    osrc = ok.Cache(K, V, 0, 0, H, S, D)
    w = ok.pack(osrc, reg)
    host = torch.from_numpy(w.view(np.int16)).pin_memory()
    dk, dvv = sentinel_like((L, B, H, S, D)), sentinel_like((L, B, H, S, D))
    dv.dv_gather(cx, dv.endpoint_of(host), 0, dv.cache(dk, dvv), dv.region(*reg), xfer=dv.DV_XFER_FUSED)
    torch.cuda.synchronize()
    o = ok.Cache(*kvgen.sentinel_cache(L, B, H, S, D), 0, 0, H, S, D)
    ok.unpack(o, reg, w)
    assert np.array_equal(to_np(dk), o.K) and np.array_equal(to_np(dvv), o.V), seed
l0, _ = dv.dv_stats()
print("ok")
"""


@pytest.mark.parametrize("rdch,rdst", [(8192, 4), (4096, 2), (32768, 8)])
def test_bulk_host_reads_match_oracle(rdch, rdst):
    """The opt-in TMA bulk-read unpack (k_unpack_bulk, DV_RDBULK=1; profiles/r02_host_reads.md):
    fused gathers from pinned host, chunk sizes / stage counts that leave ragged last chunks, equal
    the oracle's unpack (sentinel outside the region untouched)."""
    env = dict(os.environ, DV_RDBULK="1", DV_RDCH=str(rdch), DV_RDST=str(rdst))
    r = subprocess.run([sys.executable, "-c", BULK_SCRIPT, ROOT], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


# ------------------------------------------------------------------------------------------------
# Inbox rings with credits (include/dv.h dv_endpoint; SURVEY §8(a) A5 "inbox credits per slot",
# §8(b) DV_EBUSY; the token machines consume a mailbox)
def _ring_case(n_steps, seed):
    L, B, H, S, D, p = 3, 2, 4, 64 + n_steps, 16, 4
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=seed)
    return (L, B, H, S, D, p), K, V


@pytest.mark.parametrize("inbox_host", [False, True])
def test_ring_credits_stream_1000_chunks_through_two_slots(inbox_host):
    """1,000 token chunks (one position of every layer each, seq 1..1000) go through an inbox of
    only TWO ring slots: the sender's stream writes seq s into slot s % 2 only after the receiver
    released credit s - 2; the receiver (another stream, stalled now and then by spin kernels)
    waits on the flag, unpacks into its cache and releases the credit. Every position of the
    receiver's cache equals the oracle's stream of the same region."""
    n = 1000
    (L, B, H, S, D, p), K, V = _ring_case(n, 101)
    k, v = to_dev(K), to_dev(V)
    src = dv.cache(k, v)
    chunk = ok.region_bytes(0, L, 0, B, 0, 1, H, D, 2)
    if inbox_host:
        inbox = pinned_u16(2 * chunk // 2)
        fl, cr = flags(1, pinned=True), flags(1, pinned=True)
    else:
        inbox = torch.full((2 * chunk // 2,), -1, dtype=torch.int16, device="cuda")
        fl, cr = flags(1), flags(1)
    ep = dv.endpoint_of(inbox, fl, n_slots=2, slot_bytes=chunk, credits=cr)
    dk, dvv = sentinel_like((L, B, H, S, D)), sentinel_like((L, B, H, S, D))
    dst = dv.cache(dk, dvv)
    cx = ctx()
    s_send, s_recv = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for t in range(1, n + 1):
        reg = dv.region(0, L, 0, B, p + t - 1, p + t)
        dv.dv_scatter(cx, src, reg, ep, 0, flag_slot=0, seq=t, xfer=dv.DV_XFER_FUSED, stream=s_send.cuda_stream)
        if t % 97 == 0:
            dv.dvt_spin(200_000, 1, stream=s_recv.cuda_stream)   # a slow receiver
        if t % 89 == 0:
            dv.dvt_spin(100_000, 1, stream=s_send.cuda_stream)   # a slow sender
        dv.dv_gather(cx, ep, 0, dst, reg, flag_slot=0, wait_seq=t, stream=s_recv.cuda_stream)
    torch.cuda.synchronize()
    assert int(fl[0]) == n and int(cr[0]) == n
    o = ok.Cache(*kvgen.sentinel_cache(L, B, H, S, D), 0, 0, H, S, D)
    ok.stream({(0, 0): ok.Cache(K, V, 0, 0, H, S, D)}, ok.Setup([0, L], [0, B], S), {(0, 0): o},
              ok.Setup([0, L], [0, B], S), (0, L, 0, B, p, p + n))
    assert np.array_equal(to_np(dk), o.K) and np.array_equal(to_np(dvv), o.V)


def test_ring_without_credits_overwrites_unread_slots():
    """Negative control for the test above: the same 2-slot ring WITHOUT credits lets the sender
    overwrite slots the (stalled) receiver has not read -- the receiver's cache then differs from
    the oracle. (Shows the credit test can fail.)"""
    n = 64
    (L, B, H, S, D, p), K, V = _ring_case(n, 102)
    k, v = to_dev(K), to_dev(V)
    src = dv.cache(k, v)
    chunk = ok.region_bytes(0, L, 0, B, 0, 1, H, D, 2)
    inbox = torch.full((2 * chunk // 2,), -1, dtype=torch.int16, device="cuda")
    fl = flags(1)
    ep = dv.endpoint_of(inbox, fl, n_slots=2, slot_bytes=chunk)   # no credits
    dk, dvv = sentinel_like((L, B, H, S, D)), sentinel_like((L, B, H, S, D))
    cx = ctx()
    s_send, s_recv = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    dv.dvt_spin(5_000_000, 1, stream=s_recv.cuda_stream)          # receiver stalled 5 ms
    for t in range(1, n + 1):
        reg = dv.region(0, L, 0, B, p + t - 1, p + t)
        dv.dv_scatter(cx, src, reg, ep, 0, flag_slot=0, seq=t, stream=s_send.cuda_stream)
        dv.dv_gather(cx, ep, 0, dv.cache(dk, dvv), reg, flag_slot=0, wait_seq=t, stream=s_recv.cuda_stream)
    torch.cuda.synchronize()
    o = ok.Cache(*kvgen.sentinel_cache(L, B, H, S, D), 0, 0, H, S, D)
    ok.stream({(0, 0): ok.Cache(K, V, 0, 0, H, S, D)}, ok.Setup([0, L], [0, B], S), {(0, 0): o},
              ok.Setup([0, L], [0, B], S), (0, L, 0, B, p, p + n))
    assert not (np.array_equal(to_np(dk), o.K) and np.array_equal(to_np(dvv), o.V))


def test_ring_nowait_returns_ebusy_without_partial_effect():
    """DV_NOWAIT: a sender whose ring slot still holds an unconsumed chunk gets DV_EBUSY and
    nothing is enqueued (inbox bytes and flag unchanged); once the receiver has consumed seq 1
    the same call succeeds. Also the validation of ring descriptors."""
    (L, B, H, S, D, p), K, V = _ring_case(8, 103)
    k, v = to_dev(K), to_dev(V)
    src = dv.cache(k, v)
    chunk = ok.region_bytes(0, L, 0, B, 0, 1, H, D, 2)
    inbox = torch.full((2 * chunk // 2,), -1, dtype=torch.int16, device="cuda")
    fl, cr = flags(1), flags(1)
    ep = dv.endpoint_of(inbox, fl, n_slots=2, slot_bytes=chunk, credits=cr)
    cx = ctx()
    regs = [dv.region(0, L, 0, B, p + t, p + t + 1) for t in range(4)]
    nw = dv.DV_XFER_FUSED | dv.DV_NOWAIT
    dv.dv_scatter(cx, src, regs[0], ep, 0, flag_slot=0, seq=1, xfer=nw)
    dv.dv_scatter(cx, src, regs[1], ep, 0, flag_slot=0, seq=2, xfer=nw)
    torch.cuda.synchronize()
    before = inbox.clone()
    with pytest.raises(dv.DVError) as ei:
        dv.dv_scatter(cx, src, regs[2], ep, 0, flag_slot=0, seq=3, xfer=nw)
    assert ei.value.status == dv.DV_EBUSY
    torch.cuda.synchronize()
    assert torch.equal(inbox, before) and int(fl[0]) == 2
    dk, dvv = sentinel_like((L, B, H, S, D)), sentinel_like((L, B, H, S, D))
    dv.dv_gather(cx, ep, 0, dv.cache(dk, dvv), regs[0], flag_slot=0, wait_seq=1)
    torch.cuda.synchronize()
    assert int(cr[0]) == 1
    dv.dv_scatter(cx, src, regs[2], ep, 0, flag_slot=0, seq=3, xfer=nw)   # slot 1 is free now
    torch.cuda.synchronize()
    assert int(fl[0]) == 3
    w = to_np(inbox)
    osrc = ok.Cache(K, V, 0, 0, H, S, D)
    assert np.array_equal(w[chunk // 2:], ok.pack(osrc, (0, L, 0, B, p + 2, p + 3)))   # slot 3 % 2 = 1
    assert np.array_equal(w[:chunk // 2], ok.pack(osrc, (0, L, 0, B, p + 1, p + 2)))   # slot 0 = seq 2
    # ring descriptors are validated: chunk larger than a slot, slot not a multiple of 16, no flag
    bad = dv.endpoint_of(inbox, fl, n_slots=2, slot_bytes=chunk - 16, credits=cr)
    with pytest.raises(dv.DVError) as ei:
        dv.dv_scatter(cx, src, regs[3], bad, 0, flag_slot=0, seq=4)
    assert ei.value.status == dv.DV_EINVAL
    bad = dv.endpoint_of(inbox, fl, n_slots=2, slot_bytes=chunk + 8, credits=cr)
    with pytest.raises(dv.DVError) as ei:
        dv.dv_scatter(cx, src, regs[3], bad, 0, flag_slot=0, seq=4)
    assert ei.value.status == dv.DV_EALIGN
    with pytest.raises(dv.DVError) as ei:
        dv.dv_scatter(cx, src, regs[3], ep, 0, flag_slot=-1, seq=4)
    assert ei.value.status == dv.DV_EINVAL


def test_ring_stream_out_in_two_sources_one_inbox():
    """Level 1 with a 2-slot ring inbox: two prompt blocks (layer split [0,3) [3,6)) stream 40
    token steps each into ONE token block (all 6 layers) through the same ring inbox; each source
    has its own flag and credit slot. The token cache equals the oracle's disaggregation result
    (PAPER.md:266)."""
    L, B, H, S, D, p, n = 6, 2, 3, 64, 16, 8, 40
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=104)
    ps, ts = dv.Setup([0, 3, 6], [0, B], S), dv.Setup([0, L], [0, B], S)
    tensors = [(to_dev(K[a:b]), to_dev(V[a:b])) for a, b in ((0, 3), (3, 6))]
    srcs = [dv.cache(kk, vv, a, 0) for (kk, vv), a in zip(tensors, (0, 3))]   # tensors own the memory
    chunk = ok.region_bytes(0, L, 0, B, 0, 1, H, D, 2)
    inbox = torch.full((2 * chunk // 2,), -1, dtype=torch.int16, device="cuda")
    fl, cr = flags(2), flags(2)
    ep = dv.endpoint_of(inbox, fl, n_slots=2, slot_bytes=chunk, credits=cr)
    dk, dvv = sentinel_like((L, B, H, S, D)), sentinel_like((L, B, H, S, D))
    dst = dv.cache(dk, dvv)
    cx = ctx()
    s_send = [torch.cuda.Stream(), torch.cuda.Stream()]
    s_recv = torch.cuda.Stream()
    torch.cuda.synchronize()
    for t in range(1, n + 1):
        reg = dv.region(0, L, 0, B, p + t - 1, p + t)
        for i in range(2):
            dv.dv_stream_out(cx, srcs[i], reg, ps, i, 0, ts, [ep], seq=t, stream=s_send[i].cuda_stream)
        if t % 7 == 0:
            dv.dvt_spin(150_000, 1, stream=s_recv.cuda_stream)
        dv.dv_stream_in(cx, dst, reg, ps, ts, 0, 0, ep, t, stream=s_recv.cuda_stream)
    torch.cuda.synchronize()
    assert fl.tolist() == [n, n] and cr.tolist() == [n, n]
    o = ok.Cache(*kvgen.sentinel_cache(L, B, H, S, D), 0, 0, H, S, D)
    osrc = {(0, 0): ok.Cache(K[:3], V[:3], 0, 0, H, S, D), (1, 0): ok.Cache(K[3:], V[3:], 3, 0, H, S, D)}
    ok.stream(osrc, ok.Setup([0, 3, 6], [0, B], S), {(0, 0): o}, ok.Setup([0, L], [0, B], S), (0, L, 0, B, p, p + n))
    assert np.array_equal(to_np(dk), o.K) and np.array_equal(to_np(dvv), o.V)


# ------------------------------------------------------------------------------------------------
# NEXT-2: streaming overlapped with compute (PAPER.md:123-135 Opt 2/3, :310)
@pytest.mark.parametrize("xfer", [dv.DV_XFER_DECOUPLED, dv.DV_XFER_FUSED])
def test_streaming_under_concurrent_compute_matches_oracle(xfer):
    """200 token steps streamed (dv_stream_out into a 16-slot host ring, high-priority stream) while
    bf16 GEMMs and an HBM copy saturate the GPU on another stream; each step's stream-out is
    ordered after the previous step's compute (Opt 3). Every chunk, read the moment its flag
    appears, equals the oracle's pack of that position."""
    L, B, H, S, D, p, n, R = 8, 8, 16, 256, 128, 24, 200, 16
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=601)
    k, v = to_dev(K), to_dev(V)
    c = dv.cache(k, v)
    osrc = ok.Cache(K, V, 0, 0, H, S, D)
    step = ok.region_bytes(0, L, 0, B, 0, 1, H, D, 2)
    log = pinned_u16(R * step // 2)
    fl = flags(1, pinned=True)
    ring = dv.endpoint_array([dv.endpoint_of(log, fl, n_slots=R, slot_bytes=step)])
    stage = dv.Setup([0, L], [0, B], S)
    cx = ctx()
    comp, strm = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    big2 = torch.empty_like(big)
    torch.cuda.synchronize()
    seq0 = int(fl[0])
    evs = []
    bad = []
    for i in range(n):
        with torch.cuda.stream(comp):
            torch.matmul(a, a)
            big2.copy_(big)
            e = torch.cuda.Event()
            e.record(comp)
            evs.append(e)
        if i > 0:
            strm.wait_event(evs[i - 1])
        q = p + i
        dv.dv_stream_out(cx, c, (0, L, 0, B, q, q + 1), stage, 0, 0, stage, ring, seq=seq0 + i + 1, xfer=xfer,
                         stream=strm)
        # a consumer thread would read each chunk as its flag appears; here: check the chunk the
        # moment its flag is visible, before the ring slot can be reused (R steps later)
        if i >= R // 2:
            t = i - R // 2 + 1
            while int(fl[0]) < seq0 + t:
                pass
            j = seq0 + t
            w = log[(j % R) * step // 2:((j % R) + 1) * step // 2].numpy().view(np.uint16)
            if not np.array_equal(w, ok.pack(osrc, (0, L, 0, B, p + t - 1, p + t))):
                bad.append(t)
    torch.cuda.synchronize()
    assert int(fl[0]) == seq0 + n and not bad, bad[:5]


# ------------------------------------------------------------------------------------------------
# Persistent stream engine (include/dv.h dv_engine_*; the per-layer latency path).
# While an engine runs, a kernel that is not loaded yet (CUDA lazy loading) or a new stream cannot
# start: every test creates its streams and warms the kernels it uses before the engine runs.
def _engine_case(seed, L=4, B=2, H=4, S=48, D=32, p=8):
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=seed)
    return (L, B, H, S, D, p), K, V


def _wait_done(eng, plans, n, timeout=10.0):
    t0 = time.time()
    while any(eng.done(pl) < n for pl in plans):
        assert time.time() - t0 < timeout, [eng.done(pl) for pl in plans]


@pytest.mark.parametrize("dst_host", [False, True])
def test_engine_per_layer_plans_match_oracle(dst_host):
    """One engine plan per layer (a dyn scatter into a host / device log: token step k of layer l
    lands at k*step + l*layer bytes), kicked per layer per token step from a stream; each layer's
    flag word reaches seq + k; the log equals the oracle's packs. Then park ->
    torch.cuda.synchronize() returns -> a kick relaunches the engine for a new plan."""
    (L, B, H, S, D, p), K, V = _engine_case(701)
    k, v = to_dev(K), to_dev(V)
    c = dv.cache(k, v)
    osrc = ok.Cache(K, V, 0, 0, H, S, D)
    T = S - p
    lay = ok.region_bytes(0, 1, 0, B, 0, 1, H, D, 2)
    stepb = L * lay
    log = pinned_u16(T * stepb // 2) if dst_host else torch.full((T * stepb // 2,), -1, dtype=torch.int16, device="cuda")
    fl = flags(L, pinned=dst_host)
    ep = dv.endpoint_of(log, fl)
    log2 = torch.full((stepb // 2,), -1, dtype=torch.int16, device="cuda")
    fl2 = flags(1)
    st = torch.cuda.Stream()
    torch.cuda.synchronize()
    cx = ctx()
    eng = dv.Engine(cx, 4)
    try:
        plans = [eng.plan_scatter(c, (l, l + 1, 0, B, p, p + 1), ep, l * lay, stepb, flag_slot=l, seq=1, max_step=T - 1)
                 for l in range(L)]
        for t in range(T):
            for l in range(L):
                eng.kick(plans[l], t, stream=st)
        _wait_done(eng, plans, T)
        eng.park()
        torch.cuda.synchronize()                 # returns: the engine is parked
        assert fl.tolist() == [T] * L
        got = to_np(log)
        for t in range(T):
            for l in range(L):
                o = (t * stepb + l * lay) // 2
                assert np.array_equal(got[o:o + lay // 2], ok.pack(osrc, (l, l + 1, 0, B, p + t, p + t + 1))), (t, l)
        # a kick relaunches the parked engine; a plan registered while parked runs
        pl2 = eng.plan_scatter(c, (0, L, 0, B, p, p + 1), dv.endpoint_of(log2, fl2), 0, 0, flag_slot=0, seq=5, max_step=0)
        eng.kick(pl2, 0, stream=st)
        _wait_done(eng, [pl2], 1)
        eng.park()
        torch.cuda.synchronize()
        assert int(fl2[0]) == 5 and np.array_equal(to_np(log2), ok.pack(osrc, (0, L, 0, B, p, p + 1)))
        assert [eng.done(pl) for pl in plans] == [T] * L   # parking kept every plan's progress
    finally:
        eng.close()


def test_engine_producer_rings_doorbell_remap_matches_oracle():
    """A producer kernel rings the engine itself (dvt_fill_ring: its last CTA releases the doorbell
    after every CTA's stores): each token step rewrites position p + k of every layer with a new
    seed, then the engine remaps that position into a second cache (a C5 replica store shape) and
    releases the flag -- a consumer stream waiting on the flag copies the replica's position out
    before the next step; every copy equals the generator for that step's seed."""
    (L, B, H, S, D, p), K, V = _engine_case(702)
    k, v = to_dev(K), to_dev(V)
    c = dv.cache(k, v)
    rk, rv = sentinel_like((L, B, H, S, D)), sentinel_like((L, B, H, S, D))
    rep = dv.cache(rk, rv)
    fl = flags(1)
    sig = dv.endpoint_of(fl, fl)
    cx = ctx()
    T = 16
    ticket = torch.zeros(1, dtype=torch.int32, device="cuda")
    dummy = torch.zeros(1, dtype=torch.int64, device="cuda")
    prod, cons = torch.cuda.Stream(), torch.cuda.Stream()
    outs = [(torch.empty((L, B, H, D), dtype=torch.int16, device="cuda"),
             torch.empty((L, B, H, D), dtype=torch.int16, device="cuda")) for _ in range(T)]
    # warm every kernel used while the engine runs
    dv.dvt_fill_ring(c, 1, (0, L, 0, B, 0, 1), dummy.data_ptr(), 0, ticket.data_ptr(), stream=prod)
    with torch.cuda.stream(cons):
        outs[0][0].copy_(rk[:, :, :, p])
    torch.cuda.synchronize()
    eng = dv.Engine(cx, 4)
    try:
        pl = eng.plan_remap(c, rep, (0, L, 0, B, p, p + 1), sig, flag_slot=0, seq=1, max_step=T - 1)
        db = eng.doorbell(pl)
        for t in range(T):
            dv.dvt_fill_ring(c, 1000 + t, (0, L, 0, B, p + t, p + t + 1), db, t, ticket.data_ptr(), stream=prod)
            dv.dv_wait(cx, sig, 0, 1 + t, stream=cons)
            with torch.cuda.stream(cons):
                outs[t][0].copy_(rk[:, :, :, p + t])
                outs[t][1].copy_(rv[:, :, :, p + t])
        prod.synchronize()
        cons.synchronize()
        eng.park()
        torch.cuda.synchronize()
        assert int(fl[0]) == T
        for t, (ok_, ov_) in enumerate(outs):
            Kt, Vt = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=1000 + t)
            assert np.array_equal(to_np(ok_), Kt[:, :, :, p + t]) and np.array_equal(to_np(ov_), Vt[:, :, :, p + t]), t
    finally:
        eng.close()


def test_engine_validation():
    (L, B, H, S, D, p), K, V = _engine_case(703)
    k, v = to_dev(K), to_dev(V)
    c = dv.cache(k, v)
    cx = ctx()
    buf = torch.empty(1 << 16, dtype=torch.int16, device="cuda")
    with pytest.raises(dv.DVError) as ei:
        dv.Engine(cx, 17)                            # one cluster: at most 16 CTAs
    assert ei.value.status == dv.DV_EINVAL
    eng = dv.Engine(cx, 2)
    try:
        with pytest.raises(dv.DVError) as ei:       # step S - p would run past max_seq
            eng.plan_scatter(c, (0, L, 0, B, p, p + 1), dv.endpoint_of(buf), 0, 0, max_step=S - p)
        assert ei.value.status == dv.DV_ERANGE
        pl = eng.plan_scatter(c, (0, 1, 0, B, p, p + 1), dv.endpoint_of(buf), 0, 0, max_step=3)
        with pytest.raises(dv.DVError) as ei:
            eng.kick(pl, 4)
        assert ei.value.status == dv.DV_ERANGE
        with pytest.raises(dv.DVError) as ei:
            eng.kick(pl + 1, 0)
        assert ei.value.status == dv.DV_EINVAL
    finally:
        eng.close()
    torch.cuda.synchronize()


def test_engine_never_runs_past_max_step():
    """A producer ringing a doorbell beyond the plan's validated max_step must not make the engine
    copy out of range: steps 0..max_step run, the rest never do."""
    (L, B, H, S, D, p), K, V = _engine_case(704)
    k, v = to_dev(K), to_dev(V)
    c = dv.cache(k, v)
    osrc = ok.Cache(K, V, 0, 0, H, S, D)
    lay = ok.region_bytes(0, L, 0, B, 0, 1, H, D, 2)
    buf = torch.full((6 * lay // 2,), -1, dtype=torch.int16, device="cuda")
    fl = flags(1)
    word = torch.tensor([6, 0], dtype=torch.int64, device="cuda")   # "step 5" for the doorbell (+ the next word)
    cx = ctx()
    torch.cuda.synchronize()
    eng = dv.Engine(cx, 2)
    try:
        pl = eng.plan_scatter(c, (0, L, 0, B, p, p + 1), dv.endpoint_of(buf, fl), 0, lay, flag_slot=0, seq=1,
                              max_step=3)
        db = eng.doorbell(pl)
        # ring "step 5" straight into the doorbell word (as a runaway producer would) with the
        # library's own copy kernel (loaded: nothing new may load while the engine runs)
        dv.dv_flush(cx, word.data_ptr(), 16, dv.endpoint(dv.DV_EP_DEVICE, db, 16, device=0), 0, xfer=dv.DV_XFER_FUSED)
        _wait_done(eng, [pl], 4)
        time.sleep(0.05)
        assert eng.done(pl) == 4
        eng.park()
        torch.cuda.synchronize()
        got = to_np(buf)
        for t in range(4):
            assert np.array_equal(got[t * lay // 2:(t + 1) * lay // 2], ok.pack(osrc, (0, L, 0, B, p + t, p + t + 1)))
        assert np.all(got[4 * lay // 2:] == kvgen.SENTINEL) and int(fl[0]) == 4
    finally:
        eng.close()


def test_ring_host_consumer_releases_credits():
    """A HOST consumer drains a pinned-host ring (the paper's token machines check their local CPU
    memory for KV caches): the GPU producer streams 2,000 token chunks into a 3-slot
    ring whose credit words live in pinned host memory; a host thread reads each chunk the moment
    its flag appears, checks it against the oracle's pack, and releases the credit with a plain
    host store -- the producer's stream-ordered credit waits (cuStreamWaitValue64 on host memory)
    hold it back. No chunk is ever overwritten before it was read."""
    import threading
    L, B, H, S, D, p, n, R = 2, 2, 8, 64, 64, 0, 2000, 3
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=801)
    k, v = to_dev(K), to_dev(V)
    c = dv.cache(k, v)
    osrc = ok.Cache(K, V, 0, 0, H, S, D)
    step = ok.region_bytes(0, L, 0, B, 0, 1, H, D, 2)
    exp = [ok.pack(osrc, (0, L, 0, B, q, q + 1)) for q in range(S)]
    ring = pinned_u16(R * step // 2)
    fl, cr = flags(1, pinned=True), flags(1, pinned=True)
    ep = dv.endpoint_of(ring, fl, n_slots=R, slot_bytes=step, credits=cr)
    cx = ctx()
    bad, seen = [], [0]

    def consumer():
        view = ring.numpy().view(np.uint16)
        for s_ in range(1, n + 1):
            t0 = time.time()
            while int(fl[0]) < s_:
                if time.time() - t0 > 20:
                    bad.append(("timeout", s_))
                    return
            o = (s_ % R) * step // 2
            if not np.array_equal(view[o:o + step // 2], exp[(s_ - 1) % S]):
                bad.append(s_)
            cr[0] = s_        # the credit: the slot may be reused
            seen[0] = s_
    import sys
    old_si = sys.getswitchinterval()
    sys.setswitchinterval(0.0002)
    th = threading.Thread(target=consumer)
    th.start()
    st = torch.cuda.Stream()
    for s_ in range(1, n + 1):
        q = (s_ - 1) % S
        dv.dv_scatter(cx, c, (0, L, 0, B, q, q + 1), ep, 0, flag_slot=0, seq=s_, stream=st)
    st.synchronize()
    th.join(timeout=60)
    sys.setswitchinterval(old_si)
    assert not bad, bad[:5]
    assert seen[0] == n and int(fl[0]) == n
