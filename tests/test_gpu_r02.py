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
