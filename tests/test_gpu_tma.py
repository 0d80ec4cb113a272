"""GPU parity of the TMA-row form of the FT6D key transpose (NEXT-1; DESIGN.md §6 "FT6D keys"):
the packet-major side moved by cp.async.bulk.tensor through a 5-D tensor map, the position-major
side by the CTA's threads. Every case is compared bit-exactly with the CPU oracle, and the test
checks (dvt_launch_count) that the TMA form actually ran -- or, for the shapes it does not take
(odd packet count, pinned host memory), that it did not and the other forms still agree.
"""
import random

import numpy as np
import pytest
import torch

import kvgen
import paper_2403_01876_b200 as dv
from oracle import kvstream as ok

from gpu_util import ctx, flags, sentinel_like, to_dev, to_np, to_pinned

pytestmark = pytest.mark.gpu


@pytest.fixture
def tma_on():
    dv.dvt_tune("DV_TMA", 1)
    yield
    dv.dvt_tune("DV_TMA", dv.TMA_DEFAULT)


def _mk(K, V, lb, rb, layout, hb=0, pinned=False):
    Kp = kvgen.as_ft6d_key(K) if layout == ok.LAYOUT_FT6D else K
    k = to_pinned(Kp) if pinned else to_dev(Kp)
    v = to_pinned(V) if pinned else to_dev(V)
    o = ok.Cache(Kp.copy(), V.copy(), lb, rb, K.shape[2], K.shape[3], K.shape[4], layout, hb)
    return k, v, dv.cache(k, v, lb, rb, head_begin=hb), o


def _case(rng):
    H, D = rng.choice([1, 3, 5]), rng.choice([16, 32, 64, 128, 256])
    nL, nR = rng.randint(1, 3), rng.randint(1, 3)
    S = rng.randint(40, 300)
    hb = rng.randint(0, 3)
    n = rng.randint(32, S)                       # >= 32 positions: the transpose path
    s0 = rng.randint(0, S - n)
    h0 = hb + rng.randint(0, H - 1)
    h1 = rng.randint(h0 + 1, hb + H)
    lb, rb = rng.randint(0, 4), rng.randint(0, 4)
    return H, D, nL, nR, S, hb, lb, rb, (lb, lb + nL, rb, rb + nR, s0, s0 + n, h0, h1)


@pytest.mark.parametrize("seed", range(16))
@pytest.mark.parametrize("layouts", [(ok.LAYOUT_FT6D, ok.LAYOUT_KV5D), (ok.LAYOUT_KV5D, ok.LAYOUT_FT6D)])
def test_tma_transpose_random_shapes(tma_on, seed, layouts):
    """pack, unpack (into a cache with a larger max_seq: the words past the region's end must stay
    untouched -- the tensor map's extent clips the last tile) and a direct remap == the oracle."""
    rng = random.Random(7100 + seed)
    H, D, nL, nR, S, hb, lb, rb, reg = _case(rng)
    K, V = kvgen.kv5d_cache("hash", lb, nL, rb, nR, H, S, D, seed=seed, head_begin=hb)
    k, v, c, o = _mk(K, V, lb, rb, layouts[0], hb=hb)
    n0 = dv.dvt_launch_count("tma_transpose")
    exp = ok.pack(o, reg)
    buf = sentinel_like((exp.size,))
    dv.dv_scatter(ctx(), c, dv.region(*reg), dv.endpoint_of(buf))
    torch.cuda.synchronize()
    assert np.array_equal(to_np(buf), exp)
    S2 = reg[5] + rng.randint(1, 70)
    Ks, Vs = kvgen.sentinel_cache(nL, nR, H, S2, D)
    dk, dvv, dc, do = _mk(Ks, Vs, lb, rb, layouts[1], hb=hb)
    dv.dv_gather(ctx(), dv.endpoint_of(buf), 0, dc, dv.region(*reg))
    torch.cuda.synchronize()
    ok.unpack(do, reg, exp)
    assert np.array_equal(to_np(dk), do.K) and np.array_equal(to_np(dvv), do.V)
    ek, ev, ec, eo = _mk(Ks, Vs, lb, rb, layouts[1], hb=hb)
    dv.dv_remap(ctx(), c, ec, dv.region(*reg))
    torch.cuda.synchronize()
    ok.remap(o, eo, reg)
    assert np.array_equal(to_np(ek), eo.K) and np.array_equal(to_np(ev), eo.V)
    # pack (FT6D source) or unpack (FT6D destination), and the remap, went through the TMA form
    assert dv.dvt_launch_count("tma_transpose") - n0 == 2


@pytest.mark.parametrize("layouts", [(ok.LAYOUT_FT6D, ok.LAYOUT_KV5D), (ok.LAYOUT_KV5D, ok.LAYOUT_FT6D)])
def test_tma_transpose_not_taken_for_odd_packets_or_host(tma_on, layouts):
    """D = 8 (one 16-byte packet per row: U odd) and a pinned-host wire keep the other forms
    (no TMA launch) and still match the oracle."""
    H, nL, nR, S, reg = 3, 2, 2, 80, (0, 2, 0, 2, 5, 77, 0, 0)
    for D, host in ((8, False), (128, True)):
        K, V = kvgen.kv5d_cache("hash", 0, nL, 0, nR, H, S, D, seed=D)
        k, v, c, o = _mk(K, V, 0, 0, layouts[0])
        n0 = dv.dvt_launch_count("tma_transpose")
        exp = ok.pack(o, reg)
        buf = sentinel_like((exp.size,), pinned=host)
        dv.dv_scatter(ctx(), c, dv.region(*reg), dv.endpoint_of(buf), xfer=dv.DV_XFER_FUSED)
        torch.cuda.synchronize()
        assert np.array_equal(to_np(buf), exp)
        Ks, Vs = kvgen.sentinel_cache(nL, nR, H, S, D)
        dk, dvv, dc, do = _mk(Ks, Vs, 0, 0, layouts[1])
        dv.dv_gather(ctx(), dv.endpoint_of(buf), 0, dc, dv.region(*reg), xfer=dv.DV_XFER_FUSED)
        torch.cuda.synchronize()
        ok.unpack(do, reg, exp)
        assert np.array_equal(to_np(dk), do.K) and np.array_equal(to_np(dvv), do.V)
        assert dv.dvt_launch_count("tma_transpose") == n0


def test_tma_transpose_publishes_after_its_stores(tma_on):
    """A remap KV5D -> FT6D (TMA stores on the packet-major side) that releases a flag: a consumer
    stream waits for the flag, then copies the destination -- the copy sees every word (repeated
    over 20 regions, each consumer copy compared with the oracle)."""
    L, B, H, S, D = 2, 2, 4, 288, 128
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=3)
    k, v, c, o = _mk(K, V, 0, 0, ok.LAYOUT_KV5D)
    Ks, Vs = kvgen.sentinel_cache(L, B, H, S, D)
    dk, dvv, dc, do = _mk(Ks, Vs, 0, 0, ok.LAYOUT_FT6D)
    fl = flags(1)
    ep = dv.endpoint_of(torch.empty(64, dtype=torch.int16, device="cuda"), fl)
    cons = torch.cuda.Stream()
    snap = torch.empty_like(dk)
    n0 = dv.dvt_launch_count("tma_transpose")
    for i in range(20):
        reg = (0, L, 0, B, 12 * i, 12 * i + 40)
        dv.dv_remap(ctx(), c, dc, dv.region(*reg), signal=ep, flag_slot=0, seq=i + 1)
        dv.dv_wait(ctx(), ep, 0, i + 1, stream=cons.cuda_stream)
        with torch.cuda.stream(cons):
            snap.copy_(dk)
        cons.synchronize()
        ok.remap(o, do, reg)
        assert np.array_equal(to_np(snap), do.K)
    torch.cuda.synchronize()
    assert dv.dvt_launch_count("tma_transpose") - n0 == 20


def test_tma_transpose_full_size_prompt_layer(tma_on):
    """C2 shape with FT6D keys: a prompt layer (163.8 MB) packed with the TMA form, then unpacked
    into an FT6D cache with another max_seq -- every word checked on the device (dvt_verify), and
    the positions past the prompt in the destination untouched."""
    L, H, D, B, P, S = 3, 40, 128, 8, 1000, 2048
    k6 = torch.empty((L, B, H, D // 8, S, 8), dtype=torch.int16, device="cuda")
    v6 = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    c6 = dv.cache(k6, v6)
    seed = kvgen.config_seed(1)
    dv.dvt_fill(c6, dv.DVT_FILL_HASH, seed=seed)
    reg = dv.region(1, 2, 0, B, 0, P)
    wire = torch.full((2 * B * H * P * D,), -1, dtype=torch.int16, device="cuda")
    n0 = dv.dvt_launch_count("tma_transpose")
    dv.dv_scatter(ctx(), c6, reg, dv.endpoint_of(wire), 0)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    dv.dvt_verify(c6, cnt.data_ptr(), seed=seed, reg=reg, wire_ptr=wire.data_ptr())
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    k2 = torch.full((1, B, H, D // 8, 1536, 8), -1, dtype=torch.int16, device="cuda")
    v2 = torch.full((1, B, H, 1536, D), -1, dtype=torch.int16, device="cuda")
    c2 = dv.cache(k2, v2, 1, 0)
    dv.dv_gather(ctx(), dv.endpoint_of(wire), 0, c2, reg)
    cnt.zero_()
    dv.dvt_verify(c2, cnt.data_ptr(), seed=seed, reg=reg)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    assert int(k2[:, :, :, :, P:].ne(-1).sum()) == 0 and int(v2[:, :, :, P:].ne(-1).sum()) == 0
    assert dv.dvt_launch_count("tma_transpose") - n0 == 2
