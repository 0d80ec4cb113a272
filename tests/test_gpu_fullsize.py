"""Parity at BASELINE.json's full sizes, in the launch configurations bench.py and
tools/bench_configs.py time: sampled outputs, each expected word computed one by one from the
oracle's mapping (wire_index for wire chunks, global coordinates for caches) and kvgen's writer
definition. Plus the launch-split path (> max vectors per launch) at a small forced limit.
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import kvgen
import paper_2403_01876_b200 as dv
from oracle import kvstream as ok

pytestmark = pytest.mark.gpu
SEED = 20240399


def _ctx():
    return dv.dv_create(0, staging_bytes=1 << 30)


def _sample_wire(buf_words, region, H, D, seed, n=30000):
    rng = np.random.default_rng(3)
    l0, l1, r0, r1, s0, s1 = region
    l = rng.integers(l0, l1, n); kv = rng.integers(0, 2, n); r = rng.integers(r0, r1, n)
    h = rng.integers(0, H, n); s = rng.integers(s0, s1, n); d = rng.integers(0, D, n)
    idx = np.array([ok.wire_index(region, H, D, int(l[i]), int(kv[i]), int(r[i]), int(h[i]), int(s[i]), int(d[i]))
                    for i in range(n)])
    exp = kvgen.hash_words(kv, l, r, h, s, d, seed)
    it = torch.from_numpy(idx).to(buf_words.device)
    got = buf_words[it].cpu().numpy().view(np.uint16)
    return int(np.sum(got != exp))


def _sample_cache(k, v, c, region, seed, n=30000):
    rng = np.random.default_rng(4)
    l0, l1, r0, r1, s0, s1 = region
    l = rng.integers(l0, l1, n); kv = rng.integers(0, 2, n); r = rng.integers(r0, r1, n)
    h = rng.integers(0, c.n_heads, n); s = rng.integers(s0, s1, n); d = rng.integers(0, c.head_dim, n)
    idx = ((((l - c.layer_begin) * c.n_reqs + (r - c.req_begin)) * c.n_heads + h) * c.max_seq + s) * c.head_dim + d
    it = torch.from_numpy(idx.astype(np.int64)).to(k.device)
    got = np.where(kv == 0, k.view(-1)[it].cpu().numpy().view(np.uint16), v.view(-1)[it].cpu().numpy().view(np.uint16))
    return int(np.sum(got != kvgen.hash_words(kv, l, r, h, s, d, seed)))


class _Verify:
    """Every word, on the device (dvt_verify): the second parity check at full sizes (SURVEY §8(c)
    C-5), beside the sampled oracle comparisons."""

    def __init__(self):
        self.cnt = torch.zeros(1, dtype=torch.int64, device="cuda")

    def __call__(self, c, reg, wire=None, valid=(0, 1 << 30)):
        self.cnt.zero_()
        dv.dvt_verify(c, self.cnt.data_ptr(), seed=SEED, reg=dv.region(*reg),
                      wire_ptr=wire.data_ptr() if wire is not None else 0, valid=valid)
        torch.cuda.synchronize()
        return int(self.cnt.item())


def test_verifier_matches_kvgen_and_detects_one_flipped_word():
    """Pins dvt_verify: a cache filled on the HOST by kvgen verifies clean (device generator ==
    kvgen), its oracle-packed wire verifies clean, and one flipped word anywhere is counted once."""
    L, B, H, S, D = 3, 2, 5, 24, 32
    K, V = kvgen.kv5d_cache("hash", 2, L, 1, B, H, S, D, seed=SEED)
    k = torch.from_numpy(K.view(np.int16)).cuda()
    v = torch.from_numpy(V.view(np.int16)).cuda()
    c = dv.cache(k, v, 2, 1)
    ver = _Verify()
    assert ver(c, (2, 5, 1, 3, 0, S)) == 0
    reg = (3, 5, 1, 3, 4, 19)
    wire = torch.from_numpy(ok.pack(ok.Cache(K, V, 2, 1, H, S, D), reg).view(np.int16)).cuda()
    assert ver(c, reg, wire) == 0
    rng = np.random.default_rng(0)
    for _ in range(5):
        i = int(rng.integers(0, wire.numel()))
        wire[i] ^= 0x10
        assert ver(c, reg, wire) == 1
        wire[i] ^= 0x10
        j = tuple(int(rng.integers(0, n)) for n in k.shape)
        v[j] ^= 1
        assert ver(c, (2, 5, 1, 3, 0, S)) == 1
        v[j] ^= 1


def test_c2_full_size_token_step_and_prompt_layer():
    """C2 (OPT-13B, b8, S2048, 13.4 GB cache): token steps fused and staged, prompt layer fused and
    staged (pipelined), into pinned host -- sampled parity vs oracle mapping + kvgen."""
    L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    c = dv.cache(k, v)
    dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=SEED)
    cx = _ctx()
    ver = _Verify()
    step = 2 * L * B * H * D * 2
    log = torch.full((step,), -1, dtype=torch.int16, pin_memory=True)
    for xf in (dv.DV_XFER_FUSED, dv.DV_XFER_STAGED, dv.DV_XFER_AUTO):
        reg = (0, L, 0, B, P + xf, P + xf + 1)
        dv.dv_scatter(cx, c, dv.region(*reg), dv.endpoint_of(log), 0, xfer=xf)
        torch.cuda.synchronize()
        assert _sample_wire(log, reg, H, D, SEED) == 0
        assert ver(c, reg, log) == 0
    layer = 2 * B * H * P * D * 2
    pbuf = torch.full((layer // 2,), -1, dtype=torch.int16, pin_memory=True)
    for xf in (dv.DV_XFER_FUSED, dv.DV_XFER_STAGED):
        reg = (7 + xf, 8 + xf, 0, B, 0, P)
        dv.dv_scatter(cx, c, dv.region(*reg), dv.endpoint_of(pbuf), 0, xfer=xf)
        torch.cuda.synchronize()
        assert _sample_wire(pbuf, reg, H, D, SEED) == 0
        assert ver(c, reg, pbuf) == 0
    # and back: gather the prompt layer into an S=4096 cache (other max_seq), staged pipelined
    k2 = torch.full((1, B, H, 4096, D), -1, dtype=torch.int16, device="cuda")
    v2 = torch.full_like(k2, -1)
    c2 = dv.cache(k2, v2, 9, 0)
    dv.dv_gather(cx, dv.endpoint_of(pbuf), 0, c2, dv.region(9, 10, 0, B, 0, P))
    torch.cuda.synchronize()
    assert _sample_cache(k2, v2, c2, (9, 10, 0, B, 0, P), SEED) == 0
    assert ver(c2, (9, 10, 0, B, 0, P)) == 0
    assert int(k2[0, :, :, P:].ne(-1).sum()) == 0
    cx.close()


def test_c3_full_size_direct_remap_16_layers():
    H, D, b, p = 72, 128, 8, 1000
    ps = dv.Setup([0, 16, 32, 48, 64], [0, b], 1024)
    ts = dv.Setup([0, 13, 30, 47, 64], [0, b], 2048)
    pk = torch.empty((16, b, H, 1024, D), dtype=torch.int16, device="cuda")
    pv = torch.empty_like(pk)
    pc = dv.cache(pk, pv, 0, 0)
    dv.dvt_fill(pc, dv.DVT_FILL_HASH, seed=SEED, valid=(0, p))
    t0k = torch.full((13, b, H, 2048, D), -1, dtype=torch.int16, device="cuda")
    t0v = torch.full_like(t0k, -1)
    t1k = torch.full((17, b, H, 2048, D), -1, dtype=torch.int16, device="cuda")
    t1v = torch.full_like(t1k, -1)
    c0, c1 = dv.cache(t0k, t0v, 0, 0), dv.cache(t1k, t1v, 13, 0)
    cx = _ctx()
    dv.dv_stream_out_direct(cx, pc, dv.region(0, 16, 0, b, 0, p), ps, 0, 0, ts, [c0, c1, None, None])
    torch.cuda.synchronize()
    assert _sample_cache(t0k, t0v, c0, (0, 13, 0, b, 0, p), SEED) == 0
    assert _sample_cache(t1k, t1v, c1, (13, 16, 0, b, 0, p), SEED) == 0
    ver = _Verify()   # every word of the 4.72 GB hand-off
    assert ver(c0, (0, 13, 0, b, 0, p)) == 0 and ver(c1, (13, 16, 0, b, 0, p)) == 0
    assert int(t0k[:, :, :, p:].ne(-1).sum()) == 0 and int(t1k[3:].ne(-1).sum()) == 0
    cx.close()


def test_c4_full_size_swap_in_from_log():
    H, D, b, S, nL, p0, i = 112, 128, 4, 2048, 9, 1024, 2048
    k = torch.empty((nL, b, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    c = dv.cache(k, v)
    dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=SEED)
    cx = _ctx()
    step_b = 2 * nL * b * H * D * 2
    log = torch.empty(i * step_b // 2, dtype=torch.int16, pin_memory=True)
    ep = dv.endpoint_of(log)
    dv.dv_scatter(cx, c, dv.region(0, nL, 0, b, 0, p0), ep, 0)
    for t in range(i - p0):
        dv.dv_scatter(cx, c, dv.region(0, nL, 0, b, p0 + t, p0 + t + 1), ep, (p0 + t) * step_b)
    sk = torch.full_like(k, -1)
    sv = torch.full_like(v, -1)
    sc = dv.cache(sk, sv)
    dv.dv_gather(cx, ep, 0, sc, dv.region(0, nL, 0, b, 0, p0))
    dv.dv_gather_chunks(cx, ep, p0 * step_b, sc, dv.region(0, nL, 0, b, p0, p0 + 1), i - p0, 1)
    torch.cuda.synchronize()
    assert _sample_cache(sk, sv, sc, (0, nL, 0, b, 0, i), SEED) == 0
    assert _Verify()(sc, (0, nL, 0, b, 0, i)) == 0   # every word of the 4.23 GB prefix
    cx.close()


def test_c5_full_size_replica_token_steps_and_recovery():
    """C5 (OPT-66B, b 16, P = 8 stage shape: 8 layers, S 2048; 9.66 GB per cache) in the form
    bench.py --workload c5 times: prompt replica p = 1024 into the successor's replica store with
    dv_stream_out_direct, then token steps, then the two recovery copies of PAPER.md:288 into wiped
    caches -- sampled parity vs kvgen's definition + every word checked on the device."""
    H, D, b, S, p, Ls, T = 72, 128, 16, 2048, 1024, 8, 6
    lb = 8   # stage x = 1 of 8: layers [8, 16)
    own_k = torch.empty((Ls, b, H, S, D), dtype=torch.int16, device="cuda")
    own_v = torch.empty_like(own_k)
    own = dv.cache(own_k, own_v, lb, 0)
    dv.dvt_fill(own, dv.DVT_FILL_HASH, seed=SEED)
    rep_k = torch.full_like(own_k, -1)
    rep_v = torch.full_like(own_v, -1)
    rep = dv.cache(rep_k, rep_v, lb, 0)
    fl = torch.zeros(1, dtype=torch.int64, device="cuda")
    sig = dv.endpoint(dv.DV_EP_DEVICE, fl.data_ptr(), 8, fl.data_ptr(), 1)
    setup = dv.Setup([lb, lb + Ls], [0, b], S)
    cx = _ctx()
    dv.dv_stream_out_direct(cx, own, dv.region(lb, lb + Ls, 0, b, 0, p), setup, 0, 0, setup, [rep], [sig], seq=1)
    for t in range(1, T + 1):
        dv.dv_stream_out_direct(cx, own, dv.region(lb, lb + Ls, 0, b, p + t - 1, p + t), setup, 0, 0, setup,
                                [rep], [sig], seq=1 + t)
    torch.cuda.synchronize()
    n = p + T
    assert int(fl[0]) == 1 + T
    assert _sample_cache(rep_k, rep_v, rep, (lb, lb + Ls, 0, b, 0, n), SEED) == 0
    ver = _Verify()
    assert ver(rep, (lb, lb + Ls, 0, b, 0, n)) == 0
    assert int(rep_k[:, :, :, n:].ne(-1).sum()) == 0
    # recovery (NEXT-3): the failed stage's own cache comes back from the replica
    own_k.fill_(-1)
    own_v.fill_(-1)
    dv.dv_remap(cx, rep, own, dv.region(lb, lb + Ls, 0, b, 0, n))
    torch.cuda.synchronize()
    assert _sample_cache(own_k, own_v, own, (lb, lb + Ls, 0, b, 0, n), SEED) == 0
    assert ver(own, (lb, lb + Ls, 0, b, 0, n)) == 0
    cx.close()


def test_ft6d_full_size_prompt_layer_pack_and_remap():
    """C2 shape with FasterTransformer's 6-D keys (NEXT-1): a prompt layer (163.8 MB) packed through
    the register packet transpose, and remapped FT6D -> KV5D into a cache with another max_seq --
    sampled parity vs the oracle's wire order and kvgen + every word on the device."""
    L, H, D, B, P, S = 4, 40, 128, 8, 1000, 2048
    k6 = torch.empty((L, B, H, D // 8, S, 8), dtype=torch.int16, device="cuda")
    v6 = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    c6 = dv.cache(k6, v6)
    dv.dvt_fill(c6, dv.DVT_FILL_HASH, seed=SEED)
    cx = _ctx()
    reg = (2, 3, 0, B, 0, P)
    wire = torch.full((2 * B * H * P * D,), -1, dtype=torch.int16, device="cuda")
    dv.dv_scatter(cx, c6, dv.region(*reg), dv.endpoint_of(wire), 0)
    torch.cuda.synchronize()
    assert _sample_wire(wire, reg, H, D, SEED) == 0
    ver = _Verify()
    assert ver(c6, reg, wire) == 0
    k5 = torch.full((1, B, H, 1536, D), -1, dtype=torch.int16, device="cuda")
    v5 = torch.full_like(k5, -1)
    c5 = dv.cache(k5, v5, 2, 0)
    dv.dv_remap(cx, c6, c5, dv.region(*reg))
    torch.cuda.synchronize()
    assert _sample_cache(k5, v5, c5, reg, SEED) == 0
    assert ver(c5, reg) == 0
    assert int(k5[:, :, :, P:].ne(-1).sum()) == 0
    cx.close()


def test_launch_split_path_matches_oracle():
    """Copies larger than the per-launch vector limit are split at run boundaries; forced here with
    DV_MAX_VEC=1000 in a subprocess (the limit is read once per process)."""
    code = r'''
import numpy as np, torch, kvgen, paper_2403_01876_b200 as dv
from oracle import kvstream as ok
L, B, H, S, D = 3, 4, 5, 40, 64
K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=5)
k = torch.from_numpy(K.view(np.int16)).cuda(); v = torch.from_numpy(V.view(np.int16)).cuda()
c = dv.cache(k, v)
reg = (0, L, 0, B, 3, 37)
exp = ok.pack(ok.Cache(K, V, 0, 0, H, S, D), reg)
buf = torch.full((exp.size,), -1, dtype=torch.int16, device="cuda")
fl = torch.zeros(1, dtype=torch.int64, device="cuda")
cx = dv.dv_create(0)
n0, _ = dv.dv_stats()
dv.dv_scatter(cx, c, dv.region(*reg), dv.endpoint_of(buf, fl), 0, flag_slot=0, seq=3)
torch.cuda.synchronize()
n1, _ = dv.dv_stats()
assert np.array_equal(buf.cpu().numpy().view(np.uint16), exp)
assert int(fl[0]) == 3 and n1 - n0 > 1, (n1 - n0)
print("SPLIT_OK", n1 - n0)
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, DV_MAX_VEC="1000"), cwd=root,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "SPLIT_OK" in r.stdout, r.stdout + r.stderr
