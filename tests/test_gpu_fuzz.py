"""Seeded random differential test: hundreds of random operations (level 1/2, KV5D/FT6D on either
side, TP head ranges, fused/staged/auto, device/host endpoints, log chunks, graph-style dynamic
steps) through the C ABI, each compared word for word with the CPU oracle."""
import os
import random

import numpy as np
import pytest
import torch

import kvgen
import paper_2403_01876_b200 as dv
from oracle import kvstream as ok

pytestmark = pytest.mark.gpu

XF = [dv.DV_XFER_AUTO, dv.DV_XFER_FUSED, dv.DV_XFER_STAGED]


def to_dev(a, pinned=False):
    t = torch.from_numpy(np.ascontiguousarray(a).view(np.int16))
    if pinned:
        p = torch.empty(t.shape, dtype=torch.int16, pin_memory=True)
        p.copy_(t)
        return p
    return t.cuda()


def to_np(t):
    return t.cpu().numpy().view(np.uint16)


def mk_cache(rng, lb, nl, rb, nr, hb, nh, S, D, layout, seed, pinned=False, sentinel=False):
    if sentinel:
        K, V = kvgen.sentinel_cache(nl, nr, nh, S, D)
    else:
        K, V = kvgen.kv5d_cache("hash", lb, nl, rb, nr, nh, S, D, seed=seed, head_begin=hb)
    Kp = kvgen.as_ft6d_key(K) if layout == ok.LAYOUT_FT6D else K
    k, v = to_dev(Kp, pinned), to_dev(V, pinned)
    return k, v, dv.cache(k, v, lb, rb, head_begin=hb), ok.Cache(Kp.copy(), V.copy(), lb, rb, nh, S, D, layout, hb)


def rand_region(rng, lb, nl, rb, nr, hb, nh, S):
    l0 = rng.randint(lb, lb + nl - 1); l1 = rng.randint(l0 + 1, lb + nl)
    r0 = rng.randint(rb, rb + nr - 1); r1 = rng.randint(r0 + 1, rb + nr)
    s0 = rng.randint(0, S - 1); s1 = rng.randint(s0 + 1, min(S, s0 + rng.choice([1, 2, 5, 40, S])))
    if rng.random() < 0.5:
        return (l0, l1, r0, r1, s0, s1, 0, 0)
    h0 = rng.randint(hb, hb + nh - 1); h1 = rng.randint(h0 + 1, hb + nh)
    return (l0, l1, r0, r1, s0, s1, h0, h1)


# DV_FUZZ_SCALE=k multiplies the number of seeded blocks (a long stress run; default 1)
_SCALE = max(1, int(os.environ.get("DV_FUZZ_SCALE", "1")))


@pytest.mark.parametrize("block", list(range(18)) + list(range(1000, 1000 + 18 * (_SCALE - 1))))
def test_random_ops_against_oracle(block):
    """Blocks 12..17 draw the less common head dims: 8 (one 16-byte packet), 40 / 80 (5 / 10
    packets: odd register-transpose groups, PK 1 / 2), 96 (PK 4) and 256 (32 packets, PK 16 x 2)."""
    rng = random.Random(12345 + block)
    cx = dv.dv_create(0, staging_bytes=rng.choice([1 << 20, 8 << 20, 0]))
    for it in range(40):
        D = rng.choice([16, 64, 128] if (block < 12 or (block >= 1000 and block % 3)) else [8, 40, 80, 96, 256])
        nl, nr, nh = rng.randint(1, 4), rng.randint(1, 3), rng.randint(1, 5)
        lb, rb, hb = rng.randint(0, 5), rng.randint(0, 5), rng.randint(0, 3)
        S = rng.randint(4, 48)
        lay = [rng.choice([ok.LAYOUT_KV5D, ok.LAYOUT_FT6D]) for _ in range(2)]
        seed = rng.randint(0, 1 << 30)
        op = rng.choice(["scatter_gather", "remap", "chunks", "dyn"])
        xf = rng.choice(XF)
        host = rng.random() < 0.4
        k, v, c, o = mk_cache(rng, lb, nl, rb, nr, hb, nh, S, D, lay[0], seed, pinned=(op == "remap" and host))
        reg = rand_region(rng, lb, nl, rb, nr, hb, nh, S)
        # destination: superset cache with other offsets / max_seq / layout
        S2 = (S if op == "chunks" else reg[5]) + rng.randint(0, 8)
        dk, dvv, dc, do = mk_cache(rng, lb, nl, rb, nr, hb, nh, S2, D, lay[1], 0, sentinel=True,
                                   pinned=(op == "remap" and not host and rng.random() < 0.5))
        ctx_info = (block, it, op, xf, host, lay, reg)
        if op in ("scatter_gather", "dyn"):
            words = ok.region_bytes(reg[0], reg[1], reg[2], reg[3], reg[4], reg[5],
                                    (reg[7] - reg[6]) if reg[7] > reg[6] else nh, D, 2) // 2
            if op == "dyn":
                kmax = S - reg[5]
                kk = rng.randint(0, kmax) if kmax > 0 else 0
                buf = torch.full(((kmax + 1) * words,), -1, dtype=torch.int16, device="cuda")
                d_step = torch.tensor([kk], dtype=torch.int32, device="cuda")
                dv.dv_scatter_dyn(cx, c, dv.region(*reg), dv.endpoint_of(buf), 0, words * 2, d_step.data_ptr(), kmax)
                torch.cuda.synchronize()
                sreg = ok.shifted(reg, kk)
                got = to_np(buf)
                assert np.array_equal(got[kk * words:(kk + 1) * words], ok.pack(o, sreg)), ctx_info
                continue
            buf = (torch.full((words + 8,), -1, dtype=torch.int16, pin_memory=True) if host
                   else torch.full((words + 8,), -1, dtype=torch.int16, device="cuda"))
            dv.dv_scatter(cx, c, dv.region(*reg), dv.endpoint_of(buf), 16, xfer=xf)
            torch.cuda.synchronize()
            exp = ok.pack(o, reg)
            assert np.array_equal(to_np(buf)[8:8 + words], exp), ctx_info
            dv.dv_gather(cx, dv.endpoint_of(buf), 16, dc, dv.region(*reg), xfer=xf)
            torch.cuda.synchronize()
            ok.unpack(do, reg, exp)
        elif op == "remap":
            dv.dv_remap(cx, c, dc, dv.region(*reg), xfer=xf)
            torch.cuda.synchronize()
            ok.remap(o, do, reg)
        else:  # chunks: a log of single- or multi-position chunks
            n = reg[5] - reg[4]
            step = n + rng.randint(0, 2)
            nck = max(1, (S - reg[5]) // step + 1)
            first = reg
            log_np = np.concatenate([ok.pack(o, ok.shifted(first, kq * step)) for kq in range(nck)])
            log = to_dev(log_np, pinned=host)
            dv.dv_gather_chunks(cx, dv.endpoint_of(log), 0, dc, dv.region(*first), nck, step, xfer=xf)
            torch.cuda.synchronize()
            ok.unpack_chunks(do, first, log_np, nck, step)
        assert np.array_equal(to_np(dk), do.K) and np.array_equal(to_np(dvv), do.V), ctx_info
    cx.close()


def _bounds(rng, lo, hi, k):
    cuts = sorted(rng.sample(range(lo + 1, hi), k - 1)) if k > 1 else []
    return [lo] + cuts + [hi]


@pytest.mark.parametrize("block", list(range(8)) + list(range(1000, 1000 + 8 * (_SCALE - 1))))
def test_random_stream_out_in_against_oracle(block):
    """Random pipeline setups on both sides (layer partitions, microbatch splits, optional TP head
    splits, either cache layout per block), inbox (device or pinned host) or direct form."""
    rng = random.Random(777 + block)
    cx = dv.dv_create(0)
    for it in range(6):
        D = rng.choice([16, 64])
        L, R, Hn = rng.randint(1, 8), rng.randint(1, 4), rng.randint(1, 6)
        tp = rng.random() < 0.5
        sl, dl = _bounds(rng, 0, L, rng.randint(1, min(L, 3))), _bounds(rng, 0, L, rng.randint(1, min(L, 3)))
        sr, dr = _bounds(rng, 0, R, rng.randint(1, min(R, 2))), _bounds(rng, 0, R, rng.randint(1, min(R, 2)))
        sh = _bounds(rng, 0, Hn, rng.randint(1, min(Hn, 3))) if tp else None
        dh = _bounds(rng, 0, Hn, rng.randint(1, min(Hn, 3))) if tp else None
        S1, S2 = rng.randint(4, 24), rng.randint(4, 24)
        p = rng.randint(1, min(S1, S2))
        ps, ts = ok.Setup(sl, sr, S1, sh), ok.Setup(dl, dr, S2, dh)
        dps, dts = dv.Setup(sl, sr, S1, sh), dv.Setup(dl, dr, S2, dh)
        seed = rng.randint(0, 1 << 30)
        form = rng.choice(["inbox_dev", "inbox_host", "direct"])
        xf = rng.choice(XF + [dv.DV_XFER_DECOUPLED])   # decoupled: flags are the only completion

        def blocks(s, lb_, rb_, hb_):
            hbs = hb_ if hb_ is not None else [0, Hn]
            for i in range(len(lb_) - 1):
                for u in range(len(rb_) - 1):
                    for t in range(len(hbs) - 1):
                        key = (i, u, t) if hb_ is not None else (i, u)
                        yield key, (i, u, t), lb_[i], lb_[i + 1] - lb_[i], rb_[u], rb_[u + 1] - rb_[u], hbs[t], hbs[t + 1] - hbs[t]
        src, osrc, dst, odst = {}, {}, {}, {}
        for key, (i, u, t), a, nl, c0, nr, h0, nh in blocks(ps, sl, sr, sh):
            k, v, c, o = mk_cache(rng, a, nl, c0, nr, h0, nh, S1, D, rng.choice([0, 1]), seed)
            src[key], osrc[key] = (k, v, c, (i, u, t)), o
        for key, (j, w, t), a, nl, c0, nr, h0, nh in blocks(ts, dl, dr, dh):
            k, v, c, o = mk_cache(rng, a, nl, c0, nr, h0, nh, S2, D, rng.choice([0, 1]), 0, sentinel=True)
            dst[key], odst[key] = (k, v, c, (j, w, t)), o
        reg = (0, L, 0, R, 0, p)
        dkeys = sorted(dst, key=lambda kk: dts.flat(*dst[kk][3]))
        nsrc = ps.n_stages * ps.n_micro * ps.n_tp
        keep = []
        if form == "direct":
            caches = [dst[kk][2] for kk in dkeys]
            for key, (k, v, c, (i, u, t)) in src.items():
                dv.dv_stream_out_direct(cx, c, dv.region(*reg), dps, i, u, dts, caches, None, seq=1, my_tp=t)
        else:
            eps = []
            for kk in dkeys:
                c = dst[kk][2]
                words = c.n_layers * 2 * c.n_reqs * c.n_heads * p * D
                buf = (torch.full((words,), -1, dtype=torch.int16, pin_memory=True) if form == "inbox_host"
                       else torch.full((words,), -1, dtype=torch.int16, device="cuda"))
                fl = (torch.zeros(nsrc, dtype=torch.int64, pin_memory=True) if form == "inbox_host"
                      else torch.zeros(nsrc, dtype=torch.int64, device="cuda"))
                keep += [buf, fl]
                eps.append(dv.endpoint_of(buf, fl))
            for key, (k, v, c, (i, u, t)) in src.items():
                dv.dv_stream_out(cx, c, dv.region(*reg), dps, i, u, dts, eps, seq=1, xfer=xf, my_tp=t)
            for n_, kk in enumerate(dkeys):
                j, w, t = dst[kk][3]
                dv.dv_stream_in(cx, dst[kk][2], dv.region(*reg), dps, dts, j, w, eps[n_], 1, xfer=xf, my_tp=t)
        torch.cuda.synchronize()
        ok.stream(osrc, ps, odst, ts, reg)
        for kk in dst:
            k, v = dst[kk][0], dst[kk][1]
            assert np.array_equal(to_np(k), odst[kk].K) and np.array_equal(to_np(v), odst[kk].V), \
                (block, it, form, xf, sl, dl, sr, dr, sh, dh, kk)
    cx.close()


@pytest.mark.parametrize("block", list(range(6)) + list(range(1000, 1000 + 6 * (_SCALE - 1))))
def test_random_ring_pipelines_against_oracle(block):
    """Random pipelines streaming T token rounds (one position each) through RING inboxes of random
    depth (1..3 slots, include/dv.h) with per-source credits in device or pinned-host memory;
    every source block sends on its own stream, the receivers on another, with random stalls on
    both sides (the credits must hold the senders back). The final token caches equal the
    oracle's stream of the whole region."""
    rng = random.Random(4242 + block)
    cx = dv.dv_create(0)
    for it in range(3):
        D = rng.choice([16, 64])
        L, R, Hn = rng.randint(1, 6), rng.randint(1, 3), rng.randint(1, 4)
        sl, dl = _bounds(rng, 0, L, rng.randint(1, min(L, 3))), _bounds(rng, 0, L, rng.randint(1, min(L, 3)))
        sr, dr = _bounds(rng, 0, R, rng.randint(1, min(R, 2))), _bounds(rng, 0, R, rng.randint(1, min(R, 2)))
        T, p = rng.randint(4, 12), rng.randint(0, 4)
        S = p + T + rng.randint(0, 3)
        ps, ts = ok.Setup(sl, sr, S), ok.Setup(dl, dr, S)
        dps, dts = dv.Setup(sl, sr, S), dv.Setup(dl, dr, S)
        seed = rng.randint(0, 1 << 30)
        depth = rng.randint(1, 3)
        host = rng.random() < 0.5
        xf = rng.choice([dv.DV_XFER_FUSED, dv.DV_XFER_AUTO, dv.DV_XFER_DECOUPLED] if host else
                        [dv.DV_XFER_FUSED, dv.DV_XFER_AUTO])
        src, osrc, dst, odst = {}, {}, {}, {}
        for i in range(len(sl) - 1):
            for u in range(len(sr) - 1):
                k, v, c, o = mk_cache(rng, sl[i], sl[i + 1] - sl[i], sr[u], sr[u + 1] - sr[u], 0, Hn, S, D,
                                      rng.choice([0, 1]), seed)
                src[(i, u)], osrc[(i, u)] = (k, v, c), o
        for j in range(len(dl) - 1):
            for w in range(len(dr) - 1):
                k, v, c, o = mk_cache(rng, dl[j], dl[j + 1] - dl[j], dr[w], dr[w + 1] - dr[w], 0, Hn, S, D,
                                      rng.choice([0, 1]), 0, sentinel=True)
                dst[(j, w)], odst[(j, w)] = (k, v, c), o
        nsrc = len(src)
        eps, keep = {}, []
        for (j, w), (k, v, c) in dst.items():
            slot = c.n_layers * 2 * c.n_reqs * Hn * D * 2          # one position of this block
            mk = (lambda n, dt: torch.zeros(n, dtype=dt, pin_memory=True)) if host else \
                 (lambda n, dt: torch.zeros(n, dtype=dt, device="cuda"))
            buf, fl, cr = mk(depth * slot // 2, torch.int16), mk(nsrc, torch.int64), mk(nsrc, torch.int64)
            keep += [buf, fl, cr]
            eps[(j, w)] = dv.endpoint_of(buf, fl, n_slots=depth, slot_bytes=slot, credits=cr)
        dorder = sorted(dst, key=lambda kk: dts.flat(*kk))
        ep_list = [eps[kk] for kk in dorder]
        s_send = {key: torch.cuda.Stream() for key in src}
        s_recv = torch.cuda.Stream()
        torch.cuda.synchronize()
        for t in range(1, T + 1):
            reg = dv.region(0, L, 0, R, p + t - 1, p + t)
            for (i, u), (k, v, c) in src.items():
                if rng.random() < 0.15:
                    dv.dvt_spin(rng.randint(20_000, 200_000), 1, stream=s_send[(i, u)].cuda_stream)
                dv.dv_stream_out(cx, c, reg, dps, i, u, dts, ep_list, seq=t, xfer=xf,
                                 stream=s_send[(i, u)].cuda_stream)
            if rng.random() < 0.3:
                dv.dvt_spin(rng.randint(20_000, 300_000), 1, stream=s_recv.cuda_stream)
            for (j, w) in dorder:
                dv.dv_stream_in(cx, dst[(j, w)][2], reg, dps, dts, j, w, eps[(j, w)], t, stream=s_recv.cuda_stream)
        torch.cuda.synchronize()
        ok.stream(osrc, ps, odst, ts, (0, L, 0, R, p, p + T))
        for kk in dst:
            k, v = dst[kk][0], dst[kk][1]
            assert np.array_equal(to_np(k), odst[kk].K) and np.array_equal(to_np(v), odst[kk].V), \
                (block, it, depth, host, xf, sl, dl, sr, dr, kk)
    cx.close()
