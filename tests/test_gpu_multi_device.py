"""Cross-GPU correctness in ONE process driving two GPUs (dv_peer_enable, NVLink P2P): run only
on boxes with >= 2 GPUs (skipped on the one-GPU test box; the multi-process forms are in
test_multiproc.py::test_cross_gpu_processes, and bench.py --gpus N's "nvlink" suite verifies every
delivered word across processes on N GPUs). SURVEY §8(e); PAPER.md:266 (hand-off), :286-290
(replication / recovery)."""
import threading
import time

import numpy as np
import pytest
import torch

import kvgen
import paper_2403_01876_b200 as dv
from oracle import kvstream as ok

from gpu_util import to_np

# the second GPU; DV_MULTIDEV_LOOPBACK=1 runs these tests on a one-GPU box with both "devices" = 0
# (checks the tests themselves; the claims need two GPUs)
import os  # noqa: E402
_LOOP = os.environ.get("DV_MULTIDEV_LOOPBACK") == "1"
G1 = 1 if torch.cuda.device_count() >= 2 else 0
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2 and not _LOOP,
                                 reason="needs >= 2 GPUs (NVLink peer paths)")]


def _dev(a, d):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(f"cuda:{d}")


@pytest.fixture(scope="module")
def ctxs():
    dv.dv_peer_enable(0, G1)
    dv.dv_peer_enable(G1, 0)
    c = [dv.dv_create(0), dv.dv_create(G1)]
    yield c
    for x in c:
        x.close()


@pytest.mark.parametrize("form", ["inbox-fused", "inbox-copy-engine", "direct", "direct-ft6d"])
def test_peer_stream_two_devices(ctxs, form):
    """Source cache on GPU 0, destination (inbox or cache) on GPU 1: dv_stream_out from GPU 0 into
    GPU 1's memory (SM stores or copy engine over NVLink, system-scope release), dv_stream_in on
    GPU 1 -- equal to the oracle's stream (a layer split 2 -> 3 stages, S 40 -> 64)."""
    L, B, H, S, D, S2 = 6, 2, 4, 40, 32, 64
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=501)
    ps, ts = dv.Setup([0, 3, 6], [0, B], S), dv.Setup([0, 2, 4, 6], [0, B], S2)
    reg = dv.region(0, L, 0, B, 0, S)
    ft6d = form == "direct-ft6d"
    src = []
    for i, (a, b) in enumerate(((0, 3), (3, 6))):
        k, v = _dev(K[a:b], 0), _dev(V[a:b], 0)
        src.append((k, v, dv.cache(k, v, a, 0)))
    dst = []
    for j, (a, b) in enumerate(((0, 2), (2, 4), (4, 6))):
        shape = (b - a, B, H, S2, D)
        kshape = (b - a, B, H, D * 2 // 16, S2, 8) if ft6d else shape
        k = torch.full(kshape, -1, dtype=torch.int16, device=f"cuda:{G1}")
        v = torch.full(shape, -1, dtype=torch.int16, device=f"cuda:{G1}")
        dst.append((k, v, dv.cache(k, v, a, 0)))
    flags = torch.zeros((3, 2), dtype=torch.int64, device=f"cuda:{G1}")
    s0 = torch.cuda.Stream(device=0)
    s1 = torch.cuda.Stream(device=G1)
    if form.startswith("inbox"):
        inboxes, eps = [], []
        for j in range(3):
            n = ok.region_bytes(ts.layer_bounds[j], ts.layer_bounds[j + 1], 0, B, 0, S, H, D, 2)
            ib = torch.empty(n // 2, dtype=torch.int16, device=f"cuda:{G1}")
            inboxes.append(ib)
            eps.append(dv.endpoint(dv.DV_EP_PEER, ib.data_ptr(), n, flags[j].data_ptr(), 2, device=G1))
        xf = dv.DV_XFER_FUSED if form == "inbox-fused" else dv.DV_XFER_STAGED
        for i in range(2):
            if G1 != 0:   # another GPU's memory: system-scope release
                assert not dv.dvt_release_scope(ctxs[0], eps[0].flags, eps[0].base)
            dv.dv_stream_out(ctxs[0], src[i][2], reg, ps, i, 0, ts, eps, seq=7, xfer=xf, stream=s0)
        for j in range(3):
            ep1 = dv.endpoint(dv.DV_EP_DEVICE, inboxes[j].data_ptr(), eps[j].bytes, flags[j].data_ptr(), 2, device=G1)
            dv.dv_stream_in(ctxs[1], dst[j][2], reg, ps, ts, j, 0, ep1, 7, stream=s1)
    else:
        sigs = [dv.endpoint(dv.DV_EP_PEER, flags[j].data_ptr(), 16, flags[j].data_ptr(), 2, device=G1) for j in range(3)]
        for i in range(2):
            dv.dv_stream_out_direct(ctxs[0], src[i][2], reg, ps, i, 0, ts, [d[2] for d in dst], sigs, seq=7, stream=s0)
        ep1 = [dv.endpoint(dv.DV_EP_DEVICE, flags[j].data_ptr(), 16, flags[j].data_ptr(), 2, device=G1) for j in range(3)]
        for pc in dv.dv_route(ps, ts, reg, H, D, 2):     # wait for every (source, destination) piece
            dv.dv_wait(ctxs[1], ep1[pc.dst_stage], pc.src_stage, 7, stream=s1)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(G1)
    odst = {}
    for j, (a, b) in enumerate(((0, 2), (2, 4), (4, 6))):
        Ks, Vs = kvgen.sentinel_cache(b - a, B, H, S2, D)
        odst[(j, 0)] = ok.Cache(kvgen.as_ft6d_key(Ks) if ft6d else Ks, Vs, a, 0, H, S2, D,
                                ok.LAYOUT_FT6D if ft6d else ok.LAYOUT_KV5D)
    osrc = {(0, 0): ok.Cache(K[:3], V[:3], 0, 0, H, S, D), (1, 0): ok.Cache(K[3:], V[3:], 3, 0, H, S, D)}
    ok.stream(osrc, ok.Setup([0, 3, 6], [0, B], S), odst, ok.Setup([0, 2, 4, 6], [0, B], S2), (0, L, 0, B, 0, S))
    for j in range(3):
        assert np.array_equal(to_np(dst[j][0]), odst[(j, 0)].K) and np.array_equal(to_np(dst[j][1]), odst[(j, 0)].V), j
    assert int(flags.max()) == 7


def test_fused_producer_into_the_other_gpu(ctxs):
    """Device plans across GPUs: the producer on GPU 0 (dvt_fill_rows) stores its rows into its
    own cache and, through plan sets (dv_dplan_stream_out_direct), straight into GPU 1's caches of
    another layer partition and max_seq over NVLink, releasing GPU 1's flags (system scope); GPU 1's
    stream waits for every piece, then its caches == oracle.stream."""
    L, B, H, S, D, S2, p = 6, 2, 4, 40, 32, 64, 33
    seed = 503
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=seed, valid_pos=(0, p))
    ps, ts = dv.Setup([0, 3, 6], [0, B], S), dv.Setup([0, 2, 4, 6], [0, B], S2)
    reg = dv.region(0, L, 0, B, 0, p)
    src = []
    for i, (a, b) in enumerate(((0, 3), (3, 6))):
        k = torch.full((b - a, B, H, S, D), -2, dtype=torch.int16, device="cuda:0")
        v = torch.full_like(k, -2)
        src.append((k, v, dv.cache(k, v, a, 0)))
    dst = []
    for j, (a, b) in enumerate(((0, 2), (2, 4), (4, 6))):
        k = torch.full((b - a, B, H, S2, D), -1, dtype=torch.int16, device=f"cuda:{G1}")
        v = torch.full_like(k, -1)
        dst.append((k, v, dv.cache(k, v, a, 0)))
    flags = torch.zeros((3, 2), dtype=torch.int64, device=f"cuda:{G1}")
    sigs = [dv.endpoint(dv.DV_EP_PEER, flags[j].data_ptr(), 16, flags[j].data_ptr(), 2, device=G1) for j in range(3)]
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(G1)
    s0, s1 = torch.cuda.Stream(device=0), torch.cuda.Stream(device=G1)
    sets = []
    for i, (a, b) in enumerate(((0, 3), (3, 6))):
        st = dv.dv_dplan_stream_out_direct(ctxs[0], src[i][2], reg, ps, i, 0, ts, [d[2] for d in dst], sigs, seq=9)
        if G1 != 0:
            assert all(st.plan[q].sys_scope for q in range(st.n))
        sets.append(st)
        with torch.cuda.device(0):
            dv.dvt_fill_rows(src[i][2], seed, dv.region(a, b, 0, B, 0, p), st, 0, stream=s0.cuda_stream)
    ep1 = [dv.endpoint(dv.DV_EP_DEVICE, flags[j].data_ptr(), 16, flags[j].data_ptr(), 2, device=G1) for j in range(3)]
    for pc in dv.dv_route(ps, ts, reg, H, D, 2):
        dv.dv_wait(ctxs[1], ep1[pc.dst_stage], pc.src_stage, 9, stream=s1)
    snaps = []
    with torch.cuda.stream(s1):
        for j in range(3):
            snaps.append((dst[j][0].clone(), dst[j][1].clone()))
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(G1)
    odst = {}
    for j, (a, b) in enumerate(((0, 2), (2, 4), (4, 6))):
        Ks, Vs = kvgen.sentinel_cache(b - a, B, H, S2, D)
        odst[(j, 0)] = ok.Cache(Ks, Vs, a, 0, H, S2, D)
    osrc = {(0, 0): ok.Cache(K[:3], V[:3], 0, 0, H, S, D), (1, 0): ok.Cache(K[3:], V[3:], 3, 0, H, S, D)}
    ok.stream(osrc, ok.Setup([0, 3, 6], [0, B], S), odst, ok.Setup([0, 2, 4, 6], [0, B], S2), (0, L, 0, B, 0, p))
    for j in range(3):   # what GPU 1 saw right after its waits
        assert np.array_equal(to_np(snaps[j][0]), odst[(j, 0)].K) and np.array_equal(to_np(snaps[j][1]), odst[(j, 0)].V), j
    for st in sets:
        dv.dv_dplan_free(ctxs[0], st)


def test_flag_released_on_one_gpu_observed_on_the_other(ctxs):
    """A5 across GPUs: GPU 0 stores a chunk into GPU 1's memory and releases a seq flag there
    (st.release.sys). Three observers must never see the flag before the payload: (1) GPU 1's
    stream (dv_wait) followed by a copy; (2) an in-kernel consumer on GPU 1 spinning with
    system-scope acquire loads (dv_device.cuh via dvt_consume), launched before the producer;
    (3) a host thread polling the flag with dv_query, then reading the payload."""
    n_chunks = 50
    L, B, H, S, D = 4, 4, 8, 64, 64
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=502)
    k, v = _dev(K, 0), _dev(V, 0)
    c = dv.cache(k, v)
    osrc = ok.Cache(K, V, 0, 0, H, S, D)
    chunk = ok.region_bytes(0, L, 0, B, 0, 1, H, D, 2)
    box = torch.full((n_chunks * chunk // 2,), -1, dtype=torch.int16, device=f"cuda:{G1}")
    fl = torch.zeros(1, dtype=torch.int64, device=f"cuda:{G1}")
    ep = dv.endpoint(dv.DV_EP_PEER, box.data_ptr(), n_chunks * chunk, fl.data_ptr(), 1, device=G1)
    ep1 = dv.endpoint(dv.DV_EP_DEVICE, box.data_ptr(), n_chunks * chunk, fl.data_ptr(), 1, device=G1)
    got_stream = torch.empty_like(box)
    got_kernel = torch.empty_like(box)
    ok_k = torch.ones(n_chunks, dtype=torch.int32, device=f"cuda:{G1}")
    s_cons = [torch.cuda.Stream(device=G1) for _ in range(2)]
    host_bad = []
    stop = threading.Event()

    def poller():
        seen = 0
        while seen < n_chunks and not stop.is_set():
            t = seen + 1
            if dv.dv_query(ctxs[1], ep1, 0, t):
                w = box[(t - 1) * chunk // 2:t * chunk // 2].cpu().numpy().view(np.uint16)
                if not np.array_equal(w, ok.pack(osrc, (0, L, 0, B, t - 1, t))):
                    host_bad.append(t)
                seen = t
    # load every kernel this test launches before any consumer spins (CUDA lazy loading would make
    # a first launch wait for the spinning consumers)
    for d in (0, G1):
        with torch.cuda.device(d):
            dv.dvt_spin(1000, 1)
            dv.dvt_consume(fl.data_ptr(), 0, box.data_ptr(), got_kernel.data_ptr(), 16, ok_k.data_ptr())
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(G1)
    for t in range(1, n_chunks + 1):   # consumers first: kernels spin on GPU 1
        o = (t - 1) * chunk
        with torch.cuda.device(G1):        # test-library kernels launch on the current device
            dv.dvt_consume(fl.data_ptr(), t, box.data_ptr() + o, got_kernel.data_ptr() + o, chunk,
                           ok_k[t - 1:t].data_ptr(), timeout_ns=5_000_000_000, stream=s_cons[0])
        dv.dv_wait(ctxs[1], ep1, 0, t, stream=s_cons[1])
        dv.dv_flush(ctxs[1], box.data_ptr() + o, chunk,
                    dv.endpoint(dv.DV_EP_DEVICE, got_stream.data_ptr(), n_chunks * chunk, device=G1), o,
                    xfer=dv.DV_XFER_FUSED, stream=s_cons[1])
    th = threading.Thread(target=poller)
    th.start()
    s0 = torch.cuda.Stream(device=0)
    for t in range(1, n_chunks + 1):
        dv.dvt_spin(20_000, 1, stream=s0)        # chunks trickle out, so observers race each release
        dv.dv_scatter(ctxs[0], c, dv.region(0, L, 0, B, t - 1, t), ep, (t - 1) * chunk, flag_slot=0, seq=t,
                      xfer=dv.DV_XFER_FUSED, stream=s0)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(G1)
    th.join(timeout=30)
    stop.set()
    exp = np.concatenate([ok.pack(osrc, (0, L, 0, B, t - 1, t)) for t in range(1, n_chunks + 1)])
    assert int(fl[0]) == n_chunks
    assert bool((ok_k == 1).all()), "an in-kernel consumer timed out"
    assert np.array_equal(to_np(got_kernel), exp), "in-kernel acquire saw a flag before its payload"
    assert np.array_equal(to_np(got_stream), exp), "stream wait on GPU 1 saw a flag before its payload"
    assert not host_bad, f"host poller saw flags before payload: {host_bad[:5]}"


def test_ring_replication_and_recovery_two_gpus(ctxs):
    """C5 at P = 2 on two GPUs in one process: each stage puts its token steps into the replica
    store on the other GPU; after a simulated failure of stage 1 its cache is rebuilt from the
    replica on GPU 0 (Fig. 10) -- equal to the pre-failure cache."""
    Ls, B, H, S, D, p, T = 3, 2, 4, 48, 32, 16, 12
    caches, reps = [], []
    for x in range(2):
        K, V = kvgen.kv5d_cache("hash", x * Ls, Ls, 0, B, H, S, D, seed=503, valid_pos=(0, p + T))
        k, v = _dev(K, [0, G1][x]), _dev(V, [0, G1][x])
        caches.append((k, v, dv.cache(k, v, x * Ls, 0), K, V))
        pred = (x - 1) % 2
        rk = torch.full((Ls, B, H, S, D), -1, dtype=torch.int16, device=f"cuda:{[0, G1][x]}")
        rv = torch.full_like(rk, -1)
        reps.append((rk, rv, dv.cache(rk, rv, pred * Ls, 0)))
    for x in range(2):
        succ = (x + 1) % 2
        st = torch.cuda.Stream(device=[0, G1][x])
        dv.dv_remap(ctxs[x], caches[x][2], reps[succ][2], dv.region(x * Ls, x * Ls + Ls, 0, B, 0, p), stream=st)
        for t in range(1, T + 1):
            q = p + t - 1
            dv.dv_remap(ctxs[x], caches[x][2], reps[succ][2], dv.region(x * Ls, x * Ls + Ls, 0, B, q, q + 1), stream=st)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(G1)
    for x in range(2):
        succ = (x + 1) % 2
        assert np.array_equal(to_np(reps[succ][0])[:, :, :, :p + T], caches[x][3][:, :, :, :p + T])
        assert np.array_equal(to_np(reps[succ][1])[:, :, :, :p + T], caches[x][4][:, :, :, :p + T])
    # stage 1 fails: its cache is lost; recovery copies the replica held by stage 0 (GPU 0) back
    caches[1][0].fill_(-1)
    caches[1][1].fill_(-1)
    dv.dv_remap(ctxs[0], reps[0][2], caches[1][2], dv.region(Ls, 2 * Ls, 0, B, 0, p + T))
    torch.cuda.synchronize(0)
    assert np.array_equal(to_np(caches[1][0])[:, :, :, :p + T], caches[1][3][:, :, :, :p + T])
    assert np.array_equal(to_np(caches[1][1])[:, :, :, :p + T], caches[1][4][:, :, :, :p + T])
