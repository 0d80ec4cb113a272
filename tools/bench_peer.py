"""Peer (NVLink) workloads for bench.py: one process per GPU, CUDA-IPC-mapped destinations.

  C5 ring (BASELINE.json configs[4]): OPT-66B shape (72 heads, head_dim 128), b 16, P = N stages
     of 64/N layers (8 layers at N = 1, loopback); after the prompt (p = 1024) every token step
     each stage streams its new K/V (all its layers, one position) into the replica store it
     keeps at (x+1)%P with dv_stream_out_direct and a seq flag in the successor's
     memory. One STEP = one token step of every stage.
  C3 disaggregation (configs[2]): OPT-66B, b 8, p 1000; N/2 prompt GPUs -> N/2 token GPUs with a
     different layer partition (S 1024 -> 2048); one STEP = one prompt's full hand-off, layer by
     layer (Opt 2), straight into the token GPUs' caches. N = 1: both sides on one GPU (loopback).

Both print the same JSON contract line as bench.py's default workload (metric = aggregate GB/s of
KV bytes delivered, time = max over ranks).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

H, D = 72, 128


def _env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("DV_BENCH_SAME_DEVICE") == "1":
        local = 0
    return world, rank, local


def _gather(obj, world):
    if world == 1:
        return [obj]
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def _max(x, world, dev, backend):
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sendrecv(args, sbuf, dst, rbuf, src):
    """The baseline's exchange: NCCL grouped send/recv of device buffers; with the gloo backend
    (multi-process tests on one GPU) the same exchange staged through host copies."""
    if args.dist_backend == "nccl":
        ops = []
        if sbuf is not None:
            ops.append(dist.P2POp(dist.isend, sbuf, dst))
        if rbuf is not None:
            ops.append(dist.P2POp(dist.irecv, rbuf, src))
        for r_ in dist.batch_isend_irecv(ops):
            r_.wait()
        return
    torch.cuda.synchronize()
    reqs, rh = [], None
    if sbuf is not None:
        reqs.append(dist.isend(sbuf.cpu(), dst))
    if rbuf is not None:
        rh = torch.empty(rbuf.shape, dtype=rbuf.dtype)
        reqs.append(dist.irecv(rh, src))
    for r_ in reqs:
        r_.wait()
    if rbuf is not None:
        rbuf.copy_(rh)


def _impl(args, baseline):
    if not baseline:
        return "dvstream"
    return "nccl-baseline" if args.dist_backend == "nccl" else "sendrecv-baseline (gloo, host-staged; tests only)"


def run_c5(args, bench):
    world, rank, local = _env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group(args.dist_backend, **({"device_id": dev} if args.dist_backend == "nccl" else {}))
    P = world
    Ls = 64 // P if P > 1 else 8
    b, S, p = 16, 2048, 1024
    ctx = dv.dv_create(local)
    lb = rank * Ls
    own_k = torch.empty((Ls, b, H, S, D), dtype=torch.int16, device=dev)
    own_v = torch.empty_like(own_k)
    own = dv.cache(own_k, own_v, lb, 0)
    dv.dvt_fill(own, dv.DVT_FILL_HASH, seed=20240309)
    # replica store for the predecessor's layers, and the flag word the predecessor publishes
    pred = (rank - 1) % P
    rep_k = torch.full((Ls, b, H, S, D), -1, dtype=torch.int16, device=dev)
    rep_v = torch.full_like(rep_k, -1)
    flags = torch.zeros(P, dtype=torch.int64, device=dev)
    ack = torch.zeros(1, dtype=torch.int64, device=dev)   # the successor's ping-pong acks land here
    torch.cuda.synchronize()
    blob = {"k": dv.dv_ipc_export(rep_k.data_ptr()), "v": dv.dv_ipc_export(rep_v.data_ptr()),
            "f": dv.dv_ipc_export(flags.data_ptr()), "a": dv.dv_ipc_export(ack.data_ptr()),
            "layer_begin": pred * Ls}
    blobs = _gather(blob, world)
    succ = (rank + 1) % P
    sb = blobs[succ]
    kp, vp, fp = dv.dv_ipc_open(sb["k"]), dv.dv_ipc_open(sb["v"]), dv.dv_ipc_open(sb["f"])
    rep_at_succ = dv.cache_raw(kp, vp, local if world == 1 else succ, 2, sb["layer_begin"], Ls, 0, b, H, S, D)
    sig = dv.endpoint(dv.DV_EP_PEER, fp, 8 * P, fp, P, device=succ)
    setup = dv.Setup([rank * Ls, rank * Ls + Ls], [0, b], S)  # this stage as a 1-block "setup"
    st = torch.cuda.current_stream()
    sp = st.cuda_stream

    step_bytes = 2 * Ls * b * H * D * 2
    nccl = getattr(args, "peer_baseline", "none") == "nccl"
    if nccl:
        # BASELINE (north_star: "NCCL send/recv kept only as the baseline"): pack the step into a
        # device buffer, ncclSend it to the successor / ncclRecv the predecessor's, unpack it into
        # the replica store. Needs >= 2 GPUs and the nccl backend.
        assert world > 1, "--peer-baseline nccl needs >= 2 ranks"
        sbuf = torch.empty(step_bytes // 2, dtype=torch.int16, device=dev)
        rbuf = torch.empty_like(sbuf)
        rep_local = dv.cache(rep_k, rep_v, pred * Ls, 0)

    dst_arr, sig_arr = dv.cache_array([rep_at_succ]), dv.endpoint_array([sig])   # reused every step

    def step(t):
        q = p + (t - 1) % (S - p)
        if not nccl:
            dv.dv_stream_out_direct(ctx, own, (lb, lb + Ls, 0, b, q, q + 1), setup, 0, 0, setup,
                                    dst_arr, sig_arr, seq=t, stream=sp)
            return
        dv.dv_scatter(ctx, own, dv.region(lb, lb + Ls, 0, b, q, q + 1), dv.endpoint_of(sbuf), 0, stream=sp)
        _sendrecv(args, sbuf, succ, rbuf, pred)
        dv.dv_gather(ctx, dv.endpoint_of(rbuf), 0, rep_local, dv.region(pred * Ls, pred * Ls + Ls, 0, b, q, q + 1),
                     stream=sp)
    # prompt replica first (bulk, Q13), then token steps
    if not nccl:   # the NCCL baseline times the token steps only
        dv.dv_stream_out_direct(ctx, own, dv.region(lb, lb + Ls, 0, b, 0, p), setup, 0, 0, setup, [rep_at_succ],
                                [sig], seq=1, stream=sp)
    t = 1
    for _ in range(args.warmup):
        t += 1
        step(t)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0, _ = dv.dv_stats()
    a.record(st)
    for _ in range(args.steps):
        t += 1
        step(t)
    e.record(st)
    torch.cuda.synchronize()
    l1, _ = dv.dv_stats()
    ms = _max(a.elapsed_time(e), world, dev, args.dist_backend)
    host_us = None
    dev_us = None
    if not nccl:
        # the same steps queued behind a spin head start: device time per step without the host's
        # enqueue rate (the timed region above includes it: one dv_stream_out_direct per step)
        import time as _t
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dv.dvt_spin(max(2_000_000, args.steps * 40_000), 1, stream=sp)
        a2.record(st)
        h0 = _t.perf_counter()
        for _ in range(args.steps):
            t += 1
            step(t)
        host_us = (_t.perf_counter() - h0) / args.steps * 1e6
        e2.record(st)
        torch.cuda.synchronize()
        dev_us = _max(a2.elapsed_time(e2) * 1e3 / args.steps, world, dev, args.dist_backend)
    graph = None if nccl else _graph_steps(ctx, own, rep_at_succ, sig, lb, Ls, b, p, S, world, dev, args, st)
    pingpong = None if nccl else _pingpong(ctx, own, setup, rep_at_succ, sig, flags, ack, blobs[pred]["a"],
                                           lb, Ls, b, p, S, P, world, dev, args, st)
    # the predecessor's last step landed in our replica store: sampled parity vs kvgen
    if world > 1:
        dist.barrier()
    q = p + (t - 1) % (S - p)
    bad = bench.sample_region(rep_k, rep_v, pred * Ls, 0, H, S, D, (pred * Ls, pred * Ls + Ls, 0, b, q, q + 1),
                              20240309)
    bad = int(_max(bad, world, dev, args.dist_backend))
    value = P * args.steps * step_bytes / (ms * 1e-3) / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": "KV stream GB/s (ring replication, token step per stage)", "value": value, "unit": "GB/s",
            "impl": _impl(args, nccl),
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16 (opaque fp16 words)",
            "data": "synthetic (splitmix64 coordinate-hash fill)",
            "config": {"workload": f"C5 OPT-66B ring replication b16, {P} stage(s) x {Ls} layers, "
                                   f"one position per step -> successor's replica store",
                       "bytes_per_step_per_stage": step_bytes, "parallelism": f"pp{P} ring",
                       "transport": "CUDA IPC peer stores" if world > 1 else "loopback (same GPU)"},
            "gpu_launches": int(l1 - l0), "parity_spot_check": {"mismatches": bad}, "pingpong": pingpong,
            "device_us_per_step": dev_us, "host_enqueue_us_per_step": host_us, "graph": graph,
            "ideal_us_per_step_at_770GBps": step_bytes / 770e3}), flush=True)
    for x in (kp, vp, fp):
        dv.dv_ipc_close(x)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _graph_steps(ctx, own, rep_at_succ, sig, lb, Ls, b, p, S, world, dev, args, st):
    """The token step as a CUDA graph (captured once: a device step counter bump + dv_remap_dyn of
    this stage's new position into the successor's replica store with its seq flag), replayed
    per token: device time and host cost per step."""
    d_step = torch.full((1,), -1, dtype=torch.int32, device=dev)
    g = torch.cuda.CUDAGraph()
    gs = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(gs):
        with torch.cuda.graph(g, stream=gs):
            d_step.add_(1)
            dv.dv_remap_dyn(ctx, own, rep_at_succ, dv.region(lb, lb + Ls, 0, b, p, p + 1), d_step.data_ptr(),
                            S - p - 1, signal=sig, flag_slot=0, seq=2 * 10 ** 7, stream=gs.cuda_stream)
    torch.cuda.synchronize()
    reps = min(args.steps, S - p - 10)
    import time as _t
    with torch.cuda.stream(gs):
        d_step.fill_(-1)
        for _ in range(5):
            g.replay()
        d_step.fill_(-1)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dv.dvt_spin(max(2_000_000, reps * 20_000), 1, stream=gs.cuda_stream)
        a.record(gs)
        h0 = _t.perf_counter()
        for _ in range(reps):
            g.replay()
        host_us = (_t.perf_counter() - h0) / reps * 1e6
        e.record(gs)
        torch.cuda.synchronize()
    dev_us = _max(a.elapsed_time(e) * 1e3 / reps, world, dev, args.dist_backend)
    return {"device_us_per_step": dev_us, "host_us_per_step": host_us, "steps": reps,
            "gbs_per_stage": 2 * Ls * b * H * D * 2 / dev_us / 1e3,
            "how": "one captured graph per token step (step-counter bump + dv_remap_dyn), replayed"}


def _pingpong(ctx, own, setup, rep_at_succ, sig, flags, ack, pred_ack_blob, lb, Ls, b, p, S, P, world, dev,
              args, st, iters=500):
    """SURVEY §8(d) peer latency, second form: a ping-pong per token·layer (one layer, one
    position, b 16 = 589,824 B). Every iteration each stage x (1) puts the layer into the replica
    store at (x+1)%P with its seq flag (dv_stream_out_direct), (2) waits on the stream for the flag
    its predecessor puts into its own memory, (3) writes an ack into the predecessor's memory
    (dv_signal over the peer mapping) and (4) waits for its successor's ack. RTT = device time per
    iteration (a spin head start hides the host enqueue); one-way ~ RTT / 2. At N = 1 the peer is
    this GPU (loopback)."""
    pa = dv.dv_ipc_open(pred_ack_blob)
    pred_ack = dv.endpoint(dv.DV_EP_PEER, pa, 8, pa, 1)
    own_ack = dv.endpoint(dv.DV_EP_DEVICE, ack.data_ptr(), 8, ack.data_ptr(), 1)
    inbox = dv.endpoint(dv.DV_EP_DEVICE, flags.data_ptr(), 8 * P, flags.data_ptr(), P)
    sp = st.cuda_stream
    q = S - 1
    base = 10 ** 7

    def one(i):
        layer = lb + i % Ls
        dv.dv_stream_out_direct(ctx, own, dv.region(layer, layer + 1, 0, b, q, q + 1), setup, 0, 0, setup,
                                [rep_at_succ], [sig], seq=base + i, stream=sp)
        dv.dv_wait(ctx, inbox, 0, base + i, stream=sp)
        dv.dv_signal(ctx, pred_ack, 0, base + i, stream=sp)
        dv.dv_wait(ctx, own_ack, 0, base + i, stream=sp)
    for i in range(20):
        one(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dv.dvt_spin(max(4_000_000, iters * 12_000), 1, stream=sp)
    a.record(st)
    for i in range(20, 20 + iters):
        one(i)
    e.record(st)
    torch.cuda.synchronize()
    rtt = _max(a.elapsed_time(e) * 1e3 / iters, world, dev, args.dist_backend)
    if world > 1:
        dist.barrier()
    dv.dv_ipc_close(pa)
    return {"rtt_us": rtt, "one_way_us": rtt / 2, "bytes": 2 * b * H * D * 2, "iters": iters,
            "how": "put+flag -> stream wait on the predecessor's flag -> ack into its memory -> wait own ack; "
                   "device time per iteration, max over ranks"}


def _token_bounds(n):
    return {1: [0, 64], 2: [0, 29, 64], 4: [0, 13, 30, 47, 64]}.get(n) or \
        [round(64 * k / n) for k in range(n + 1)]


def run_c3(args, bench):
    world, rank, local = _env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group(args.dist_backend, **({"device_id": dev} if args.dist_backend == "nccl" else {}))
    b, Sp, St = 8, 1024, 2048
    p = int(os.environ.get("DV_C3_PROMPT", "1000"))   # test hook: shorter prompts (C3 is p = 1000)
    n_p = max(1, world // 2)
    n_t = max(1, world - n_p) if world > 1 else 1
    pb = [round(64 * k / n_p) for k in range(n_p + 1)]
    tb = _token_bounds(n_t)
    ps, ts = dv.Setup(pb, [0, b], Sp), dv.Setup(tb, [0, b], St)
    ctx = dv.dv_create(local)
    is_prompt = world == 1 or rank < n_p
    is_token = world == 1 or rank >= n_p
    mine = {}
    blob = None
    if is_token:
        j = 0 if world == 1 else rank - n_p
        k = torch.full((tb[j + 1] - tb[j], b, H, St, D), -1, dtype=torch.int16, device=dev)
        v = torch.full_like(k, -1)
        f = torch.zeros(n_p, dtype=torch.int64, device=dev)
        mine.update(tk=k, tv=v, tf=f, j=j)
        torch.cuda.synchronize()
        blob = {"k": dv.dv_ipc_export(k.data_ptr()), "v": dv.dv_ipc_export(v.data_ptr()),
                "f": dv.dv_ipc_export(f.data_ptr()), "j": j}
    if world == 1:
        blobs = [blob]
    else:
        blobs = [x for x in _gather(blob, world) if x is not None]
    blobs.sort(key=lambda x: x["j"])
    if is_prompt:
        i = 0 if world == 1 else rank
        pk = torch.empty((pb[i + 1] - pb[i], b, H, Sp, D), dtype=torch.int16, device=dev)
        pv = torch.empty_like(pk)
        pc = dv.cache(pk, pv, pb[i], 0)
        dv.dvt_fill(pc, dv.DVT_FILL_HASH, seed=20240306, valid=(0, p))
        caches, sigs, opened = [], [], []
        for bl in blobs:
            kp, vp, fp = dv.dv_ipc_open(bl["k"]), dv.dv_ipc_open(bl["v"]), dv.dv_ipc_open(bl["f"])
            opened += [kp, vp, fp]
            jj = bl["j"]
            caches.append(dv.cache_raw(kp, vp, local, 2, tb[jj], tb[jj + 1] - tb[jj], 0, b, H, St, D))
            sigs.append(dv.endpoint(dv.DV_EP_PEER, fp, 8 * n_p, fp, n_p, device=local))
        mine.update(pc=pc, i=i, caches=caches, sigs=sigs, opened=opened)
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    seq = [0]
    nccl = getattr(args, "peer_baseline", "none") == "nccl"
    if nccl:
        # BASELINE: each prompt layer packed into a device buffer, sent with NCCL
        # to the token rank that holds the layer, received and unpacked there.
        assert world > 1, "--peer-baseline nccl needs >= 2 ranks"
        lbytes = 2 * b * H * p * D * 2
        xbuf = torch.empty(lbytes // 2, dtype=torch.int16, device=dev)
        if is_token:
            j = mine["j"]
            mine["tc"] = dv.cache(mine["tk"], mine["tv"], tb[j], 0)

    def owner(bounds, layer):
        return max(x for x in range(len(bounds) - 1) if bounds[x] <= layer)

    def handoff():
        seq[0] += 1
        if nccl:
            if is_prompt:
                i = mine["i"]
                for layer in range(pb[i], pb[i + 1]):
                    dv.dv_scatter(ctx, mine["pc"], dv.region(layer, layer + 1, 0, b, 0, p), dv.endpoint_of(xbuf), 0,
                                  stream=sp)
                    _sendrecv(args, xbuf, n_p + owner(tb, layer), None, None)
            else:
                j = mine["j"]
                for layer in range(tb[j], tb[j + 1]):
                    _sendrecv(args, None, None, xbuf, owner(pb, layer))
                    dv.dv_gather(ctx, dv.endpoint_of(xbuf), 0, mine["tc"], dv.region(layer, layer + 1, 0, b, 0, p),
                                 stream=sp)
            return
        if is_prompt:
            i = mine["i"]
            for layer in range(pb[i], pb[i + 1]):      # layer by layer (Opt 2)
                dv.dv_stream_out_direct(ctx, mine["pc"], dv.region(layer, layer + 1, 0, b, 0, p), ps, i, 0, ts,
                                        mine["caches"], mine["sigs"], seq=seq[0], stream=sp)
    for _ in range(args.warmup):
        handoff()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(args.steps):
        handoff()
    e.record(st)
    torch.cuda.synchronize()
    ms = _max(a.elapsed_time(e), world, dev, args.dist_backend)
    if world > 1:
        dist.barrier()
    bad = 0
    if is_token:
        j = mine["j"]
        bad = bench.sample_region(mine["tk"], mine["tv"], tb[j], 0, H, St, D, (tb[j], tb[j + 1], 0, b, 0, p),
                                  20240306)
    bad = int(_max(bad, world, dev, args.dist_backend))
    total = 64 * 2 * b * H * p * D * 2
    if rank == 0:
        print(json.dumps({
            "metric": "KV stream GB/s (prompt-token disaggregation hand-off)", "value": args.steps * total / (ms * 1e-3) / 1e9,
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u16 (opaque fp16 words)",
            "data": "synthetic (splitmix64 coordinate-hash fill)",
            "config": {"workload": f"C3 OPT-66B b8 p1000: {n_p} prompt GPU(s) {pb} -> {n_t} token GPU(s) {tb}, "
                                   f"S 1024 -> 2048, layer by layer, direct remap",
                       "bytes_per_step": total, "parallelism": f"pp{n_p} -> pp{n_t}",
                       "transport": "CUDA IPC peer stores" if world > 1 else "loopback (same GPU, HBM)"},
            "parity_spot_check": {"mismatches": bad}, "impl": _impl(args, nccl),
            "ideal_ms_per_step_at_770GBps_per_prompt_gpu": total / n_p / 770e6}), flush=True)
    for x in mine.get("opened", []):
        dv.dv_ipc_close(x)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
