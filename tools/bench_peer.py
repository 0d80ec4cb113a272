"""Peer (NVLink) workloads: one process per GPU, CUDA-IPC-mapped destinations.

Used two ways:
  * `bench.py --gpus N` (N > 1, the driver's scaling run) calls `nvlink_suite()` after the C2
    headline: every peer path of north_star measured on the N GPUs of the box, with parity, in the
    SAME JSON line (key "nvlink");
  * `bench.py --workload c3|c5` prints one line for that workload alone (`run_c3` / `run_c5`).

The measurements (all timed on the device with CUDA events, max over ranks):
  link    in-run peer peaks: copy-engine (cudaMemcpyAsync into the successor's IPC-mapped buffer)
          and SM stores (dv_flush FUSED), all ranks sending to (x+1)%N at once (ring) and, for
          N >= 2, even ranks only (one direction per link) -- the roofline denominators;
  C5      ring replication (BASELINE.json configs[4], §4.2.3): OPT-66B shape (72 heads,
          head_dim 128), b 16, P = N stages of 64/N layers. The prompt (p = 1024) is replicated in
          bulk into the successor's replica store (reading Q13), then token steps (one position of
          all the stage's layers per step); per-layer put latency (writer end ->
          system-scope release of the seq flag, %globaltimer) and a ping-pong RTT; NCCL baseline
          (pack -> ncclSend/ncclRecv -> unpack) for the same token steps and the same prompt
          replica; every word of every replica store checked on the device (dvt_verify);
  C4      microbatch swapping on every rank at once (configs[3]): the shared
          host PCIe fabric, per-GPU vs alone, NUMA-local pinned logs;
  C3      prompt->token disaggregation (configs[2], §4.2.1): OPT-66B b 8, p 1000;
          N/2 prompt GPUs (S 1024) hand their prompt KV layer by layer (Opt 2)
          straight into N/2 token GPUs with a different layer partition (S 2048); NCCL baseline
          (per layer pack -> send to the owning token rank -> unpack); every word of every token
          cache checked on the device, and positions >= p still the sentinel.
At N = 1 the same code runs as loopback (the "peer" is this GPU: HBM-bound).
DV_BENCH_PEER_SMALL=1 shrinks the shapes (tests with all ranks on one GPU).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

H, D = 72, 128
NVLINK_NOMINAL_GBS = 900.0          # per direction per GPU (NVLink 5, 18 links; task statement)
NVLINK_GUIDE_GBS = 770.0            # measured peer copy in /opt/skills/guides/B200_PROFILING.md
SEED_C5, SEED_C3 = 20240309, 20240306


def _small():
    return os.environ.get("DV_BENCH_PEER_SMALL") == "1"


class Env:
    """Rank / device / process-group plumbing of one bench process."""

    def __init__(self, backend):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if os.environ.get("DV_BENCH_SAME_DEVICE") == "1":   # test hook: all ranks on cuda:0 (gloo)
            self.local = 0
        self.backend = backend
        self.dev = torch.device("cuda", self.local)

    def init(self):
        torch.cuda.set_device(self.local)
        if self.world > 1 and not dist.is_initialized():
            dist.init_process_group(self.backend, **({"device_id": self.dev} if self.backend == "nccl" else {}))

    def gather(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        dist.all_gather_object(out, obj)
        return out

    def max(self, x):
        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=self.dev if self.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x):
        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=self.dev if self.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def barrier(self):
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def identity(self):
        p = torch.cuda.get_device_properties(self.local)
        return {"rank": self.rank, "device": self.local, "name": p.name,
                "pci": f"{getattr(p, 'pci_domain_id', 0):04x}:{getattr(p, 'pci_bus_id', 0):02x}:"
                       f"{getattr(p, 'pci_device_id', 0):02x}", "uuid": str(getattr(p, "uuid", ""))}


def _timed(env, fn, reps=1, head_start_ns=0):
    """Device time of `reps` calls of fn on the current stream (ms, max over ranks), bracketed by a
    barrier + synchronize on both sides."""
    st = torch.cuda.current_stream()
    env.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if head_start_ns:
        dv.dvt_spin(head_start_ns, 1, stream=st.cuda_stream)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    ms = env.max(a.elapsed_time(b))
    env.barrier()
    return ms


def _sendrecv(backend, sbuf, dst, rbuf, src):
    """The baseline's exchange: NCCL grouped send/recv of device buffers; with the gloo backend
    (multi-process tests on one GPU) the same exchange staged through host copies."""
    if backend == "nccl":
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


def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:   # noqa: BLE001 -- the value this file held on this round's boxes
        return 6550.7


def _roof(achieved, peak, peak_src, env=None):
    """Roofline of a peer copy: NVLink per direction against the in-run peer peak; at N = 1 (or
    every rank on one GPU) the 'peer' is this GPU's own HBM: 2R (read + write) against the HBM copy
    peak."""
    same_gpu = env is not None and (env.world == 1 or os.environ.get("DV_BENCH_SAME_DEVICE") == "1")
    if same_gpu:
        hp = _hbm_peak()
        return {"bound": "hbm (same GPU: loopback / test mode)", "achieved": 2 * achieved, "unit": "GB/s (2R)",
                "peak": hp, "frac": 2 * achieved / hp, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    return {"bound": "nvlink", "achieved": achieved, "unit": "GB/s", "peak": peak,
            "frac": achieved / peak if peak else None, "peak_source": peak_src,
            "peak_nominal": NVLINK_NOMINAL_GBS, "frac_nominal": achieved / NVLINK_NOMINAL_GBS}


def _pct(xs, q):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(len(xs) * q))] if xs else None


# =====================================================================================================
# link probe: the in-run peer peaks
# =====================================================================================================
def link_probe(ctx, env, nbytes=None, reps=5):
    nbytes = nbytes or ((32 << 20) if _small() else (256 << 20))
    W, r = env.world, env.rank
    src = dv.dv_device_alloc(env.local, nbytes)
    dst = dv.dv_device_alloc(env.local, nbytes)
    blobs = env.gather(dv.dv_ipc_export(dst))
    succ = (r + 1) % W
    peer = dv.dv_ipc_open(blobs[succ])
    ep = dv.endpoint(dv.DV_EP_PEER if W > 1 else dv.DV_EP_DEVICE, peer, nbytes, device=succ if W > 1 else env.local)
    sp = torch.cuda.current_stream().cuda_stream
    out = {"bytes": nbytes, "reps": reps, "topology": "ring x -> (x+1)%N, all ranks at once"}
    for name, xf in (("ce", dv.DV_XFER_STAGED), ("sm", dv.DV_XFER_FUSED)):
        ms = _timed(env, lambda: dv.dv_flush(ctx, src, nbytes, ep, 0, xfer=xf, stream=sp), reps)
        out[f"ring_{name}_gbs"] = nbytes * reps / ms / 1e6      # per GPU egress (and ingress)
    if W >= 2:
        # one direction per link: even ranks send to their successor, odd ranks only receive
        send = r % 2 == 0 and succ != r
        ms = _timed(env, lambda: dv.dv_flush(ctx, src, nbytes, ep, 0, xfer=dv.DV_XFER_STAGED, stream=sp)
                    if send else None, reps)
        out["uni_ce_gbs"] = nbytes * reps / ms / 1e6
    env.barrier()
    dv.dv_ipc_close(peer)
    env.barrier()
    dv.dv_device_free(src)
    dv.dv_device_free(dst)
    out["peak_gbs"] = max(out["ring_ce_gbs"], out["ring_sm_gbs"], out.get("uni_ce_gbs", 0.0))
    out["how"] = ("dv_flush of one contiguous buffer into the successor's IPC-mapped buffer: ce = "
                  "copy engine (cudaMemcpyAsync), sm = the library's copy kernel storing over the link; "
                  "device time, max over ranks")
    return out


# =====================================================================================================
# C5 ring replication
# =====================================================================================================
class C5:
    def __init__(self, ctx, env):
        self.ctx, self.env = ctx, env
        P = env.world
        self.P = P
        self.Ls = 64 // P if P > 1 else 8
        self.b, self.S, self.p = (2, 256, 64) if _small() else (16, 2048, 1024)
        r = env.rank
        self.lb = r * self.Ls
        self.pred, self.succ = (r - 1) % P, (r + 1) % P
        shape = (self.Ls, self.b, H, self.S, D)
        self.own_k = torch.empty(shape, dtype=torch.int16, device=env.dev)
        self.own_v = torch.empty_like(self.own_k)
        self.own = dv.cache(self.own_k, self.own_v, self.lb, 0)
        dv.dvt_fill(self.own, dv.DVT_FILL_HASH, seed=SEED_C5)
        self.rep_k = torch.full(shape, -1, dtype=torch.int16, device=env.dev)
        self.rep_v = torch.full_like(self.rep_k, -1)
        self.rep = dv.cache(self.rep_k, self.rep_v, self.pred * self.Ls, 0)
        self.flags = torch.zeros(P, dtype=torch.int64, device=env.dev)
        self.ack = torch.zeros(1, dtype=torch.int64, device=env.dev)
        torch.cuda.synchronize()
        blob = {"k": dv.dv_ipc_export(self.rep_k.data_ptr()), "v": dv.dv_ipc_export(self.rep_v.data_ptr()),
                "f": dv.dv_ipc_export(self.flags.data_ptr()), "a": dv.dv_ipc_export(self.ack.data_ptr()),
                "layer_begin": self.pred * self.Ls}
        self.blobs = env.gather(blob)
        sb = self.blobs[self.succ]
        self.kp, self.vp, self.fp = dv.dv_ipc_open(sb["k"]), dv.dv_ipc_open(sb["v"]), dv.dv_ipc_open(sb["f"])
        sdev = self.succ if env.world > 1 and os.environ.get("DV_BENCH_SAME_DEVICE") != "1" else env.local
        self.rep_at_succ = dv.cache_raw(self.kp, self.vp, sdev, 2, sb["layer_begin"], self.Ls, 0, self.b, H,
                                        self.S, D)
        self.sig = dv.endpoint(dv.DV_EP_PEER, self.fp, 8 * P, self.fp, P, device=sdev)
        self.setup = dv.Setup([self.lb, self.lb + self.Ls], [0, self.b], self.S)
        self.dst_arr, self.sig_arr = dv.cache_array([self.rep_at_succ]), dv.endpoint_array([self.sig])
        self.sp = torch.cuda.current_stream().cuda_stream
        self.layer_bytes_tok = 2 * self.b * H * D * 2          # one layer, one position (576 KiB at b 16)
        self.step_bytes = self.Ls * self.layer_bytes_tok
        self.prompt_bytes = self.step_bytes * self.p
        self.seq = 0
        self.t = 0                                               # token steps streamed so far

    def _next_seq(self):
        self.seq += 1
        return self.seq

    def pos(self, t):                                            # reading Q4: step t writes p + t - 1
        return self.p + (t - 1) % (self.S - self.p)

    def prompt_replica(self, xfer=0):
        lb, Ls = self.lb, self.Ls
        dv.dv_stream_out_direct(self.ctx, self.own, (lb, lb + Ls, 0, self.b, 0, self.p), self.setup, 0, 0,
                                self.setup, self.dst_arr, self.sig_arr, seq=self._next_seq(), xfer=xfer,
                                stream=self.sp)

    def token_step(self):
        self.t += 1
        q = self.pos(self.t)
        lb = self.lb
        dv.dv_stream_out_direct(self.ctx, self.own, (lb, lb + self.Ls, 0, self.b, q, q + 1), self.setup, 0, 0,
                                self.setup, self.dst_arr, self.sig_arr, seq=self._next_seq(), stream=self.sp)

    def verify(self, n_pos):
        """Every word of this rank's replica store (the predecessor's layers) on [0, n_pos) against
        the generator (dvt_verify on the device); returns mismatches (max over ranks) and words."""
        cnt = torch.zeros(1, dtype=torch.int64, device=self.env.dev)
        reg = dv.region(self.pred * self.Ls, self.pred * self.Ls + self.Ls, 0, self.b, 0, n_pos)
        dv.dvt_verify(self.rep, cnt.data_ptr(), seed=SEED_C5, reg=reg, stream=self.sp)
        torch.cuda.synchronize()
        bad = int(self.env.max(float(cnt.item())))
        words = 2 * self.Ls * self.b * H * n_pos * D
        return {"mismatches": bad, "words_per_rank": words, "how": "dvt_verify of every replica word vs the generator"}

    def latency(self, n=300, loaded=False, partition=0):
        """Per-layer put latency with the system-scope release: writer (dvt_fill of one layer's new
        position) ends -> the put's seq flag released into the successor's memory (%globaltimer on
        the sender, dvt_trace stamps). loaded: while a bf16 GEMM loop (8192^3) keeps every SM of
        this GPU busy on a low-priority stream, the writer and the put run on a high-priority one
        (NEXT-2: the streaming beside the model's compute)."""
        env = self.env
        te = torch.zeros(n, dtype=torch.int64, device=env.dev)
        ts = torch.zeros((n, 4), dtype=torch.int64, device=env.dev)
        ts[:, 1:3] = 2 ** 63 - 1
        q = self.S - 1
        sp = self.sp
        part = None
        if loaded:
            lo, hi = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)
            if partition:   # SM partition (dv_partition_create): put on `partition` SMs, GEMM on the rest
                part = dv.dv_partition_create(env.local, partition, torch.cuda.Stream.priority_range()[1])
                hi, lo = torch.cuda.ExternalStream(part.streaming), torch.cuda.ExternalStream(part.compute)
            ga = torch.randn(8192, 8192, device=env.dev, dtype=torch.bfloat16)
            gb = torch.randn(8192, 8192, device=env.dev, dtype=torch.bfloat16)
            with torch.cuda.stream(lo):
                torch.matmul(ga, gb)
            torch.cuda.synchronize()
            sp = hi.cuda_stream
        env.barrier()
        if loaded:
            with torch.cuda.stream(lo):
                for _ in range(60):          # ~40 ms of GEMMs: longer than the spin + n puts
                    torch.matmul(ga, gb)
        dv.dvt_spin(20_000_000, 1, stream=sp)
        for i in range(n):
            layer = self.lb + i % self.Ls
            reg = dv.region(layer, layer + 1, 0, self.b, q, q + 1)
            dv.dvt_fill(self.own, dv.DVT_FILL_HASH, seed=SEED_C5, reg=reg, stream=sp, t_end_ptr=te[i].data_ptr())
            dv.dvt_trace(self.ctx, ts[i].data_ptr())
            dv.dv_stream_out_direct(self.ctx, self.own, reg, self.setup, 0, 0, self.setup, self.dst_arr,
                                    self.sig_arr, seq=self._next_seq(), stream=sp)
        dv.dvt_trace(self.ctx, 0)
        torch.cuda.synchronize()
        if part is not None:
            part.destroy()
        us = ((ts[:, 0] - te).double() / 1e3).tolist()[20:]
        p50, p99 = env.max(_pct(us, 0.5)), env.max(_pct(us, 0.99))
        scope = dv.dvt_release_scope(self.ctx, self.fp, self.kp)
        return {"p50_us": p50, "p99_us": p99, "n": len(us), "bytes": self.layer_bytes_tok, "loaded": loaded,
                "sm_partition": partition or None,
                "release_scope": "gpu" if scope else "system",
                "how": "writer end -> st.release of the seq flag in the successor's memory, sender "
                       "%globaltimer; p50/p99 max over ranks"}

    def latency_fused(self, n=300):
        """Per-layer put with the put FUSED INTO THE PRODUCER (dv_dplan_remap into the successor's
        IPC-mapped replica, include/dv.h device plans): the vectorised producer (dvt_fill_rows)
        writes one layer's new K/V into its own cache and the successor's replica and releases the
        successor's flag. Reported beside the separate path (producer, then dv_stream_out_direct):
        producer start -> flag release, p50/p99 max over ranks."""
        env = self.env
        q = self.S - 1
        plans = [dv.dv_dplan_remap(self.ctx, self.own, self.rep_at_succ,
                                   dv.region(self.lb + j, self.lb + j + 1, 0, self.b, q, q + 1), self.sig,
                                   flag_slot=0, seq=self.seq + 1) for j in range(self.Ls)]
        out = {}
        for arm in ("fused", "separate"):
            t0 = torch.full((n,), 2 ** 63 - 1, dtype=torch.int64, device=env.dev)
            te = torch.zeros(n, dtype=torch.int64, device=env.dev)
            ts = torch.zeros((n, 4), dtype=torch.int64, device=env.dev)
            ts[:, 1:3] = 2 ** 63 - 1
            env.barrier()
            dv.dvt_spin(20_000_000, 1, stream=self.sp)
            for i in range(n):
                j = i % self.Ls
                reg = dv.region(self.lb + j, self.lb + j + 1, 0, self.b, q, q + 1)
                if arm == "fused":
                    plans[j].trace = ts[i].data_ptr()
                    plans[j].seq = self._next_seq()
                    dv.dvt_fill_rows(self.own, SEED_C5, reg, plans[j], 0, t_start_ptr=t0[i].data_ptr(),
                                     t_end_ptr=te[i].data_ptr(), stream=self.sp)
                else:
                    dv.dvt_fill_rows(self.own, SEED_C5, reg, None, 0, t_start_ptr=t0[i].data_ptr(),
                                     t_end_ptr=te[i].data_ptr(), stream=self.sp)
                    dv.dvt_trace(self.ctx, ts[i].data_ptr())
                    dv.dv_stream_out_direct(self.ctx, self.own, reg, self.setup, 0, 0, self.setup, self.dst_arr,
                                            self.sig_arr, seq=self._next_seq(), stream=self.sp)
            dv.dvt_trace(self.ctx, 0)
            torch.cuda.synchronize()
            us = ((ts[:, 0] - t0).double() / 1e3).tolist()[20:]
            out[arm] = {"start_to_flag_p50_us": env.max(_pct(us, 0.5)), "start_to_flag_p99_us": env.max(_pct(us, 0.99)),
                        "n": len(us)}
            # every word the predecessor's producer stored into this rank's replica at position q
            env.barrier()
            cnt = torch.zeros(1, dtype=torch.int64, device=env.dev)
            dv.dvt_verify(self.rep, cnt.data_ptr(), seed=SEED_C5,
                          reg=dv.region(self.pred * self.Ls, self.pred * self.Ls + self.Ls, 0, self.b, q, q + 1),
                          stream=self.sp)
            torch.cuda.synchronize()
            out[arm]["replica_mismatches"] = int(env.max(float(cnt.item())))
        out["bytes"] = self.layer_bytes_tok
        out["release_scope"] = "system" if plans[0].sys_scope else "gpu"
        for pl in plans:
            dv.dv_dplan_free(self.ctx, pl)
        return out

    def pingpong(self, iters=300):
        """Put one layer (+ flag) into the successor, wait for the predecessor's put, ack into the
        predecessor's memory, wait for the successor's ack: RTT per iteration (device time)."""
        env = self.env
        pa = dv.dv_ipc_open(self.blobs[self.pred]["a"])
        pdev = self.pred if env.world > 1 and os.environ.get("DV_BENCH_SAME_DEVICE") != "1" else env.local
        pred_ack = dv.endpoint(dv.DV_EP_PEER, pa, 8, pa, 1, device=pdev)
        own_ack = dv.endpoint(dv.DV_EP_DEVICE, self.ack.data_ptr(), 8, self.ack.data_ptr(), 1, device=env.local)
        inbox = dv.endpoint(dv.DV_EP_DEVICE, self.flags.data_ptr(), 8 * self.P, self.flags.data_ptr(), self.P,
                            device=env.local)
        q = self.S - 1
        env.barrier()
        base = self.seq + 10        # every rank's flags/acks move in lockstep from here
        base = int(env.max(base))

        def one(i):
            layer = self.lb + i % self.Ls
            dv.dv_stream_out_direct(self.ctx, self.own, dv.region(layer, layer + 1, 0, self.b, q, q + 1), self.setup,
                                    0, 0, self.setup, self.dst_arr, self.sig_arr, seq=base + i, stream=self.sp)
            dv.dv_wait(self.ctx, inbox, 0, base + i, stream=self.sp)   # slot 0: the predecessor's 1-block setup
            dv.dv_signal(self.ctx, pred_ack, 0, base + i, stream=self.sp)
            dv.dv_wait(self.ctx, own_ack, 0, base + i, stream=self.sp)
        for i in range(20):
            one(i)
        env.barrier()
        st = torch.cuda.current_stream()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dv.dvt_spin(max(4_000_000, iters * 12_000), 1, stream=self.sp)
        a.record(st)
        for i in range(20, 20 + iters):
            one(i)
        e.record(st)
        torch.cuda.synchronize()
        rtt = env.max(a.elapsed_time(e) * 1e3 / iters)
        self.seq = base + 20 + iters
        env.barrier()
        dv.dv_ipc_close(pa)
        return {"rtt_us": rtt, "one_way_us": rtt / 2, "bytes": self.layer_bytes_tok, "iters": iters,
                "how": "put+flag -> stream wait on the predecessor's flag -> ack into its memory -> wait own ack"}

    def nccl_baseline(self, steps):
        """NCCL send/recv baseline (north_star: "NCCL send/recv kept only as the baseline"): the
        same prompt replica (per layer: pack -> send to the successor / recv from the predecessor ->
        unpack) and the same token steps (pack the step -> send/recv -> unpack). The replica store
        is reset first, so the verify after it checks what NCCL delivered."""
        env = self.env
        self.rep_k.fill_(-1)
        self.rep_v.fill_(-1)
        lb, Ls, b, p = self.lb, self.Ls, self.b, self.p
        plb = self.pred * Ls
        lay_b = 2 * b * H * p * D * 2
        sbuf = torch.empty(lay_b // 2, dtype=torch.int16, device=env.dev)
        rbuf = torch.empty_like(sbuf)
        sep, rep_ = dv.endpoint_of(sbuf), dv.endpoint_of(rbuf)

        def prompt():
            for l in range(Ls):
                dv.dv_scatter(self.ctx, self.own, (lb + l, lb + l + 1, 0, b, 0, p), sep, 0, stream=self.sp)
                _sendrecv(env.backend, sbuf, self.succ, rbuf, self.pred)
                dv.dv_gather(self.ctx, rep_, 0, self.rep, (plb + l, plb + l + 1, 0, b, 0, p), stream=self.sp)
        ms_prompt = _timed(env, prompt)
        tb = torch.empty(self.step_bytes // 2, dtype=torch.int16, device=env.dev)
        trb = torch.empty_like(tb)
        tep, trep = dv.endpoint_of(tb), dv.endpoint_of(trb)
        t0 = [0]

        def token():
            t0[0] += 1
            q = self.pos(t0[0])
            dv.dv_scatter(self.ctx, self.own, (lb, lb + Ls, 0, b, q, q + 1), tep, 0, stream=self.sp)
            _sendrecv(env.backend, tb, self.succ, trb, self.pred)
            dv.dv_gather(self.ctx, trep, 0, self.rep, (plb, plb + Ls, 0, b, q, q + 1), stream=self.sp)
        for _ in range(3):
            token()
        t0[0] = 0
        ms_tok = _timed(env, token, steps)
        out = {"prompt_replica": {"ms": ms_prompt, "gbs_per_gpu": self.prompt_bytes / ms_prompt / 1e6},
               "token_step": {"us": ms_tok * 1e3 / steps, "gbs_per_gpu": self.step_bytes * steps / ms_tok / 1e6},
               "parity": self.verify(self.p + min(steps, self.S - self.p)),
               "impl": "nccl send/recv" if env.backend == "nccl" else "gloo send/recv, host-staged (tests only)"}
        return out

    def close(self):
        for x in (self.kp, self.vp, self.fp):
            dv.dv_ipc_close(x)


def c5_suite(ctx, env, steps=200, peak=None, peak_src=None, nccl=True):
    c = C5(ctx, env)
    out = {"workload": f"C5 OPT-66B ring replication b{c.b}, {c.P} stage(s) x {c.Ls} layers, p {c.p}, S {c.S}",
           "bytes_prompt_replica_per_gpu": c.prompt_bytes, "bytes_token_step_per_gpu": c.step_bytes}
    c.prompt_replica()   # warm-up: first touch of the (IPC-mapped) replica pages, kernel loads
    torch.cuda.synchronize()
    ms = _timed(env, c.prompt_replica)
    g = c.prompt_bytes / ms / 1e6
    out["prompt_replica"] = {"ms": ms, "gbs_per_gpu": g, "gbs_aggregate": g * c.P,
                             "roofline": _roof(g, peak, peak_src, env), "timed_after_one_warm_up_call": True}
    try:   # the same bulk replica by the copy engine (2-D DMAs of p*D*e-byte runs)
        ms2 = _timed(env, lambda: c.prompt_replica(dv.DV_XFER_STAGED))
        g2 = c.prompt_bytes / ms2 / 1e6
        out["prompt_replica_copy_engine"] = {"ms": ms2, "gbs_per_gpu": g2, "roofline": _roof(g2, peak, peak_src, env)}
    except Exception as e:   # noqa: BLE001
        out["prompt_replica_copy_engine"] = {"error": f"{type(e).__name__}: {e}"}
        env.barrier()
    steps = min(steps, c.S - c.p)
    for _ in range(3):
        c.token_step()
    c.t = 0                                    # timed steps rewrite positions p .. p+steps-1
    ms = _timed(env, c.token_step, steps, head_start_ns=max(2_000_000, steps * 40_000))
    g = c.step_bytes * steps / ms / 1e6
    out["token_step"] = {"us": ms * 1e3 / steps, "gbs_per_gpu": g, "gbs_aggregate": g * c.P, "steps": steps,
                         "roofline": _roof(g, peak, peak_src, env),
                         "how": "one dv_stream_out_direct per step (all the stage's layers, one position) "
                                "into the successor's replica store + seq flag; spin head start hides the enqueue"}
    out["parity"] = c.verify(c.p + steps)
    for name, fn in (("latency_per_layer_put", c.latency),
                     ("latency_per_layer_put_under_gemm", lambda: c.latency(loaded=True)),
                     ("latency_per_layer_put_under_gemm_sm_partition_16", lambda: c.latency(loaded=True, partition=16)),
                     ("latency_per_layer_put_fused_producer", c.latency_fused),
                     ("pingpong", c.pingpong)):
        try:
            out[name] = fn()
        except Exception as e:   # noqa: BLE001 -- reported; the other C5 numbers still print
            out[name] = {"error": f"{type(e).__name__}: {e}"}
            env.barrier()
    if nccl and env.world > 1:
        out["nccl_baseline"] = c.nccl_baseline(steps)
        nb = out["nccl_baseline"]
        out["dvstream_vs_nccl"] = {
            "prompt_replica": out["prompt_replica"]["gbs_per_gpu"] / nb["prompt_replica"]["gbs_per_gpu"],
            "token_step": out["token_step"]["gbs_per_gpu"] / nb["token_step"]["gbs_per_gpu"]}
    c.close()
    env.barrier()
    del c
    torch.cuda.empty_cache()
    return out


# =====================================================================================================
# C3 prompt -> token disaggregation
# =====================================================================================================
def _token_bounds(n):
    return {1: [0, 64], 2: [0, 29, 64], 4: [0, 13, 30, 47, 64]}.get(n) or \
        [round(64 * k / n) for k in range(n + 1)]


class C3:
    def __init__(self, ctx, env):
        self.ctx, self.env = ctx, env
        W, r = env.world, env.rank
        self.b, self.Sp, self.St = (2, 64, 128) if _small() else (8, 1024, 2048)
        self.p = int(os.environ.get("DV_C3_PROMPT", "32" if _small() else "1000"))
        self.n_p = max(1, W // 2)
        self.n_t = max(1, W - self.n_p) if W > 1 else 1
        self.pb = [round(64 * k / self.n_p) for k in range(self.n_p + 1)]
        self.tb = _token_bounds(self.n_t)
        self.ps, self.ts = dv.Setup(self.pb, [0, self.b], self.Sp), dv.Setup(self.tb, [0, self.b], self.St)
        self.is_prompt = W == 1 or r < self.n_p
        self.is_token = W == 1 or r >= self.n_p
        self.sp = torch.cuda.current_stream().cuda_stream
        blob = None
        if self.is_token:
            self.j = 0 if W == 1 else r - self.n_p
            j = self.j
            self.tk = torch.full((self.tb[j + 1] - self.tb[j], self.b, H, self.St, D), -1, dtype=torch.int16,
                                 device=env.dev)
            self.tv = torch.full_like(self.tk, -1)
            self.tc = dv.cache(self.tk, self.tv, self.tb[j], 0)
            self.tf = torch.zeros(self.n_p, dtype=torch.int64, device=env.dev)
            torch.cuda.synchronize()
            blob = {"k": dv.dv_ipc_export(self.tk.data_ptr()), "v": dv.dv_ipc_export(self.tv.data_ptr()),
                    "f": dv.dv_ipc_export(self.tf.data_ptr()), "j": j, "rank": r, "device": env.local}
        blobs = [x for x in env.gather(blob) if x is not None]
        blobs.sort(key=lambda x: x["j"])
        self.token_ranks = [x["rank"] for x in blobs]
        self.opened = []
        if self.is_prompt:
            self.i = 0 if W == 1 else r
            i = self.i
            self.pk = torch.empty((self.pb[i + 1] - self.pb[i], self.b, H, self.Sp, D), dtype=torch.int16,
                                  device=env.dev)
            self.pv = torch.empty_like(self.pk)
            self.pc = dv.cache(self.pk, self.pv, self.pb[i], 0)
            dv.dvt_fill(self.pc, dv.DVT_FILL_HASH, seed=SEED_C3, valid=(0, self.p))
            caches, sigs, ft6d = [], [], []
            for bl in blobs:
                kp, vp, fp = dv.dv_ipc_open(bl["k"]), dv.dv_ipc_open(bl["v"]), dv.dv_ipc_open(bl["f"])
                self.opened += [kp, vp, fp]
                jj = bl["j"]
                caches.append(dv.cache_raw(kp, vp, bl["device"], 2, self.tb[jj], self.tb[jj + 1] - self.tb[jj], 0,
                                           self.b, H, self.St, D))
                # the same memory seen as FasterTransformer caches (6-D key, NEXT-1): the FT6D probe
                ft6d.append(dv.cache_raw(kp, vp, bl["device"], 2, self.tb[jj], self.tb[jj + 1] - self.tb[jj], 0,
                                         self.b, H, self.St, D, layout=dv.DV_LAYOUT_FT6D))
                sigs.append(dv.endpoint(dv.DV_EP_PEER, fp, 8 * self.n_p, fp, self.n_p, device=bl["device"]))
            self.caches, self.sigs = dv.cache_array(caches), dv.endpoint_array(sigs)
            self.caches_ft6d = dv.cache_array(ft6d)
            self.n_dst = len(caches)
        self.layer_bytes = 2 * self.b * H * self.p * D * 2
        self.seq = 0

    def my_prompt_bytes(self):
        return (self.pb[self.i + 1] - self.pb[self.i]) * self.layer_bytes if self.is_prompt else 0

    def handoff(self, ft6d=False, xfer=0):
        self.seq += 1
        if not self.is_prompt:
            return
        i = self.i
        dst = self.caches_ft6d if ft6d else self.caches
        for layer in range(self.pb[i], self.pb[i + 1]):       # layer by layer (Opt 2)
            dv.dv_stream_out_direct(self.ctx, self.pc, dv.region(layer, layer + 1, 0, self.b, 0, self.p), self.ps, i,
                                    0, self.ts, dst, self.sigs, seq=self.seq, xfer=xfer, stream=self.sp)

    def producer_forms(self, steps=2):
        """The hand-off with the PRODUCER in the loop (the prompt pass writing each layer's K/V --
        here the test library's vectorised writer dvt_fill_rows): 'separate' = producer, then
        dv_stream_out_direct per layer; 'fused' = the producer stores every row into its own cache
        AND, through a plan set per layer (dv_dplan_stream_out_direct: one plan per route piece),
        into the token GPUs' caches, releasing their flags itself (include/dv.h device plans).
        Token caches reset before and verified word by word after each form."""
        env = self.env
        out = {}
        sets = {}
        box = (64, self.b, H, self.St, D)   # UID words (a memory-bound producer), the same box on both sides
        if self.is_prompt:
            i = self.i
            for layer in range(self.pb[i], self.pb[i + 1]):
                sets[layer] = dv.dv_dplan_stream_out_direct(
                    self.ctx, self.pc, dv.region(layer, layer + 1, 0, self.b, 0, self.p), self.ps, i, 0, self.ts,
                    self.caches, self.sigs, seq=1)

        def run(fused):
            self.seq += 1
            if not self.is_prompt:
                return
            for layer in range(self.pb[self.i], self.pb[self.i + 1]):
                reg = dv.region(layer, layer + 1, 0, self.b, 0, self.p)
                if fused:
                    st = sets[layer]
                    for q in range(st.n):
                        st.plan[q].seq = self.seq
                    dv.dvt_fill_rows(self.pc, 0, reg, st, 0, stream=self.sp, kind=dv.DVT_FILL_UID, box=box)
                else:
                    dv.dvt_fill_rows(self.pc, 0, reg, None, 0, stream=self.sp, kind=dv.DVT_FILL_UID, box=box)
                    dv.dv_stream_out_direct(self.ctx, self.pc, reg, self.ps, self.i, 0, self.ts, self.caches, self.sigs,
                                            seq=self.seq, stream=self.sp)
        for name, fused in (("separate", False), ("fused", True)):
            if self.is_token:
                self.tk.fill_(-1)
                self.tv.fill_(-1)
            env.barrier()
            run(fused)                                    # warm-up
            ms = _timed(env, lambda fused=fused: run(fused), steps)
            out[name] = {"ms_per_handoff_with_producer": ms / steps,
                         "gbs_per_prompt_gpu": env.max(self.my_prompt_bytes()) * steps / ms / 1e6,
                         "parity": self.verify(kind=dv.DVT_FILL_UID, box=box)}
        torch.cuda.synchronize()
        for st in sets.values():
            dv.dv_dplan_free(self.ctx, st)
        if self.is_prompt:   # the other C3 forms expect the HASH-filled prompt cache back
            dv.dvt_fill(self.pc, dv.DVT_FILL_HASH, seed=SEED_C3, valid=(0, self.p))
            torch.cuda.synchronize()
        out["how"] = ("prompt layer by layer: producer + dv_stream_out_direct vs the producer fused with the "
                      "hand-off through plan sets; device time per hand-off, max over ranks; the producer writes "
                      "uid words (a few integer ops per word: memory-bound, like a KV projection's epilogue)")
        return out

    def ft6d_forms(self, steps=2):
        """NEXT-1 over the link: the hand-off into FasterTransformer token caches (6-D key: every
        key packet transposed on the way), with the shared-memory tile transpose (the automatic
        choice for memory reached over a link, DV_TRS=0) and with the register transpose forced
        (DV_TRS=4) -- which is faster over NVLink settles DESIGN §6's reading. Each form's token
        caches are reset and verified word by word."""
        env = self.env
        out = {}
        for name, trs in (("tile_form_auto", 0), ("register_form", 4)):
            if self.is_token:
                self.tk.fill_(-1)
                self.tv.fill_(-1)
            dv.dvt_tune("DV_TRS", trs)
            try:
                self.handoff(True)                         # warm-up
                ms = _timed(env, lambda: self.handoff(True), steps)
            finally:
                dv.dvt_tune("DV_TRS", 0)
            per_gpu = env.max(self.my_prompt_bytes()) * steps / ms / 1e6
            bad = 0
            if self.is_token:
                j = self.j
                c6 = dv.cache_raw(self.tk.data_ptr(), self.tv.data_ptr(), env.local, 2, self.tb[j],
                                  self.tb[j + 1] - self.tb[j], 0, self.b, H, self.St, D, layout=dv.DV_LAYOUT_FT6D)
                cnt = torch.zeros(1, dtype=torch.int64, device=env.dev)
                dv.dvt_verify(c6, cnt.data_ptr(), seed=SEED_C3, valid=(0, self.p),
                              reg=dv.region(self.tb[j], self.tb[j + 1], 0, self.b, 0, self.p), stream=self.sp)
                torch.cuda.synchronize()
                bad = int(cnt.item())
            out[name] = {"ms_per_handoff": ms / steps, "gbs_per_prompt_gpu": per_gpu,
                         "mismatches": int(env.max(float(bad)))}
        return out

    def verify(self, kind=None, box=None):
        env = self.env
        bad = 0
        sentinel_ok = True
        if self.is_token:
            j = self.j
            cnt = torch.zeros(1, dtype=torch.int64, device=env.dev)
            kw = {} if kind is None else {"kind": kind, "box": box}
            dv.dvt_verify(self.tc, cnt.data_ptr(), seed=SEED_C3 if kind is None else 0, valid=(0, self.p),
                          reg=dv.region(self.tb[j], self.tb[j + 1], 0, self.b, 0, self.p), stream=self.sp, **kw)
            torch.cuda.synchronize()
            bad = int(cnt.item())
            sentinel_ok = bool((self.tk[:, :, :, self.p:] == -1).all()) and bool((self.tv[:, :, :, self.p:] == -1).all())
        bad = int(env.max(float(bad)))
        sentinel_ok = env.max(0.0 if sentinel_ok else 1.0) == 0.0
        return {"mismatches": bad, "positions_past_prompt_untouched": sentinel_ok,
                "words": 2 * 64 * self.b * H * self.p * D,
                "how": "dvt_verify of every token-cache word on [0, p) vs the generator; [p, S) still the sentinel"}

    def nccl_baseline(self, steps):
        env = self.env
        if self.is_token:
            self.tk.fill_(-1)
            self.tv.fill_(-1)
        xbuf = torch.empty(self.layer_bytes // 2, dtype=torch.int16, device=env.dev)
        xep = dv.endpoint_of(xbuf)

        def owner(bounds, layer):
            return max(x for x in range(len(bounds) - 1) if bounds[x] <= layer)

        def run():
            if self.is_prompt and self.is_token:       # N = 1: no exchange, pack + unpack
                return
            if self.is_prompt:
                i = self.i
                for layer in range(self.pb[i], self.pb[i + 1]):
                    dv.dv_scatter(self.ctx, self.pc, dv.region(layer, layer + 1, 0, self.b, 0, self.p), xep, 0,
                                  stream=self.sp)
                    _sendrecv(env.backend, xbuf, self.token_ranks[owner(self.tb, layer)], None, None)
            else:
                j = self.j
                for layer in range(self.tb[j], self.tb[j + 1]):
                    _sendrecv(env.backend, None, None, xbuf, owner(self.pb, layer))
                    dv.dv_gather(self.ctx, xep, 0, self.tc, dv.region(layer, layer + 1, 0, self.b, 0, self.p),
                                 stream=self.sp)
        ms = _timed(env, run, steps)
        total = 64 * self.layer_bytes
        per_gpu = env.max(self.my_prompt_bytes()) * steps / ms / 1e6
        return {"ms_per_handoff": ms / steps, "gbs_aggregate": total * steps / ms / 1e6, "gbs_per_prompt_gpu": per_gpu,
                "parity": self.verify(),
                "impl": "nccl send/recv" if env.backend == "nccl" else "gloo send/recv, host-staged (tests only)"}

    def close(self):
        for x in self.opened:
            dv.dv_ipc_close(x)


def c3_suite(ctx, env, steps=3, peak=None, peak_src=None, nccl=True):
    c = C3(ctx, env)
    total = 64 * c.layer_bytes
    out = {"workload": f"C3 OPT-66B b{c.b} p{c.p}: {c.n_p} prompt GPU(s) {c.pb} -> {c.n_t} token GPU(s) {c.tb}, "
                       f"S {c.Sp} -> {c.St}, layer by layer, straight into the token caches",
           "bytes_per_handoff": total}
    c.handoff()                                 # warm-up
    env.barrier()
    ms = _timed(env, c.handoff, steps)
    per_gpu = env.max(c.my_prompt_bytes()) * steps / ms / 1e6
    out["handoff"] = {"ms": ms / steps, "gbs_aggregate": total * steps / ms / 1e6, "gbs_per_prompt_gpu": per_gpu,
                      "steps": steps, "roofline": _roof(per_gpu, peak, peak_src, env),
                      "ideal_ms_at_peak": (env.max(c.my_prompt_bytes()) / peak / 1e6) if peak else None}
    out["parity"] = c.verify()
    try:
        out["producer_fused_vs_separate"] = c.producer_forms()
    except Exception as e:   # noqa: BLE001 -- reported; the other C3 numbers still print
        out["producer_fused_vs_separate"] = {"error": f"{type(e).__name__}: {e}"}
        env.barrier()
    try:
        # the same hand-off by the copy engine (DV_XFER_STAGED: one 2-D DMA per (K or V, layer,
        # request) over the heads, runs of p*D*e bytes) -- SM stores vs copy engine over the link
        if c.is_token:
            c.tk.fill_(-1)
            c.tv.fill_(-1)
        c.handoff(xfer=dv.DV_XFER_STAGED)
        env.barrier()
        ms2 = _timed(env, lambda: c.handoff(xfer=dv.DV_XFER_STAGED), steps)
        pg2 = env.max(c.my_prompt_bytes()) * steps / ms2 / 1e6
        out["handoff_copy_engine"] = {"ms": ms2 / steps, "gbs_per_prompt_gpu": pg2,
                                      "roofline": _roof(pg2, peak, peak_src, env), "parity": c.verify()}
    except Exception as e:   # noqa: BLE001
        out["handoff_copy_engine"] = {"error": f"{type(e).__name__}: {e}"}
        env.barrier()
    try:
        out["ft6d_token_caches"] = c.ft6d_forms()
    except Exception as e:   # noqa: BLE001
        out["ft6d_token_caches"] = {"error": f"{type(e).__name__}: {e}"}
        env.barrier()
    if nccl and env.world > 1:
        out["nccl_baseline"] = c.nccl_baseline(steps)
        out["dvstream_vs_nccl"] = out["handoff"]["gbs_per_prompt_gpu"] / out["nccl_baseline"]["gbs_per_prompt_gpu"]
    c.close()
    env.barrier()
    del c
    torch.cuda.empty_cache()
    return out


# =====================================================================================================
# C4 concurrent swapping: the shared host PCIe fabric (BASELINE.json configs[3])
# =====================================================================================================
def c4_concurrent(ctx, env, steps=4):
    """Every rank is one BLOOM-176B pipeline stage (9 layers, b 4, S 2048) swapping microbatches
    with its own NUMA-local pinned host log (dv_host_alloc_near): per step, the step delta of the
    running microbatch out (2.06 MB, decoupled) and the whole i = 1024 prefix of the next one in
    (2.11 GB, copy engine; PAPER.md:572 transf_i = i*B*C). Rank 0 alone first, then all ranks at
    once: per-GPU and aggregate PCIe GB/s. Every swapped-in word verified on the device."""
    Hc, nL, b, S, i_pref = 112, 9, 4, 2048, (128 if _small() else 1024)
    seed = 20240307
    step_b = 2 * nL * b * Hc * D * 2
    nb_in = i_pref * step_b
    run_k = torch.empty((nL, b, Hc, S, D), dtype=torch.int16, device=env.dev)
    run_v = torch.empty_like(run_k)
    run = dv.cache(run_k, run_v)
    dv.dvt_fill(run, dv.DVT_FILL_HASH, seed=seed)
    free_k = torch.full_like(run_k, -1)
    free_v = torch.full_like(run_v, -1)
    free = dv.cache(free_k, free_v)
    hp, node = dv.dv_host_alloc_near(env.local, nb_in + 64 * step_b)
    try:
        log = dv.endpoint(dv.DV_EP_HOST, hp, nb_in)
        out_fl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
        out = dv.endpoint(dv.DV_EP_HOST, hp + nb_in, 64 * step_b, out_fl.data_ptr(), 1)
        sp = torch.cuda.current_stream().cuda_stream
        dv.dv_scatter(ctx, run, (0, nL, 0, b, 0, i_pref), log, 0, stream=sp)   # the microbatch's swap-out
        seq = [0]

        def step():
            seq[0] += 1
            q = i_pref + seq[0] % (S - i_pref)
            dv.dv_scatter(ctx, run, (0, nL, 0, b, q, q + 1), out, (seq[0] % 64) * step_b, flag_slot=0, seq=seq[0],
                          xfer=dv.DV_XFER_DECOUPLED, stream=sp)
            dv.dv_gather(ctx, log, 0, free, (0, nL, 0, b, 0, i_pref), stream=sp)

        def timed(active):
            def body():
                if active:
                    for _ in range(steps):
                        step()
                    dv.dv_wait(ctx, out, 0, seq[0], stream=sp)
            return _timed(env, body)
        step()
        env.barrier()
        moved = steps * (nb_in + step_b)
        ms_alone = timed(env.rank == 0)
        ms_all = timed(True)
        cnt = torch.zeros(1, dtype=torch.int64, device=env.dev)
        dv.dvt_verify(free, cnt.data_ptr(), seed=seed, reg=dv.region(0, nL, 0, b, 0, i_pref), stream=sp)
        torch.cuda.synchronize()
        bad = int(env.max(float(cnt.item())))
        per_all = moved / ms_all / 1e6
        return {"workload": f"C4 BLOOM-176B stage (9 layers, b4, S2048) per rank: swap-out of a step delta "
                            f"({step_b} B, decoupled) + swap-in of the i = {i_pref} prefix ({nb_in} B) per step",
                "steps": steps, "numa_node": node,
                "alone_gbs_rank0": moved / ms_alone / 1e6,
                "concurrent_gbs_per_gpu": per_all, "concurrent_gbs_aggregate": per_all * env.world,
                "concurrent_vs_alone": (moved / ms_all) / (moved / ms_alone),
                "parity": {"mismatches": bad, "how": "dvt_verify of every swapped-in word vs the generator"},
                "how": "per-GPU = bytes moved / device time (max over ranks); aggregate = per-GPU x N"}
    finally:
        torch.cuda.synchronize()
        dv.dv_host_free(hp)
        del run_k, run_v, free_k, free_v
        torch.cuda.empty_cache()


def nvlink_suite(ctx, env, steps=200, nccl=True):
    """Everything above in one pass; returns the dict for rank 0's JSON line (None on other ranks)."""
    t0 = time.perf_counter()
    res = {"devices": env.gather(env.identity()), "transport": "CUDA IPC peer stores (one process per GPU)"}
    if os.environ.get("DV_BENCH_SAME_DEVICE") == "1":
        res["transport"] = "CUDA IPC between processes on ONE GPU (test mode: HBM, not NVLink)"
    devs = {d["uuid"] or d["pci"] for d in res["devices"]}
    res["distinct_gpus"] = len(devs)
    for name, fn in (("link", lambda: link_probe(ctx, env)),):
        try:
            res[name] = fn()
        except Exception as e:   # noqa: BLE001 -- a failed part is reported, the line still prints
            res[name] = {"error": f"{type(e).__name__}: {e}"}
    peak = res["link"].get("peak_gbs")
    src = "in-run peer copy (link probe: max of copy-engine / SM-store ring and one-direction copies)"
    for name, fn in (("c5", lambda: c5_suite(ctx, env, steps, peak, src, nccl)),
                     ("c3", lambda: c3_suite(ctx, env, 3, peak, src, nccl)),
                     ("c4_pcie_concurrent", lambda: c4_concurrent(ctx, env))):
        try:
            res[name] = fn()
        except Exception as e:   # noqa: BLE001
            res[name] = {"error": f"{type(e).__name__}: {e}"}
            try:
                env.barrier()
            except Exception:   # noqa: BLE001
                pass
    res["wall_s"] = time.perf_counter() - t0
    return res if env.rank == 0 else None


# =====================================================================================================
# stand-alone workloads (bench.py --workload c3 | c5): one JSON line each
# =====================================================================================================
def _line(args, env, metric, value, ms_per_step, cfg, extra):
    return {"metric": metric, "value": value, "unit": "GB/s", "n_gpus": env.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": cfg.pop("scaling", "weak"), "vs_baseline": None, "dtype": "u16 (opaque fp16 words)",
            "data": "synthetic (splitmix64 coordinate-hash fill)", "config": cfg, **extra}


def run_c5(args, bench):
    env = Env(args.dist_backend)
    env.init()
    ctx = dv.dv_create(env.local)
    nccl = getattr(args, "peer_baseline", "none") == "nccl"
    link = link_probe(ctx, env) if env.world > 1 else None
    peak = link["peak_gbs"] if link else None
    if nccl:
        assert env.world > 1, "--peer-baseline nccl needs >= 2 ranks"
        c = C5(ctx, env)
        c.prompt_replica()
        nb = c.nccl_baseline(args.steps)
        c.close()
        value, msps, extra = nb["token_step"]["gbs_per_gpu"] * env.world, nb["token_step"]["us"] / 1e3, \
            {"impl": "nccl-baseline" if env.backend == "nccl" else "sendrecv-baseline (gloo, host-staged; tests only)",
             "parity_spot_check": {"mismatches": nb["parity"]["mismatches"]}, "baseline": nb}
    else:
        r = c5_suite(ctx, env, args.steps, peak, "in-run link probe", nccl=False)
        ts = r["token_step"]
        value, msps = ts["gbs_aggregate"], ts["us"] / 1e3
        extra = {"impl": "dvstream", "parity_spot_check": {"mismatches": r["parity"]["mismatches"]}, "c5": r,
                 "link": link, "gpu_launches": None}
    if env.rank == 0:
        print(json.dumps(_line(args, env, "KV stream GB/s (ring replication, token step per stage)", value, msps,
                               {"workload": f"C5 OPT-66B ring replication, {env.world} stage(s)",
                                "parallelism": f"pp{env.world} ring"}, extra)), flush=True)
    env.barrier()
    ctx.close()
    if env.world > 1:
        dist.destroy_process_group()


def run_c3(args, bench):
    env = Env(args.dist_backend)
    env.init()
    ctx = dv.dv_create(env.local)
    nccl = getattr(args, "peer_baseline", "none") == "nccl"
    link = link_probe(ctx, env) if env.world > 1 else None
    peak = link["peak_gbs"] if link else None
    if nccl:
        assert env.world > 1, "--peer-baseline nccl needs >= 2 ranks"
        c = C3(ctx, env)
        nb = c.nccl_baseline(args.steps)
        c.close()
        value, msps = nb["gbs_aggregate"], nb["ms_per_handoff"]
        extra = {"impl": "nccl-baseline" if env.backend == "nccl" else "sendrecv-baseline (gloo, host-staged; tests only)",
                 "parity_spot_check": {"mismatches": nb["parity"]["mismatches"]}, "baseline": nb}
    else:
        r = c3_suite(ctx, env, args.steps, peak, "in-run link probe", nccl=False)
        value, msps = r["handoff"]["gbs_aggregate"], r["handoff"]["ms"]
        extra = {"impl": "dvstream", "parity_spot_check": {"mismatches": r["parity"]["mismatches"]}, "c3": r,
                 "link": link}
    if env.rank == 0:
        print(json.dumps(_line(args, env, "KV stream GB/s (prompt-token disaggregation hand-off)", value, msps,
                               {"workload": "C3 OPT-66B disaggregation hand-off", "scaling": "strong",
                                "parallelism": f"pp{max(1, env.world // 2)} -> pp{max(1, env.world - env.world // 2)}"},
                               extra)), flush=True)
    env.barrier()
    ctx.close()
    if env.world > 1:
        dist.destroy_process_group()
