#!/usr/bin/env python
"""bench.py -- KV-cache streaming throughput on B200 (DejaVuLib hot path, arXiv 2403.01876).

Workload (BASELINE.json configs[1], "C2"): OPT-13B shape (40 layers, 40 heads, head_dim 128, fp16
words), batch 8, prompt 1000, max_seq 2048; token-by-token stream-out to pinned host memory on
one B200. One STEP = one generated token: its K/V (position p+t-1 of every layer, request and
head = 2*40*8*40 runs of 256 B = 6,553,600 B) is routed, packed and moved to a pinned-host log
with its sequence flag published -- all hot-path rows of SURVEY §8(a) for the host path
(route -> pack -> PCIe put -> completion flag). The paper streams tokens per step, not per layer
(PAPER.md:133); the per-layer form ("us per token-stream per layer") is reported in `extras`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--xfer auto|fused|staged]

N > 1 (torchrun): every rank is an independent pipeline stage streaming its own C2 cache to its own
pinned host memory (weak scaling, no data-path collective); time = max over ranks; `value` stays
this C2 figure at every N. The same line then carries "nvlink": the peer paths of north_star on
the N GPUs (tools/bench_peer.py nvlink_suite: in-run link peaks, C5 ring replication at P = N,
C3 N/2 -> N/2 disaggregation, their NCCL send/recv baselines, per-layer put latency with the
system-scope release, every delivered word verified on the device). Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ---- C2 workload ------------------------------------------------------------------------------------
L, H, D, B, P, S, E = 40, 40, 128, 8, 1000, 2048, 2
STEP_BYTES = 2 * L * B * H * D * E          # 6,553,600 B per token step
LAYER_BYTES = STEP_BYTES // L               # 163,840 B per token per layer
PROMPT_LAYER_BYTES = LAYER_BYTES * P        # 163,840,000 B per prompt layer
CONFIG = {"workload": "C2 OPT-13B shape (L40 H40 D128, fp16 words) b8 p1000 S2048: token-by-token "
                      "stream-out of every layer's new K/V to pinned host, 1 step = 1 token",
          "model": "OPT-13B KV-cache shape (no weights: pure data movement)",
          "global_batch": B, "seq_len": S, "prompt": P, "bytes_per_step": STEP_BYTES,
          "l2": "inputs larger than L2: 13.4 GB device cache, every step reads a fresh position "
                "(new 256-B lines); host log ring 64 steps = 419 MB"}
METRIC = "KV stream GB/s (token-step stream-out to pinned host)"
PCIE_NOMINAL_GBS = 64.0   # PCIe Gen5 x16 per direction (nominal)
def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# HBM roofline denominator (copy, read + write): the driver-written MEASURED_PEAKS.json of the box
# when present; else the value that file held on this round's first box (6534.8 GB/s; the
# profiling guide's own fallback is 6650)
_HBM = _peaks().get("hbm_gbs")
HBM_PEAK = float(_HBM) if _HBM else 6534.8
HBM_PEAK_SOURCE = "MEASURED_PEAKS.json (this box)" if _HBM else \
    "MEASURED_PEAKS.json hbm_gbs recorded earlier this round (file absent on this box)"


class Clocks:
    """nvidia-smi sampler running during the measured region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu,"
         "clocks.mem")

    def __init__(self, index):
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        rows = [r.split(", ") for r in out.strip().splitlines() if r.count(",") >= 10]
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        busy = [float(r[1]) for r in rows if r[9].strip().isdigit() and int(r[9]) > 0
                and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        mem = [float(r[10]) for r in rows if r[10].strip().replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(busy or sm) if (busy or sm) else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "mem_mhz": statistics.median(mem) if mem else None,
                "samples": len(rows), "samples_busy": len(busy)}


# =====================================================================================================
# our arm
# =====================================================================================================
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2403_01876_b200 as dv

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("DV_BENCH_SAME_DEVICE") == "1":   # test hook: all ranks on cuda:0 (gloo)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cpu_affinity = _bind_gpu_local_cpus(local)   # pinned buffers then land on the GPU's NUMA node
    backend = args.dist_backend
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    xfer = {"auto": dv.DV_XFER_AUTO, "fused": dv.DV_XFER_FUSED, "staged": dv.DV_XFER_STAGED,
            "decoupled": dv.DV_XFER_DECOUPLED}[args.xfer]
    ctx = dv.dv_create(local)
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device=dev)
    v = torch.empty_like(k)
    cache = dv.cache(k, v)
    seed = 20240304 + 1
    dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=seed)          # writer: every position written
    RING = 64
    log = torch.empty(RING * STEP_BYTES // 2, dtype=torch.int16, pin_memory=True)
    fl = torch.zeros(4, dtype=torch.int64, pin_memory=True)
    ep = dv.endpoint_of(log, fl)
    # the same log as the level-1 destination: a ring inbox of RING step-sized slots (token step t
    # lands in slot t % RING; include/dv.h rings), read by the host consumer -- no credits
    ring = dv.endpoint_array([dv.endpoint_of(log, fl, n_slots=RING, slot_bytes=STEP_BYTES)])
    stage = dv.Setup([0, L], [0, B], S)        # this GPU's stage: all C2 layers, one microbatch
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    npos = S - P

    def pos_of(t):            # token step t >= 1 writes p + t - 1 (reading Q4), wrapped inside S
        return P + (t - 1) % npos

    def step(t, xf=xfer):
        # the whole hot path per token step: route (level 1, A1) -> pack (A2) -> PCIe put (A3b) ->
        # seq flag (A5), through dv_stream_out into the host log's ring slot t % RING
        q = pos_of(t)
        dv.dv_stream_out(ctx, cache, (0, L, 0, B, q, q + 1), stage, 0, 0, stage, ring, seq=t, xfer=xf, stream=sp)

    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    t_ = 0
    for _ in range(args.warmup):
        t_ += 1
        step(t_)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    st_all, en_all = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0, dma0 = dv.dv_stats()
    st_all.record(stream)
    h0 = time.perf_counter()
    for i in range(args.steps):
        t_ += 1
        step(t_)
    host_us = (time.perf_counter() - h0) / args.steps * 1e6
    # the consumer's view: the timed region ends when the last step's flag is published (with
    # DV_XFER_DECOUPLED the DMA and flag run on the library's DMA stream, not on `stream`)
    dv.dv_wait(ctx, ep, 0, t_, stream=sp)
    en_all.record(stream)
    torch.cuda.synchronize()
    l1, dma1 = dv.dv_stats()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    elapsed_ms = st_all.elapsed_time(en_all)
    launches = l1 - l0
    # parity spot check of the last step against kvgen (the writer's definition), not timed
    last_q = pos_of(t_)
    wire = log[(t_ % RING) * STEP_BYTES // 2:(t_ % RING + 1) * STEP_BYTES // 2]
    assert int(fl[0]) == t_, "flag not published"
    spot = _spot_check(wire, last_q, seed)
    # and every word of the last 8 steps' wires on the device (dvt_verify vs the generator)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    for tt in range(max(1, t_ - 7), t_ + 1):
        w = log[(tt % RING) * STEP_BYTES // 2:(tt % RING + 1) * STEP_BYTES // 2]
        dv.dvt_verify(cache, cnt.data_ptr(), seed=seed, reg=dv.region(0, L, 0, B, pos_of(tt), pos_of(tt) + 1),
                      wire_ptr=w.data_ptr(), stream=sp)
    torch.cuda.synchronize()
    spot["full_steps_verified"] = min(8, t_)
    spot["full_words"] = min(8, t_) * STEP_BYTES // 2
    spot["full_mismatches"] = int(cnt.item())
    if world > 1:
        elapsed_ms = max_over_ranks(elapsed_ms)

    # ---- e2e: host buffers through the public API (H2D of the step's new K/V -> cache, stream-out)
    delta = torch.empty(RING * STEP_BYTES // 2, dtype=torch.int16, pin_memory=True)
    dfl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    dep = dv.endpoint_of(delta, dfl)
    for j in range(RING):   # the model's outputs for the next RING tokens, prepared on the host
        q = pos_of(j + 1)
        dv.dv_scatter(ctx, cache, dv.region(0, L, 0, B, q, q + 1), dep, j * STEP_BYTES,
                      xfer=dv.DV_XFER_FUSED, stream=sp)
    torch.cuda.synchronize()

    # input stream(s): with one, the input side (H2D + unpack) runs in lockstep with the output
    # side; two alternating streams let H2Ds overlap each other (DV_E2E_INSTREAMS, measured in
    # tools/probe_e2e_trace.py)
    s_ins = [torch.cuda.Stream() for _ in range(int(os.environ.get("DV_E2E_INSTREAMS", "1")))]
    evs = [torch.cuda.Event() for _ in range(8)]

    def e2e_step(t):
        # H2D of step t's new K/V on s_in (overlaps the D2H of step t-1 on the main stream: PCIe is
        # full duplex), then the stream-out of step t on the main stream once it has landed.
        q = pos_of(t)
        j = (t - 1) % RING
        s_in = s_ins[t % len(s_ins)]
        dv.dv_gather(ctx, dep, j * STEP_BYTES, cache, dv.region(0, L, 0, B, q, q + 1), stream=s_in)
        e = evs[t % 8]
        e.record(s_in)
        stream.wait_event(e)
        dv.dv_stream_out(ctx, cache, (0, L, 0, B, q, q + 1), stage, 0, 0, stage, ring, seq=10_000_000 + t,
                         xfer=xfer, stream=sp)
    for t in range(1, args.warmup + 1):
        e2e_step(t)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s_in in s_ins:
        s_in.wait_event(e0)
    h0 = time.perf_counter()
    for t in range(1, args.steps + 1):
        e2e_step(t)
    host_e2e_us = (time.perf_counter() - h0) / args.steps * 1e6
    dv.dv_wait(ctx, ep, 0, 10_000_000 + args.steps, stream=sp)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        e2e_ms = max_over_ranks(e2e_ms)

    extras = {}
    if not args.no_extras and rank == 0:
        extras = run_extras(dv, ctx, cache, stream, args, pos_of)
    nvlink = None
    if world > 1 and not args.no_nvlink:
        # the peer paths of north_star on the N GPUs of this box (tools/bench_peer.py): link peaks,
        # C5 ring replication, C3 disaggregation, NCCL send/recv baselines, every word verified
        from tools import bench_peer
        del k, v
        torch.cuda.empty_cache()
        env = bench_peer.Env(backend)
        env.local, env.dev = local, dev
        nvlink = bench_peer.nvlink_suite(ctx, env, steps=args.nvlink_steps)
    clk = clocks.stop()

    value = world * args.steps * STEP_BYTES / (elapsed_ms * 1e-3) / 1e9
    e2e_val = world * args.steps * STEP_BYTES / (e2e_ms * 1e-3) / 1e9
    # one fused kernel per step: its average duration <= elapsed / launches (gaps included, so the
    # achieved figure below is a lower bound)
    mean_kernel_ms = elapsed_ms / max(1, launches)
    peaks = _peaks()
    pcie_peak = extras.get("pcie_dma_d2h_peak_gbs")
    if rank != 0:
        dv.dv_destroy(ctx)
        if world > 1:
            dist.destroy_process_group()
        return
    if args.xfer in ("auto", "fused"):
        dram_traffic, pcie_traffic, tsrc = _ncu_traffic("fused")
        ach = STEP_BYTES / (mean_kernel_ms * 1e-3) / 1e9
        roof = {"bound": "pcie", "achieved": ach, "peak": pcie_peak, "unit": "GB/s",
                "frac": (ach / pcie_peak) if pcie_peak else None,
                "traffic": dram_traffic, "traffic_pcie_write": pcie_traffic,
                "traffic_source": tsrc + " (ncu dram__bytes_read+write, pcie__write_bytes per launch, median)",
                "kernel": "k_run_copy (fused pack -> pinned host zero-copy PCIe stores + st.release.sys flag)"}
    else:
        # decoupled / staged: the step's bytes cross PCIe by the copy engine (one cudaMemcpyAsync of
        # the packed step per step, back to back on the library's DMA stream); the pack kernel
        # (k_run_copy, cache -> HBM staging) is a few us of HBM work beside it. achieved = bytes per
        # step / device time per step (a lower bound of the DMA's own rate).
        dram_traffic, pcie_traffic, tsrc = _ncu_traffic("decoupled")
        ach = STEP_BYTES / (elapsed_ms / args.steps * 1e-3) / 1e9
        roof = {"bound": "pcie", "achieved": ach, "peak": pcie_peak, "unit": "GB/s",
                "frac": ach / pcie_peak if pcie_peak else None,
                "traffic": dram_traffic,
                "traffic_source": tsrc + ": ncu dram__bytes_read+write per launch of the pack kernel (HBM "
                                  "side; the copy engine's PCIe bytes are not a kernel counter), median",
                "kernel": "copy-engine D2H of the packed step (cudaMemcpyAsync on the library DMA "
                          "stream), fed by k_run_copy pack (cache -> HBM staging), flag by a stream "
                          "write on the library flag stream",
                "pack_kernel_us": extras.get("token_step_pack_hbm_us"),
                "pack_kernel_hbm_frac": extras.get("token_step_pack_hbm_frac"),
                "pack_kernel_vs_contiguous_same_size": extras.get("token_step_pack_vs_contiguous_same_size"),
                "pack_kernel_note": "a 6.55 MB launch is bound by fixed costs (dependent-launch floor "
                                    "extras.dependent_launch_floor_us), not by the gather pattern: the "
                                    "same kernel on a near-contiguous 6.55 MB takes "
                                    "extras.token_step_pack_contiguous_same_size_us"}
    roof.update({
        "peak_same_size_dma": extras.get("pcie_dma_d2h_same_size_gbs"),
        "algorithmic_bytes_per_launch": STEP_BYTES,
        "peak_nominal": PCIE_NOMINAL_GBS, "frac_nominal": roof["achieved"] / PCIE_NOMINAL_GBS,
        "peak_source": "in-run copy-engine D2H into pinned memory, this box: the best of 3 trials of 256 MiB "
                       "copies and of back-to-back step-sized (6.55 MB) copies; PCIe Gen5 x16 nominal 64 GB/s"})
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u16 (opaque fp16 words)",
        "data": "synthetic (splitmix64 coordinate-hash fill, seed 20240305)",
        "config": _config(world),
        "run": {"xfer": args.xfer, "cpu_affinity": cpu_affinity,
                "api": "dv_stream_out (level 1: route -> pack -> put -> flag) into a 64-slot ring in pinned host memory"},
        "e2e": {"value": e2e_val, "unit": "GB/s", "h2d_bytes_per_step": STEP_BYTES,
                "d2h_bytes_per_step": STEP_BYTES,
                "how": "per step: dv_gather of the token's K/V from pinned host into the device cache "
                       "(H2D + unpack, input stream) then dv_stream_out into the pinned-host ring log (route + pack + D2H, "
                       "main stream); step t+1's H2D overlaps step t's D2H (PCIe full duplex)"},
        "gpu_launches": int(launches),
        "copy_engine_dmas": int(dma1 - dma0),   # library cudaMemcpyAsync calls in the timed region
        "host_enqueue_us_per_step": {"value": host_us, "e2e": host_e2e_us},
        "roofline": roof,
        "clocks": clk,
        "parity_spot_check": spot,
        "us_per_token_layer": (extras.get("token_layer_latency", {}).get("host") or {}).get("p50_us"),
        "extras": extras,
    }
    if world > 1:
        line["nvlink"] = nvlink if nvlink is not None else {"skipped": "--no-nvlink"}
    if args.cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(seconds=args.cpu_seconds)
    print(json.dumps(line), flush=True)
    dv.dv_destroy(ctx)
    if world > 1:
        dist.destroy_process_group()


def _bind_gpu_local_cpus(index):
    """Bind this process to the CPUs NVML reports as local to GPU `index` (one rank per GPU on a
    multi-socket box: the first touch of its pinned host buffers then allocates on the socket whose
    PCIe root the GPU hangs off). Returns the CPU list, or None if NVML is unavailable."""
    try:
        import pynvml
        pynvml.nvmlInit()
        vis = [x.strip() for x in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if x.strip()]
        ident = vis[index] if index < len(vis) else str(index)
        h = (pynvml.nvmlDeviceGetHandleByIndex(int(ident)) if ident.isdigit()
             else pynvml.nvmlDeviceGetHandleByUUID(ident))
        pynvml.nvmlDeviceSetCpuAffinity(h)
        cpus = sorted(os.sched_getaffinity(0))
        return f"{cpus[0]}-{cpus[-1]} ({len(cpus)} cpus)" if cpus else None
    except Exception:   # noqa: BLE001 -- affinity is an optimisation, never a failure
        return None


def _config(world):
    """The workload's config -- identical in both arms (ours and --impl reference) at every N."""
    return dict(CONFIG, parallelism=f"independent stages x{world}" if world > 1 else "1 stage")


def _ncu_traffic(name="decoupled"):
    """DRAM and PCIe bytes per launch of the headline kernel from the committed ncu capture of this
    same command (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,pcie__write_bytes.sum),
    median over the captured launches of the pack kernel. Returns (dram, pcie, source) where the
    source names the file and the sha256 of its content (so the line pins the exact capture)."""
    import csv
    import hashlib
    files = {"decoupled": ["r02d_io_counters.csv", "r02b_io_counters.csv", "r02_io_counters.csv", "r01g_io_counters.csv"],
             "fused": ["r02_io_counters_fused.csv", "r01_io_counters_final.csv"]}[name]
    for fn in files:
        path = os.path.join(ROOT, "profiles", fn)
        try:
            raw = open(path, "rb").read()
        except OSError:
            continue
        rows = [r for r in csv.reader(l for l in raw.decode().splitlines() if l.startswith('"'))]
        hdr, body = rows[0], rows[1:]
        per = {}
        for r in body:
            d = dict(zip(hdr, r))
            if "k_run_copy" not in d.get("Kernel Name", "k_run_copy"):
                continue
            per.setdefault(d["ID"], {})[d["Metric Name"]] = float(d["Metric Value"])
        dram = sorted(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in per.values())
        pcie = sorted(v.get("pcie__write_bytes.sum", 0) for v in per.values())
        if dram:
            return (dram[len(dram) // 2], pcie[len(pcie) // 2],
                    f"profiles/{fn} sha256:{hashlib.sha256(raw).hexdigest()[:16]}")
    return None, None, None


def _spot_check(wire, q, seed):
    """Sampled parity of one streamed step vs kvgen's definition (the writer's words). The wire of a
    one-position region is the canonical [l][kv][r][h][d] order (Q3); bench.py does not
    import the oracle outside its cpu_baseline leg -- the oracle's own parity runs are in tests/."""
    import numpy as np

    import kvgen
    w = wire.cpu().numpy().view(np.uint16)
    rng = np.random.default_rng(0)
    n = 4096
    l = rng.integers(0, L, n); kv = rng.integers(0, 2, n); r = rng.integers(0, B, n)
    h = rng.integers(0, H, n); d = rng.integers(0, D, n)
    idx = (((l * 2 + kv) * B + r) * H + h) * D + d
    exp = kvgen.hash_words(kv, l, r, h, np.full(n, q), d, seed)
    bad = int(np.sum(w[idx] != exp))
    assert bad == 0, f"{bad} sampled words differ from the writer's definition"
    return {"samples": n, "mismatches": bad}


def sample_region(k, v, layer_begin, req_begin, n_heads, max_seq, head_dim, region, seed, n=20000):
    """Sampled parity of a KV5D cache region against kvgen's definition (words at global coords)."""
    import numpy as np
    import torch

    import kvgen
    rng = np.random.default_rng(7)
    l0, l1, r0, r1, s0, s1 = region
    nR = k.shape[1]
    l = rng.integers(l0, l1, n); r = rng.integers(r0, r1, n); s = rng.integers(s0, s1, n)
    h = rng.integers(0, n_heads, n); d = rng.integers(0, head_dim, n); kv = rng.integers(0, 2, n)
    exp = kvgen.hash_words(kv, l, r, h, s, d, seed)
    idx = ((((l - layer_begin) * nR + (r - req_begin)) * n_heads + h) * max_seq + s) * head_dim + d
    it = torch.from_numpy(idx.astype(np.int64)).to(k.device)
    gk = k.view(-1)[it].cpu().numpy().view(np.uint16)
    gv = v.view(-1)[it].cpu().numpy().view(np.uint16)
    return int(np.sum(np.where(kv == 0, gk, gv) != exp))


def _time(fn, stream, reps, warm=2, tail=None, head_start_ns=0):
    """Mean device time per call. head_start_ns: a spin kernel first, so the calls queue up behind
    it and the timing sees device time, not the host's enqueue rate (short kernels)."""
    import torch
    import paper_2403_01876_b200 as dv
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if head_start_ns:
        dv.dvt_spin(head_start_ns, 1, stream=stream.cuda_stream)
    a.record(stream)
    for _ in range(reps):
        fn()
    if tail:
        tail()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def _latency_fused_producer(dv, ctx, cache, stream, n=440):
    """Per-layer token latency with the stream-out FUSED INTO THE PRODUCER (device plans,
    include/dv.h dv_dplan_*) vs the separate stream-out kernel behind it (dv_scatter, PDL): the
    same vectorised producer (dvt_fill_rows) writes one layer's new K/V (C2: 160 KiB); stamps at the
    producer's start, its end and the flag release. start -> flag = "write the layer's K/V and make
    it visible at the destination" (tools/probe_fused_latency.py has the loaded variant)."""
    import torch
    sp = stream.cuda_stream
    out = {}
    for dst_host in (True, False):
        dev = "cpu" if dst_host else "cuda"
        log = torch.empty(L * LAYER_BYTES // 2, dtype=torch.int16, device=dev, pin_memory=dst_host)
        fl = torch.zeros(L, dtype=torch.int64, device=dev, pin_memory=dst_host)
        ep = dv.endpoint_of(log, fl)
        plans = [dv.dv_dplan_scatter(ctx, cache, dv.region(l, l + 1, 0, B, P, P + 1), ep, l * LAYER_BYTES, 0,
                                     flag_slot=l, seq=1, max_step=S - P - 1) for l in range(L)]
        res = {}
        seq = [10 ** 6]
        for arm in ("fused", "separate"):
            t0 = torch.full((n,), 2 ** 63 - 1, dtype=torch.int64, device="cuda")
            te = torch.zeros(n, dtype=torch.int64, device="cuda")
            ts = torch.zeros((n, 4), dtype=torch.int64, device="cuda")
            ts[:, 1:3] = 2 ** 63 - 1

            def one(i, arm=arm, t0=t0, te=te, ts=ts):
                layer, step = i % L, i // L
                reg = dv.region(layer, layer + 1, 0, B, P + step, P + step + 1)
                if arm == "fused":
                    plans[layer].trace = ts[i].data_ptr()
                    dv.dvt_fill_rows(cache, 20240305, reg, plans[layer], step, t_start_ptr=t0[i].data_ptr(),
                                     t_end_ptr=te[i].data_ptr(), stream=sp)
                else:
                    dv.dvt_fill_rows(cache, 20240305, reg, None, 0, t_start_ptr=t0[i].data_ptr(),
                                     t_end_ptr=te[i].data_ptr(), stream=sp)
                    dv.dvt_trace(ctx, ts[i].data_ptr())
                    seq[0] += 1
                    dv.dv_scatter(ctx, cache, reg, ep, layer * LAYER_BYTES, flag_slot=layer, seq=seq[0],
                                  xfer=dv.DV_XFER_FUSED, stream=sp)
            for i in range(L):
                one(i)
            dv.dvt_trace(ctx, 0)
            torch.cuda.synchronize()
            dv.dvt_spin(20_000_000, 1, stream=sp)
            for i in range(n):
                one(i)
            dv.dvt_trace(ctx, 0)
            torch.cuda.synchronize()
            a = sorted(((ts[:, 0] - t0).double() / 1e3).tolist()[L:])
            b = sorted(((ts[:, 0] - te).double() / 1e3).tolist()[L:])
            res[arm] = {"start_to_flag_p50_us": a[len(a) // 2], "start_to_flag_p99_us": a[int(len(a) * 0.99)],
                        "producer_end_to_flag_p50_us": b[len(b) // 2], "n": len(a)}
        out["host" if dst_host else "hbm"] = res
        torch.cuda.synchronize()
        for pl in plans:
            dv.dv_dplan_free(ctx, pl)
    return out


def _latency_under_gemm(dv, ctx, cache, lep, pos_of, n=400, n_gemm=60):
    """Per-layer token latency to pinned host (writer end -> flag, C2 layer of 160 KiB) while a bf16
    GEMM loop (8192^3) saturates the GPU -- NEXT-2's concurrent compute -- in two arrangements:
    'priority': GEMM on a low-priority stream, writer + stream-out on a high-priority one (all SMs
    shared); 'partition_<k>': dv_partition_create -- GEMM on the compute partition's stream,
    writer + stream-out on the k-SM streaming partition's stream (DESIGN.md §6 "SM partitions").
    Also the GEMM's TFLOP/s during each run (the partition's price)."""
    import torch
    lo_pr, hi_pr = torch.cuda.Stream.priority_range()
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    bm = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    out = {}
    seq = [4 * 10 ** 8]
    part = dv.dv_partition_create(torch.cuda.current_device(), 16, hi_pr)
    try:
        arr = {"priority": (torch.cuda.Stream(priority=hi_pr), torch.cuda.Stream(priority=lo_pr)),
               f"partition_{part.sms_streaming}": (torch.cuda.ExternalStream(part.streaming),
                                                    torch.cuda.ExternalStream(part.compute))}
        for name, (cs, gs) in arr.items():
            sp = cs.cuda_stream
            with torch.cuda.stream(gs):
                torch.matmul(a, bm)
            for i in range(2 * L):   # warm the kernels on these streams
                reg = dv.region(i % L, i % L + 1, 0, B, P, P + 1)
                dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=20240305, reg=reg, stream=sp)
                seq[0] += 1
                dv.dv_scatter(ctx, cache, reg, lep, (i % L) * LAYER_BYTES, flag_slot=0, seq=seq[0],
                              xfer=dv.DV_XFER_FUSED, stream=sp)
            te = torch.zeros(n, dtype=torch.int64, device="cuda")
            ts = torch.zeros((n, 4), dtype=torch.int64, device="cuda")
            ts[:, 1:3] = 2 ** 63 - 1
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(gs)
            with torch.cuda.stream(gs):
                for _ in range(n_gemm):
                    torch.matmul(a, bm)
            g1.record(gs)
            dv.dvt_spin(20_000_000, 1, stream=sp)
            for i in range(n):
                layer = i % L
                q = pos_of(2 + i // L)
                reg = dv.region(layer, layer + 1, 0, B, q, q + 1)
                dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=20240305, reg=reg, stream=sp, t_end_ptr=te[i].data_ptr())
                dv.dvt_trace(ctx, ts[i].data_ptr())
                seq[0] += 1
                dv.dv_scatter(ctx, cache, reg, lep, layer * LAYER_BYTES, flag_slot=0, seq=seq[0],
                              xfer=dv.DV_XFER_FUSED, stream=sp)
            dv.dvt_trace(ctx, 0)
            torch.cuda.synchronize()
            d = sorted(((ts[:, 0] - te).double() / 1e3).tolist()[L:])
            out[name] = {"p50_us": d[len(d) // 2], "p99_us": d[int(len(d) * 0.99)], "n": len(d),
                         "gemm_tflops_during": n_gemm * 2 * 8192 ** 3 / (g0.elapsed_time(g1) * 1e-3) / 1e12}
        out["sms"] = {"streaming": part.sms_streaming, "compute": part.sms_compute}
    finally:
        torch.cuda.synchronize()
        part.destroy()
    return out


def run_extras(dv, ctx, cache, stream, args, pos_of):
    """Secondary measurements reported beside the headline (same run, same box)."""
    import torch
    sp = stream.cuda_stream
    ex = {}
    # PCIe DMA peaks (roofline denominators for the host path), 256 MiB pinned
    n = 256 << 20
    hb = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    db = torch.empty(n, dtype=torch.uint8, device="cuda")
    # best of 3 trials of 5 copies each: the link's rate varies by a few % run to run under the
    # power cap, and a peak is the best observed, not one sample
    ms = min(_time(lambda: hb.copy_(db, non_blocking=True), stream, 5) for _ in range(3))
    ex["pcie_dma_d2h_gbs"] = n / ms / 1e6
    ms = min(_time(lambda: db.copy_(hb, non_blocking=True), stream, 5) for _ in range(3))
    ex["pcie_dma_h2d_gbs"] = n / ms / 1e6
    # the same 6.55 MB per transfer as one token step, back to back (fixed costs included)
    ms = min(_time(lambda: hb[:STEP_BYTES].copy_(db[:STEP_BYTES], non_blocking=True), stream, 100)
             for _ in range(3))
    ex["pcie_dma_d2h_same_size_gbs"] = STEP_BYTES / ms / 1e6
    # the roofline's denominator: the best D2H rate the copy engine showed in this run (either size)
    ex["pcie_dma_d2h_peak_gbs"] = max(ex["pcie_dma_d2h_gbs"], ex["pcie_dma_d2h_same_size_gbs"])
    del hb, db

    # token step: fused vs staged (host), and pack-only into HBM
    log = torch.empty(STEP_BYTES // 2 * 8, dtype=torch.int16, pin_memory=True)
    ep = dv.endpoint_of(log)
    dbuf = torch.empty(STEP_BYTES // 2 * 8, dtype=torch.int16, device="cuda")
    dep = dv.endpoint_of(dbuf)
    cnt = [0]

    tfl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    epf = dv.endpoint_of(log, tfl)

    def tok(epx, xf, flag=False):
        def f():
            cnt[0] += 1
            q = pos_of(cnt[0])
            dv.dv_scatter(ctx, cache, dv.region(0, L, 0, B, q, q + 1), epx, (cnt[0] % 8) * STEP_BYTES,
                          flag_slot=0 if flag else -1, seq=cnt[0], xfer=xf, stream=sp)
        return f
    reps = 200
    for name, epx, xf in (("fused", ep, dv.DV_XFER_FUSED), ("staged", ep, dv.DV_XFER_STAGED),
                          ("decoupled", epf, dv.DV_XFER_DECOUPLED)):
        dec = name == "decoupled"
        ms = _time(tok(epx, xf, dec), stream, reps,
                   tail=(lambda: dv.dv_wait(ctx, epf, 0, cnt[0], stream=sp)) if dec else None)
        ex[f"token_step_host_{name}_gbs"] = STEP_BYTES / ms / 1e6
        ex[f"token_step_host_{name}_us"] = ms * 1e3
    for name, xf in (("fused", dv.DV_XFER_FUSED), ("staged", dv.DV_XFER_STAGED)):
        def g(xf=xf):
            cnt[0] += 1
            q = pos_of(cnt[0])
            dv.dv_gather(ctx, ep, (cnt[0] % 8) * STEP_BYTES, cache, dv.region(0, L, 0, B, q, q + 1), xfer=xf,
                         stream=sp)
        ms = _time(g, stream, reps)
        ex[f"token_step_gather_host_{name}_gbs"] = STEP_BYTES / ms / 1e6
    ms = _time(tok(dep, dv.DV_XFER_FUSED), stream, reps, head_start_ns=4_000_000)
    ex["token_step_pack_hbm_us"] = ms * 1e3
    ex["token_step_pack_hbm_gbs_2R"] = 2 * STEP_BYTES / ms / 1e6
    ex["token_step_pack_hbm_frac"] = ex["token_step_pack_hbm_gbs_2R"] / HBM_PEAK
    ex["hbm_peak_gbs"] = HBM_PEAK
    ex["hbm_peak_source"] = HBM_PEAK_SOURCE
    # the practical floor for a launch of this size: a contiguous 6.55 MB device-to-device copy
    # (cudaMemcpyAsync via torch), source ring larger than L2, same head start, back to back
    src_d = torch.empty(STEP_BYTES * 40, dtype=torch.uint8, device="cuda")   # 262 MB ring > L2
    dst_d = torch.empty(STEP_BYTES, dtype=torch.uint8, device="cuda")
    ce = [0]

    def d2d():
        ce[0] += 1
        o = (ce[0] % 40) * STEP_BYTES
        dst_d.copy_(src_d[o:o + STEP_BYTES], non_blocking=True)
    ms = _time(d2d, stream, reps, head_start_ns=4_000_000)
    ex["token_step_same_size_d2d_copy_us"] = ms * 1e3
    ex["token_step_pack_vs_same_size_copy"] = ex["token_step_same_size_d2d_copy_us"] / ex["token_step_pack_hbm_us"]
    del src_d, dst_d
    # the same pack kernel on a near-contiguous 6.55 MB (positions [0,320) of one layer and
    # request: 80 runs of 80 KiB, cycled over layers / requests) and the smallest dependent launch
    # (one position of one head: 512 B) -- DESIGN.md §6 "Token-step pack, where its 4 us go"
    def contig():
        cnt[0] += 1
        lay, rq = cnt[0] % L, (cnt[0] // L) % B
        dv.dv_scatter(ctx, cache, dv.region(lay, lay + 1, rq, rq + 1, 0, 320), dep, (cnt[0] % 8) * STEP_BYTES,
                      stream=sp)

    def tiny():
        cnt[0] += 1
        q = pos_of(cnt[0])
        dv.dv_scatter(ctx, cache, dv.region(0, 1, 0, 1, q, q + 1, 0, 1), dep, (cnt[0] % 8) * 1024, stream=sp)
    ex["token_step_pack_contiguous_same_size_us"] = _time(contig, stream, reps, head_start_ns=4_000_000) * 1e3
    ex["token_step_pack_vs_contiguous_same_size"] = (ex["token_step_pack_contiguous_same_size_us"]
                                                     / ex["token_step_pack_hbm_us"])
    ex["dependent_launch_floor_us"] = _time(tiny, stream, reps, head_start_ns=4_000_000) * 1e3
    ex["xfer_main"] = "fused" if args.xfer in ("auto", "fused") else args.xfer

    # per-layer token latency: from "layer l's new K/V written" to "bytes resident at
    # the destination and seq flag visible". The writer is dvt_fill of that layer's new position
    # (a PDL-aware producer); times are %globaltimer stamps taken by the writer after its stores
    # and by the stream-out kernel right after its st.release.sys of the flag.
    lat = {}
    fl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    lep = dv.endpoint_of(log, fl)
    dlog = torch.empty(LAYER_BYTES // 2 * L, dtype=torch.int16, device="cuda")
    dfl = torch.zeros(1, dtype=torch.int64, device="cuda")
    n = 1040   # SURVEY §8(d) latency runs: 1000 token·layer samples after a 40-sample warm-up

    def lat_run(epx, seq0, watch):
        """n per-layer stream-outs, each right behind its writer; returns (te, ts, tw) stamps."""
        te = torch.zeros(n, dtype=torch.int64, device="cuda")
        ts = torch.zeros((n, 4), dtype=torch.int64, device="cuda")
        ts[:, 1:3] = 2 ** 63 - 1
        tw = torch.zeros(n, dtype=torch.int64, device="cuda")
        wst = torch.cuda.Stream()
        if watch:
            # an independent observer: one GPU thread on its own stream polls the flag (system-
            # scope acquire loads; over PCIe for the host flag) and stamps when each seq becomes
            # visible (its PCIe polling competes with the stream-out's own flush, so it runs in a
            # separate pass from the published-flag stamps)
            dv.dvt_watch(epx.flags, seq0, n, tw.data_ptr(), 5_000_000_000, stream=wst.cuda_stream)
        # head start: the GPU must run behind the host (as it does in serving), so the stream-out
        # launch is queued before its producer finishes and PDL can take effect
        dv.dvt_spin(20_000_000, 1, stream=sp)
        for i in range(n):
            q = pos_of(1 + i // L)
            layer = i % L
            reg = dv.region(layer, layer + 1, 0, B, q, q + 1)
            dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=20240305, reg=reg, stream=sp, t_end_ptr=te[i].data_ptr())
            if not watch:
                dv.dvt_trace(ctx, ts[i].data_ptr())
            dv.dv_scatter(ctx, cache, reg, epx, layer * LAYER_BYTES, flag_slot=0, seq=seq0 + i,
                          xfer=dv.DV_XFER_FUSED, stream=sp)
        dv.dvt_trace(ctx, 0)
        torch.cuda.synchronize()
        return te, ts, tw

    def pct(x):
        x = sorted(x[L:])
        return x[len(x) // 2], x[int(len(x) * 0.99)], x[0]

    for name, epx in (("host", lep), ("hbm", dv.endpoint_of(dlog, dfl))):
        # every kernel of the loop (and the watcher) runs once first: with CUDA lazy loading,
        # loading a kernel while the watcher spins would wait for the watcher
        tw0 = torch.zeros(1, dtype=torch.int64, device="cuda")
        dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=20240305, reg=dv.region(0, 1, 0, B, P, P + 1), stream=sp,
                    t_end_ptr=tw0.data_ptr())
        dv.dv_scatter(ctx, cache, dv.region(0, 1, 0, B, P, P + 1), epx, 0, flag_slot=0, seq=10 ** 7,
                      xfer=dv.DV_XFER_FUSED, stream=sp)
        dv.dvt_watch(epx.flags, 0, 1, tw0.data_ptr(), 1000, stream=sp)
        torch.cuda.synchronize()
        te, ts, _ = lat_run(epx, 10 ** 8, False)
        p50, p99, mn = pct(((ts[:, 0] - te).double() / 1e3).tolist())
        te, _, tw = lat_run(epx, 10 ** 8 + n, True)
        o50, o99, _ = pct(((tw - te).double() / 1e3).tolist())
        lat[name] = {"p50_us": p50, "p99_us": p99, "min_us": mn, "n": n - L,
                     "how": "writer-end -> flag-published, %globaltimer",
                     "observed": {"p50_us": o50, "p99_us": o99,
                                  "how": "separate pass: writer-end -> a polling GPU thread reads the seq "
                                         "(dvt_watch; for the host flag each poll is a PCIe read)"}}
    # the same with a CUDA event between writer and stream-out (breaks PDL, adds the launch gap)
    samples = []
    for i in range(n):
        q = pos_of(1 + i // L)
        layer = i % L
        reg = dv.region(layer, layer + 1, 0, B, q, q + 1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=20240305, reg=reg, stream=sp)
        a.record(stream)
        dv.dv_scatter(ctx, cache, reg, lep, layer * LAYER_BYTES, flag_slot=0, seq=2 * 10 ** 8 + i,
                      xfer=dv.DV_XFER_FUSED, stream=sp)
        b.record(stream)
        samples.append((a, b))
    torch.cuda.synchronize()
    us = sorted(a.elapsed_time(b) * 1e3 for a, b in samples)
    lat["host_event_bracketed"] = {"p50_us": us[len(us) // 2], "p99_us": us[int(len(us) * 0.99)], "n": len(us)}
    t0 = time.perf_counter()
    for layer in range(L):
        dv.dv_scatter(ctx, cache, dv.region(layer, layer + 1, 0, B, P, P + 1), lep, layer * LAYER_BYTES,
                      flag_slot=0, seq=3 * 10 ** 8 + layer, xfer=dv.DV_XFER_FUSED, stream=sp)
    lat["host_enqueue_us_per_call"] = (time.perf_counter() - t0) / L * 1e6
    torch.cuda.synchronize()
    ex["token_layer_latency"] = lat
    try:
        ex["token_layer_latency_fused_producer"] = _latency_fused_producer(dv, ctx, cache, stream)
    except Exception as e:   # noqa: BLE001 -- reported; the rest of the line stands
        ex["token_layer_latency_fused_producer"] = {"error": f"{type(e).__name__}: {e}"}
    try:
        ex["token_layer_latency_under_gemm"] = _latency_under_gemm(dv, ctx, cache, lep, pos_of)
    except Exception as e:   # noqa: BLE001 -- reported; the rest of the line stands
        ex["token_layer_latency_under_gemm"] = {"error": f"{type(e).__name__}: {e}"}

    # CUDA graph of one token step's 40 per-layer stream-outs (captured once, replayed per token
    # with a device-side step counter): host cost per step and device time per step
    d_step = torch.zeros(1, dtype=torch.int32, device="cuda")
    g = torch.cuda.CUDAGraph()
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        with torch.cuda.graph(g, stream=gs):
            for layer in range(L):
                dv.dv_scatter_dyn(ctx, cache, dv.region(layer, layer + 1, 0, B, P, P + 1), lep, layer * LAYER_BYTES,
                                  0, d_step.data_ptr(), S - P - 1, flag_slot=0, seq=4 * 10 ** 8)
    torch.cuda.synchronize()
    reps = 200
    with torch.cuda.stream(gs):
        for i in range(5):
            d_step.fill_(i)
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(gs)
        for i in range(reps):
            d_step.fill_(i % (S - P))
            g.replay()
        b.record(gs)
        t_host = time.perf_counter() - t0
        torch.cuda.synchronize()
    ex["graph_token_step_40_layer_calls"] = {
        "host_us_per_step": t_host / reps * 1e6, "gpu_us_per_step": a.elapsed_time(b) / reps * 1e3,
        "eager_host_us_per_step": lat["host_enqueue_us_per_call"] * L}

    # prompt layer (163.8 MB) stream-out: fused vs staged, and HBM pack
    pbuf = torch.empty(PROMPT_LAYER_BYTES // 2, dtype=torch.int16, pin_memory=True)
    pep = dv.endpoint_of(pbuf)
    pd = torch.empty(PROMPT_LAYER_BYTES // 2, dtype=torch.int16, device="cuda")
    pdep = dv.endpoint_of(pd)
    lay = [0]

    def prm(epx, xf):
        def f():
            lay[0] = (lay[0] + 1) % L
            dv.dv_scatter(ctx, cache, dv.region(lay[0], lay[0] + 1, 0, B, 0, P), epx, 0, xfer=xf, stream=sp)
        return f
    for name, epx, xf in (("fused", pep, dv.DV_XFER_FUSED), ("staged", pep, dv.DV_XFER_STAGED)):
        ms = _time(prm(epx, xf), stream, 5)
        ex[f"prompt_layer_host_{name}_gbs"] = PROMPT_LAYER_BYTES / ms / 1e6
    ms = _time(prm(pdep, dv.DV_XFER_FUSED), stream, 10)
    ex["prompt_layer_pack_hbm_gbs_2R"] = 2 * PROMPT_LAYER_BYTES / ms / 1e6
    ex["prompt_layer_pack_hbm_frac"] = ex["prompt_layer_pack_hbm_gbs_2R"] / HBM_PEAK
    del pbuf, pd

    # the paper's prior-art copy methods on the same token step (Fig. 11 "Baseline" and Opt (1))
    out = torch.empty(STEP_BYTES // 2, dtype=torch.int16, pin_memory=True)
    stg = torch.empty(STEP_BYTES // 2, dtype=torch.int16, device="cuda")
    q = pos_of(1)
    reg = dv.region(0, L, 0, B, q, q + 1)
    ms = _time(lambda: dv.dvb_per_run_copy(cache, reg, out.data_ptr(), stream=sp), stream, 2, warm=1)
    ex["baseline_per_run_memcpy_us"] = ms * 1e3
    ms = _time(lambda: dv.dvb_buffered_copy(cache, reg, stg.data_ptr(), out.data_ptr(), stream=sp), stream, 10)
    ex["baseline_buffered_2d_memcpy_us"] = ms * 1e3
    ex["speedup_buffered_vs_per_run"] = ex["baseline_per_run_memcpy_us"] / ex["baseline_buffered_2d_memcpy_us"]
    ex["speedup_ours_vs_buffered"] = ex["baseline_buffered_2d_memcpy_us"] / ex["token_step_host_fused_us"]

    # NEXT-2: token streaming overlapped with a synthetic model step:
    # paired ABBA trials, step / compute slowdown with a 95 % CI, m, every streamed word verified
    from tools import bench_overlap
    ex["overlap"] = bench_overlap.measure(ctx, cache, 20240305)
    return ex


# =====================================================================================================
# CPU oracle arm (cpu_baseline and --impl reference)
# =====================================================================================================
class OracleStep:
    """The oracle's token step on a host-resident C2 cache: route -> pack -> transfer into a host
    log. Only the positions it streams are materialised (np.zeros is lazy), filled by kvgen."""

    def __init__(self, n_pos=16):
        import numpy as np

        import kvgen
        from oracle import kvstream as ok
        self.ok, self.np = ok, np
        self.K = np.zeros((L, B, H, S, D), np.uint16)
        self.V = np.zeros((L, B, H, S, D), np.uint16)
        self.n_pos = n_pos
        for j in range(n_pos):
            q = P + j
            for kv, arr in ((0, self.K), (1, self.V)):
                arr[:, :, :, q, :] = kvgen.logical_block("hash", kv, range(L), range(B), H, [q], D,
                                                         20240305)[:, :, :, 0, :]
        self.cache = ok.Cache(self.K, self.V, 0, 0, H, S, D)
        self.setup = ok.Setup([0, L], [0, B], S)
        self.log = np.empty(STEP_BYTES // 2 * 4, np.uint16)
        self.t = 0

    def step(self, pool=None):
        ok = self.ok
        q = P + self.t % self.n_pos
        reg = (0, L, 0, B, q, q + 1)
        o = (self.t % 4) * (STEP_BYTES // 2)
        for p in ok.route(self.setup, self.setup, reg, H, D, E):
            r = p.region()
            if pool is None:
                wire = ok.transfer(ok.pack(self.cache, r))
                self.log[o:o + wire.size] = wire
                continue
            # all cores (SURVEY §8(d) oracle timing (ii)): the same oracle calls, one per layer
            # slab of the piece, on a thread pool (numpy releases the GIL while copying)
            slab = LAYER_BYTES // 2 * (r[5] - r[4])

            def one(layer, r=r):
                w = ok.transfer(ok.pack(self.cache, (layer, layer + 1) + tuple(r[2:])))
                j = o + (layer - r[0]) * slab
                self.log[j:j + w.size] = w
            list(pool.map(one, range(r[0], r[1])))
        self.t += 1


def cpu_baseline(seconds=10.0):
    o = OracleStep()
    o.step()
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < seconds:
        o.step()
        n += 1
    dt = time.perf_counter() - t0
    out = {"value": n * STEP_BYTES / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
           "sample": f"{n} C2 token steps (route+pack+transfer of 6,553,600 B each) over "
                     f"{o.n_pos} distinct positions of a lazily materialised 13.4 GB host cache, "
                     f"{dt:.1f} s, numpy single-threaded"}
    from concurrent.futures import ThreadPoolExecutor
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    with ThreadPoolExecutor(cores) as pool:
        o.step(pool)
        t0 = time.perf_counter()
        m = 0
        while time.perf_counter() - t0 < seconds / 2:
            o.step(pool)
            m += 1
        dt2 = time.perf_counter() - t0
    out["all_cores"] = {"value": m * STEP_BYTES / dt2 / 1e9, "unit": "GB/s", "cores": cores,
                        "sample": f"{m} C2 token steps, the same oracle calls per layer slab on a "
                                  f"{cores}-thread pool, {dt2:.1f} s"}
    # the host's own roofline: one 1 GiB numpy copy (single thread), and the CPU model
    import numpy as np
    a = np.ones(1 << 30, np.uint8)
    b = np.empty_like(a)
    np.copyto(b, a)
    t0 = time.perf_counter()
    np.copyto(b, a)
    out["host_copy_1GiB_gbs"] = (1 << 30) / (time.perf_counter() - t0) / 1e9
    del a, b
    try:
        out["cpu_model"] = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if "model name" in l)
    except (OSError, StopIteration):
        out["cpu_model"] = None
    out["os_cpu_count"] = os.cpu_count()
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    o = OracleStep()
    for _ in range(args.warmup):
        o.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.step()
    dt = time.perf_counter() - t0
    val = args.steps * STEP_BYTES / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s",
            "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u16 (opaque fp16 words)", "data": "synthetic",
            "config": _config(int(os.environ.get("WORLD_SIZE", "1"))),
            "run": {"oracle": "numpy, one host process (rank 0 at N > 1)"},
            "cpu_baseline": {"value": val, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} timed C2 token steps of the numpy oracle on host cores"},
            "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--xfer", default="decoupled", choices=["auto", "fused", "staged", "decoupled"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--no-nvlink", action="store_true", help="N > 1: skip the peer-path suite in the JSON line")
    ap.add_argument("--nvlink-steps", type=int, default=200, help="N > 1: C5 token steps timed in the peer suite")
    ap.add_argument("--peer-baseline", default="none", choices=["none", "nccl"],
                    help="c3/c5: run the NCCL send/recv baseline (pack -> ncclSend/ncclRecv -> unpack) instead of dvstream's peer stores")
    ap.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"],
                    help="c2 (default, BASELINE configs[1]): token steps -> pinned host; "
                         "c3: prompt->token disaggregation over NVLink; c4: microbatch swap over PCIe; "
                         "c5: ring replication over NVLink")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and int(os.environ.get("RANK", "0")) != 0:
        args.cpu_baseline = False
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c2":
        run_ours(args)
    elif args.workload == "c4":
        from tools import bench_swap
        bench_swap.run_c4(args, sys.modules[__name__])
    else:
        from tools import bench_peer
        (bench_peer.run_c3 if args.workload == "c3" else bench_peer.run_c5)(args, sys.modules[__name__])


if __name__ == "__main__":
    main()
