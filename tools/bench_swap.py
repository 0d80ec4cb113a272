"""C4 swap workload for bench.py (`--workload c4`, BASELINE.json configs[3]): BLOOM-176B shape (112
heads, head_dim 128), one pipeline stage of 9 layers, microbatch b = 4, S = 2048, host arenas in the
log form. One STEP = one rotation event of PAPER.md:270-272 at
this stage: the delta of microbatch x-1's last token step (one position, 2.06 MB) is swapped out to
its host log (decoupled: pack + copy-engine DMA + flag), then microbatch x+1's whole prefix
(i = 2048 positions, PAPER.md:572 transf_i = i*B*C: the 1024-token prompt chunk + 1024 step chunks,
4.23 GB) is swapped in from its host log into the freed device slot (copy-engine DMA + unpack).
The metric is GB/s of KV bytes moved per step (dominated by the swap-in over PCIe H2D). N > 1:
every rank is an independent stage (weak scaling; the shared resource is the host PCIe fabric).
Two microbatch logs alternate to bound pinned memory (8.5 GB per rank).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

H, D, b, S, nL, P0, I = 112, 128, 4, 2048, 9, 1024, 2048
SEED = 20240307


def run_c4(args, bench):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if os.environ.get("DV_BENCH_SAME_DEVICE") == "1" else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group(args.dist_backend, **({"device_id": dev} if args.dist_backend == "nccl" else {}))
    ctx = dv.dv_create(local, staging_bytes=1 << 30)
    C = 2 * H * D * 2
    step_b = b * C * nL                     # one position of the stage: 2,064,384 B
    nb_in = I * step_b                      # the swap-in prefix: 4,227,858,432 B
    # the running microbatch's slot (source of the swap-outs) and the free slot (swap-in target)
    run_k = torch.empty((nL, b, H, S, D), dtype=torch.int16, device=dev)
    run_v = torch.empty_like(run_k)
    run = dv.cache(run_k, run_v)
    dv.dvt_fill(run, dv.DVT_FILL_HASH, seed=SEED)
    free_k = torch.full_like(run_k, -1)
    free_v = torch.full_like(run_v, -1)
    free = dv.cache(free_k, free_v)
    # two host logs (microbatches x+1 alternate between them), built by the stream-outs of the
    # prompt (one chunk) and of 1024 token steps (one chunk each)
    logs, eps = [], []
    for j in range(2):
        lg = torch.empty(nb_in // 2, dtype=torch.int16, pin_memory=True)
        ep = dv.endpoint_of(lg)
        dv.dv_scatter(ctx, run, (0, nL, 0, b, 0, P0), ep, 0)
        for t in range(I - P0):
            dv.dv_scatter(ctx, run, (0, nL, 0, b, P0 + t, P0 + t + 1), ep, (P0 + t) * step_b)
        logs.append(lg)
        eps.append(ep)
    out_log = torch.empty(step_b * 64 // 2, dtype=torch.int16, pin_memory=True)
    out_fl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    out_ep = dv.endpoint_of(out_log, out_fl)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    seq = [0]

    def step(t):
        seq[0] += 1
        q = P0 + (t % (I - P0))
        # (c) swap-out of x-1's step delta to its host log (decoupled: the flag completes it)
        dv.dv_scatter(ctx, run, (0, nL, 0, b, q, q + 1), out_ep, (t % 64) * step_b, flag_slot=0, seq=seq[0],
                      xfer=dv.DV_XFER_DECOUPLED, stream=sp)
        # (d) swap-in of x+1's whole prefix into the freed slot (Q10: ordered after the swap-out on
        # the stream; the decoupled DMA reads staging, not the slot)
        ep = eps[t % 2]
        dv.dv_gather(ctx, ep, 0, free, (0, nL, 0, b, 0, P0), stream=sp)
        dv.dv_gather_chunks(ctx, ep, P0 * step_b, free, (0, nL, 0, b, P0, P0 + 1), I - P0, 1, stream=sp)

    steps = min(args.steps, 20)
    for t in range(args.warmup):
        step(t)
    dv.dv_wait(ctx, out_ep, 0, seq[0], stream=sp)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for t in range(args.warmup, args.warmup + steps):
        step(t)
    dv.dv_wait(ctx, out_ep, 0, seq[0], stream=sp)
    e.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(e)
    if world > 1:
        t_ = torch.tensor([ms], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        ms = float(t_.item())
    # parity: the freed slot holds the generator's words on [0, I) (sampled, against kvgen), and
    # every word on the device
    bad = bench.sample_region(free_k, free_v, 0, 0, H, S, D, (0, nL, 0, b, 0, I), SEED)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    dv.dvt_verify(free, cnt.data_ptr(), seed=SEED, reg=dv.region(0, nL, 0, b, 0, I))
    torch.cuda.synchronize()
    bad += int(cnt.item())
    if world > 1:
        b_ = torch.tensor([float(bad)], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(b_, op=dist.ReduceOp.MAX)
        bad = int(b_.item())
    moved = step_b + nb_in
    value = world * steps * moved / (ms * 1e-3) / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": "KV stream GB/s (microbatch swap: step-delta swap-out + prefix swap-in)", "value": value,
            "unit": "GB/s", "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": ms / steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16 (opaque fp16 words)",
            "data": "synthetic (splitmix64 coordinate-hash fill)",
            "config": {"workload": "C4 BLOOM-176B swap, one stage of 9 layers, b4, S2048: swap-out of one step's "
                                   "delta (2.06 MB, decoupled) + swap-in of the i = 2048 prefix (4.23 GB) from "
                                   "the host log form", "bytes_per_step": moved, "parallelism": f"{world} stage(s)"},
            "parity_spot_check": {"mismatches": bad, "how": "20k sampled words vs kvgen + every word on the device"},
            "ideal_ms_per_step_at_64GBps": moved / 64e6}), flush=True)
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
