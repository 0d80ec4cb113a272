"""Worker for the multi-process tests (launched by tests/test_multiproc.py, one process per rank).

Modes:
  route  (CPU, gloo): every rank computes the route of a disaggregation hand-off independently with
         dv_route; ranks all-gather what they will send / expect to receive and check agreement.
  ipc    (GPU, all ranks on cuda:0, gloo for plumbing): ranks 0..P-1 are prompt stages, ranks
         P..P+T-1 token stages; token ranks allocate inboxes + flags (dv_device_alloc), export CUDA
         IPC blobs; prompt ranks map them (dv_ipc_open, a real cross-process mapping) and
         dv_stream_out into them; token ranks dv_stream_in; result checked against the oracle.
  direct (GPU): like ipc, but prompt ranks write straight into the token ranks' caches
         (exported torch tensors) with dv_stream_out_direct and a flag in the token rank's memory.
Prints "OK <rank>" on success; raises otherwise.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import kvgen  # noqa: E402
import paper_2403_01876_b200 as dv  # noqa: E402
from oracle import kvstream as ok  # noqa: E402

PSPLIT = [0, 6, 12]
TSPLIT = [0, 5, 9, 12]
PREQ = [0, 4]
TREQ = [0, 2, 4]
H, D, P_LEN, SP, ST, SEED = 3, 16, 9, 12, 20, 77


def blocks(lb, rb):
    return [(i, u) for i in range(len(lb) - 1) for u in range(len(rb) - 1)]


def mode_route(rank, world):
    ps, ts = dv.Setup(PSPLIT, PREQ, SP), dv.Setup(TSPLIT, TREQ, ST)
    reg = dv.region(0, 12, 0, 4, 0, P_LEN)
    pieces = dv.dv_route(ps, ts, reg, H, D, 2)
    def key(p):
        return (p.src_stage, p.src_micro, p.dst_stage, p.dst_micro, p.layer_begin, p.layer_end, p.req_begin,
                p.req_end, p.bytes, p.dst_wire_off)
    # rank r plays every source block and every destination block whose flat index = r mod world
    sends = sorted(key(p) for p in pieces if (p.src_stage * ps.n_micro + p.src_micro) % world == rank)
    recvs = sorted(key(p) for p in pieces if (p.dst_stage * ts.n_micro + p.dst_micro) % world == rank)
    g_s, g_r = [None] * world, [None] * world
    dist.all_gather_object(g_s, sends)
    dist.all_gather_object(g_r, recvs)
    all_s = sorted(x for s in g_s for x in s)
    all_r = sorted(x for r in g_r for x in r)
    assert all_s == all_r, "sender and receiver ranks disagree on the pieces"
    exp = ok.route(ok.Setup(PSPLIT, PREQ, SP), ok.Setup(TSPLIT, TREQ, ST), (0, 12, 0, 4, 0, P_LEN), H, D, 2)
    assert len(all_s) == len(exp)
    tot = sum(x[8] for x in all_s)
    assert tot == ok.region_bytes(0, 12, 0, 4, 0, P_LEN, H, D, 2)


def _device(rank):
    """cuda:0 for every rank (the one-GPU test box), or rank % device_count with DV_MP_CROSS=1 (a
    multi-GPU box: the same IPC mappings then cross NVLink)."""
    if os.environ.get("DV_MP_CROSS") == "1":
        return rank % torch.cuda.device_count()
    return 0


def mode_ipc(rank, world, direct):
    dev = _device(rank)
    torch.cuda.set_device(dev)
    ctx = dv.dv_create(dev)
    pb, tb = blocks(PSPLIT, PREQ), blocks(TSPLIT, TREQ)
    assert world == len(pb) + len(tb)
    ps, ts = dv.Setup(PSPLIT, PREQ, SP), dv.Setup(TSPLIT, TREQ, ST)
    reg = dv.region(0, 12, 0, 4, 0, P_LEN)
    n_src = len(pb)
    mine = {}
    info = None
    if rank >= n_src:                                       # token block
        j, w = tb[rank - n_src]
        a, b_, c0, c1 = TSPLIT[j], TSPLIT[j + 1], TREQ[w], TREQ[w + 1]
        k = torch.full((b_ - a, c1 - c0, H, ST, D), -1, dtype=torch.int16, device="cuda")
        v = torch.full_like(k, -1)
        mine = {"k": k, "v": v, "cache": dv.cache(k, v, a, c0)}
        words = (b_ - a) * (c1 - c0) * H * P_LEN * D * 2
        inbox = dv.dv_device_alloc(dev, words * 2)
        flagp = dv.dv_device_alloc(dev, 8 * n_src)
        fz = torch.zeros(n_src, dtype=torch.int64, device="cuda")
        dv.dv_flush(ctx, fz.data_ptr(), 8 * n_src, dv.endpoint(dv.DV_EP_DEVICE, flagp, 8 * n_src, device=dev), 0,
                    xfer=dv.DV_XFER_STAGED)
        torch.cuda.synchronize()
        info = {"inbox": dv.dv_ipc_export(inbox), "flags": dv.dv_ipc_export(flagp), "words": words,
                "k": dv.dv_ipc_export(k.data_ptr()), "v": dv.dv_ipc_export(v.data_ptr()),
                "shape": (b_ - a, c1 - c0, a, c0), "block": (j, w), "dev": dev}
        mine.update(inbox=inbox, flagp=flagp, words=words)
    infos = [None] * world
    dist.all_gather_object(infos, info)
    if rank < n_src:                                        # prompt block: send
        i, u = pb[rank]
        a, b_, c0, c1 = PSPLIT[i], PSPLIT[i + 1], PREQ[u], PREQ[u + 1]
        K, V = kvgen.kv5d_cache("hash", a, b_ - a, c0, c1 - c0, H, SP, D, seed=SEED, valid_pos=(0, P_LEN))
        k = torch.from_numpy(K.view(np.int16)).cuda()
        v = torch.from_numpy(V.view(np.int16)).cuda()
        src = dv.cache(k, v, a, c0)
        eps, caches, sigs, opened = [], [], [], []
        for r in range(n_src, world):
            inf = infos[r]
            ib = dv.dv_ipc_open(inf["inbox"])
            fp = dv.dv_ipc_open(inf["flags"])
            opened += [ib, fp]
            # memory mapped from another process is never "this GPU's own HBM": system-scope release
            assert not dv.dvt_release_scope(ctx, fp, ib) and not dv.dvt_release_scope(ctx, fp + 8, ib + 64)
            eps.append(dv.endpoint(dv.DV_EP_PEER, ib, inf["words"] * 2, fp, n_src, device=inf["dev"]))
            sigs.append(dv.endpoint(dv.DV_EP_PEER, fp, 8, fp, n_src, device=inf["dev"]))
            if direct:
                kp, vp = dv.dv_ipc_open(inf["k"]), dv.dv_ipc_open(inf["v"])
                opened += [kp, vp]
                nl, nr, la, ra = inf["shape"]
                caches.append(dv.cache_raw(kp, vp, inf["dev"], 2, la, nl, ra, nr, H, ST, D))
        if direct:
            dv.dv_stream_out_direct(ctx, src, reg, ps, i, u, ts, caches, sigs, seq=5)
        else:
            dv.dv_stream_out(ctx, src, reg, ps, i, u, ts, eps, seq=5)
        torch.cuda.synchronize()
        dist.barrier()
        for p_ in opened:
            dv.dv_ipc_close(p_)
        dist.barrier()   # every mapping closed before the exporters free their memory
    else:                                                   # token block: receive
        j, w = tb[rank - n_src]
        iep = dv.endpoint(dv.DV_EP_DEVICE, mine["inbox"], mine["words"] * 2, mine["flagp"], n_src, device=dev)
        assert dv.dvt_release_scope(ctx, mine["flagp"], mine["inbox"])   # own allocation: gpu scope
        if direct:
            # wait for every source block that routes to us, then the bytes are already in place
            for pc in dv.dv_route(ps, ts, reg, H, D, 2):
                if (pc.dst_stage, pc.dst_micro) == (j, w):
                    dv.dv_wait(ctx, iep, pc.src_stage * ps.n_micro + pc.src_micro, 5)
        else:
            dv.dv_stream_in(ctx, mine["cache"], reg, ps, ts, j, w, iep, 5)
        torch.cuda.synchronize()
        dist.barrier()
        # oracle: the single-machine logical KV of this block (definition, north_star / PAPER.md:266)
        a, c0 = TSPLIT[j], TREQ[w]
        nl, nr = TSPLIT[j + 1] - a, TREQ[w + 1] - c0
        exp = kvgen.kv5d_cache("hash", a, nl, c0, nr, H, ST, D, seed=SEED)
        gk = mine["k"].cpu().numpy().view(np.uint16)
        gv = mine["v"].cpu().numpy().view(np.uint16)
        assert np.array_equal(gk[:, :, :, :P_LEN], exp[0][:, :, :, :P_LEN]), f"rank {rank} K mismatch"
        assert np.array_equal(gv[:, :, :, :P_LEN], exp[1][:, :, :, :P_LEN]), f"rank {rank} V mismatch"
        assert np.all(gk[:, :, :, P_LEN:] == kvgen.SENTINEL)
        dist.barrier()
        dv.dv_device_free(mine["inbox"])
        dv.dv_device_free(mine["flagp"])
    ctx.close()


def mode_ring(rank, world, n=300):
    """Rank 1 (receiver) owns a 2-slot ring inbox + flags + credits (dv_device_alloc, exported over
    CUDA IPC); rank 0 (sender) maps them and streams n token chunks with seq 1..n. The sender's
    credit waits poll IPC-mapped memory (the acquire-spin kernel path), its DV_NOWAIT call for seq 3
    before the receiver has started returns DV_EBUSY; the receiver's cache equals kvgen's words."""
    dev = _device(rank)
    torch.cuda.set_device(dev)
    ctx = dv.dv_create(dev)
    L, B, Hh, S, Dd, p = 3, 2, 4, 8 + n, 16, 4
    chunk = 2 * L * B * Hh * Dd * 2
    info = None
    if rank == 1:
        inbox = dv.dv_device_alloc(dev, 2 * chunk)
        fc = dv.dv_device_alloc(dev, 16)          # flag word, then credit word
        z = torch.zeros(2, dtype=torch.int64, device="cuda")
        dv.dv_flush(ctx, z.data_ptr(), 16, dv.endpoint(dv.DV_EP_DEVICE, fc, 16, device=dev), 0, xfer=dv.DV_XFER_STAGED)
        torch.cuda.synchronize()
        info = {"inbox": dv.dv_ipc_export(inbox), "fc": dv.dv_ipc_export(fc), "dev": dev}
    infos = [None] * world
    dist.all_gather_object(infos, info)
    seed = 321
    if rank == 0:
        K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, Hh, S, Dd, seed=seed)
        k = torch.from_numpy(K.view(np.int16)).cuda()
        v = torch.from_numpy(V.view(np.int16)).cuda()
        src = dv.cache(k, v)
        ib, fc = dv.dv_ipc_open(infos[1]["inbox"]), dv.dv_ipc_open(infos[1]["fc"])
        assert dv.dv_ipc_blob_bytes(infos[1]["inbox"]) >= 2 * chunk
        ep = dv.endpoint(dv.DV_EP_PEER, ib, 2 * chunk, fc, 1, device=infos[1]["dev"], n_slots=2, slot_bytes=chunk,
                         credits_ptr=fc + 8)
        regs = [dv.region(0, L, 0, B, p + t - 1, p + t) for t in range(1, n + 1)]
        nw = dv.DV_XFER_FUSED | dv.DV_NOWAIT
        dv.dv_scatter(ctx, src, regs[0], ep, 0, flag_slot=0, seq=1, xfer=nw)
        dv.dv_scatter(ctx, src, regs[1], ep, 0, flag_slot=0, seq=2, xfer=nw)
        try:
            dv.dv_scatter(ctx, src, regs[2], ep, 0, flag_slot=0, seq=3, xfer=nw)
            raise AssertionError("expected DV_EBUSY: the receiver has not consumed seq 1")
        except dv.DVError as e:
            assert e.status == dv.DV_EBUSY, e
        dist.barrier()                             # receiver starts consuming
        for t in range(3, n + 1):                  # blocking: credit waits on IPC-mapped memory
            dv.dv_scatter(ctx, src, regs[t - 1], ep, 0, flag_slot=0, seq=t)
        torch.cuda.synchronize()
        dist.barrier()
        dv.dv_ipc_close(ib)
        dv.dv_ipc_close(fc)
        dist.barrier()
    else:
        dk = torch.full((L, B, Hh, S, Dd), -1, dtype=torch.int16, device="cuda")
        dvv = torch.full_like(dk, -1)
        dst = dv.cache(dk, dvv)
        fcp = dv.dv_ipc_open(info["fc"])           # own allocation: maps to itself
        ibp = dv.dv_ipc_open(info["inbox"])
        ep = dv.endpoint(dv.DV_EP_DEVICE, ibp, 2 * chunk, fcp, 1, device=dev, n_slots=2, slot_bytes=chunk,
                         credits_ptr=fcp + 8)
        dist.barrier()
        for t in range(1, n + 1):
            if t % 50 == 0:
                dv.dvt_spin(300_000, 1)            # a slow receiver now and then
            dv.dv_gather(ctx, ep, 0, dst, dv.region(0, L, 0, B, p + t - 1, p + t), flag_slot=0, wait_seq=t)
        torch.cuda.synchronize()
        dist.barrier()
        K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, Hh, S, Dd, seed=seed)
        gk, gv = dk.cpu().numpy().view(np.uint16), dvv.cpu().numpy().view(np.uint16)
        assert np.array_equal(gk[:, :, :, p:p + n], K[:, :, :, p:p + n]), "K mismatch"
        assert np.array_equal(gv[:, :, :, p:p + n], V[:, :, :, p:p + n]), "V mismatch"
        assert np.all(gk[:, :, :, :p] == kvgen.SENTINEL) and np.all(gk[:, :, :, p + n:] == kvgen.SENTINEL)
        dist.barrier()
        dv.dv_device_free(ibp)
        dv.dv_device_free(fcp)
    ctx.close()


def main():
    mode = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if mode == "route":
        mode_route(rank, world)
    elif mode == "ring":
        mode_ring(rank, world)
    else:
        mode_ipc(rank, world, direct=(mode == "direct"))
    dist.barrier()
    dist.destroy_process_group()
    print(f"OK {rank}", flush=True)


if __name__ == "__main__":
    main()
