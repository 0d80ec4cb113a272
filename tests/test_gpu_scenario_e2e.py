"""End-to-end DéjàVu scenario on one GPU, every block a separate cache (loopback peers), all three
use cases of the paper in one run (§4.2):

  1. prompt pipeline, 2 stages [0,4) [4,8), computes the prompt layer by layer; after each layer it
     streams that layer straight into the token pipeline (Opt 2; §4.2.1 hand-off),
     whose partition differs: 3 stages [0,3) [3,6) [6,8) and 2 microbatches of 2 requests (split);
  2. token generation: every step each token block writes its new position, replicates the step
     to its ring successor (§4.2.3) and swaps the step's delta out to its host log
     (§4.2.2 swap-out of the step's update);
  3. at step F token stage 1 fails: its cache and the replica it hosts are wiped; recovery copies
     the replica from stage 2 and the predecessor's cache from stage 0; generation
     resumes; and a swapped-out microbatch is swapped back in from its host log.
Expected final state: every cache (own caches, replicas, swapped-in slot) equals kvgen's writer
definition on [0, p+T) and the sentinel beyond -- the single-machine KV (north_star).
"""
import numpy as np
import pytest
import torch

import kvgen
import paper_2403_01876_b200 as dv

pytestmark = pytest.mark.gpu

H, D, S = 4, 64, 48
P, T, F = 10, 12, 5
SEED = 20240377
PB, TB, RB = [0, 4, 8], [0, 3, 6, 8], [0, 2, 4]


def new(nl, nr, lb, rb, fill=False):
    k = torch.full((nl, nr, H, S, D), -1, dtype=torch.int16, device="cuda")
    v = torch.full_like(k, -1)
    c = dv.cache(k, v, lb, rb)
    return k, v, c


def write(c, l0, l1, r0, r1, s0, s1):
    """The synthetic model writes its K/V (dvt_fill = kvgen's generator on the device)."""
    dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=SEED, reg=dv.region(l0, l1, r0, r1, s0, s1))


def expect(k, v, lb, rb, n):
    nl, nr = k.shape[0], k.shape[1]
    K, V = kvgen.kv5d_cache("hash", lb, nl, rb, nr, H, S, D, seed=SEED)
    gk, gv = k.cpu().numpy().view(np.uint16), v.cpu().numpy().view(np.uint16)
    assert np.array_equal(gk[:, :, :, :n], K[:, :, :, :n]) and np.array_equal(gv[:, :, :, :n], V[:, :, :, :n])
    assert np.all(gk[:, :, :, n:] == kvgen.SENTINEL) and np.all(gv[:, :, :, n:] == kvgen.SENTINEL)


def test_dejavu_scenario_on_one_gpu():
    cx = dv.dv_create(0)
    psetup, tsetup = dv.Setup(PB, [0, 4], S), dv.Setup(TB, RB, S)
    prompt = {i: new(PB[i + 1] - PB[i], 4, PB[i], 0) for i in range(2)}
    token = {(j, w): new(TB[j + 1] - TB[j], 2, TB[j], RB[w]) for j in range(3) for w in range(2)}
    keys = sorted(token, key=lambda x: tsetup.flat(*x))
    sig = torch.zeros(16 * 16, dtype=torch.int64, device="cuda")
    sigs = [dv.endpoint_of(sig[:1], sig[16 * n:16 * (n + 1)]) for n in range(len(keys))]
    # ---- 1. prompt pass, layer by layer, each layer streamed to the token pipeline at once
    for i in range(2):
        for layer in range(PB[i], PB[i + 1]):
            write(prompt[i][2], layer, layer + 1, 0, 4, 0, P)
            dv.dv_stream_out_direct(cx, prompt[i][2], dv.region(layer, layer + 1, 0, 4, 0, P), psetup, i, 0, tsetup,
                                    [token[kk][2] for kk in keys], sigs, seq=layer + 1)
    for n, kk in enumerate(keys):  # token blocks wait for every prompt layer that routes to them
        for pc in dv.dv_route(psetup, tsetup, dv.region(0, 8, 0, 4, 0, P), H, D, 2):
            if (pc.dst_stage, pc.dst_micro) == kk:
                dv.dv_wait(cx, sigs[n], psetup.flat(pc.src_stage, pc.src_micro), pc.layer_end)
    # ---- 2. token generation with ring replication and swap-out to host logs
    replica = {(j, w): new(TB[(j - 1) % 3 + 1] - TB[(j - 1) % 3], 2, TB[(j - 1) % 3], RB[w]) for j in range(3)
               for w in range(2)}
    step_bytes = {kk: 2 * token[kk][0].shape[0] * 2 * H * D * 2 for kk in keys}
    logs = {kk: torch.empty((T + P) * step_bytes[kk] // 2, dtype=torch.int16, pin_memory=True) for kk in keys}
    for kk in keys:   # the prompt part of each host log (one chunk of P positions)
        j, w = kk
        dv.dv_scatter(cx, token[kk][2], dv.region(TB[j], TB[j + 1], RB[w], RB[w + 1], 0, P), dv.endpoint_of(logs[kk]), 0)
    for kk in keys:   # prompt replica (Q13)
        j, w = kk
        dv.dv_remap(cx, token[kk][2], replica[((j + 1) % 3, w)][2], dv.region(TB[j], TB[j + 1], RB[w], RB[w + 1], 0, P))

    def token_step(t):
        q = P + t - 1
        for kk in keys:
            j, w = kk
            reg = dv.region(TB[j], TB[j + 1], RB[w], RB[w + 1], q, q + 1)
            write(token[kk][2], TB[j], TB[j + 1], RB[w], RB[w + 1], q, q + 1)
            dv.dv_remap(cx, token[kk][2], replica[((j + 1) % 3, w)][2], reg)                  # replication
            dv.dv_scatter(cx, token[kk][2], reg, dv.endpoint_of(logs[kk]), q * step_bytes[kk],
                          xfer=dv.DV_XFER_FUSED)                                            # swap-out delta
    for t in range(1, F + 1):
        token_step(t)
    # ---- 3. failure of token stage 1 (both microbatches) and recovery
    torch.cuda.synchronize()
    n_done = P + F
    for w in range(2):
        for x in token[(1, w)][:2] + replica[(1, w)][:2]:
            x.fill_(-1)
        dv.dv_remap(cx, replica[(2, w)][2], token[(1, w)][2], dv.region(TB[1], TB[2], RB[w], RB[w + 1], 0, n_done))
        dv.dv_remap(cx, token[(0, w)][2], replica[(1, w)][2], dv.region(TB[0], TB[1], RB[w], RB[w + 1], 0, n_done))
    for t in range(F + 1, T + 1):
        token_step(t)
    torch.cuda.synchronize()
    n = P + T
    for kk in keys:
        j, w = kk
        expect(token[kk][0], token[kk][1], TB[j], RB[w], n)
        pj = (j - 1) % 3
        expect(replica[kk][0], replica[kk][1], TB[pj], RB[w], n)
    # ---- swap-in of microbatch (2, 1) from its host log into an empty slot: prompt chunk + steps
    kk = (2, 1)
    k2, v2, c2 = new(TB[3] - TB[2], 2, TB[2], RB[1])
    ep = dv.endpoint_of(logs[kk])
    dv.dv_gather(cx, ep, 0, c2, dv.region(TB[2], TB[3], RB[1], RB[2], 0, P))
    dv.dv_gather_chunks(cx, ep, P * step_bytes[kk], c2, dv.region(TB[2], TB[3], RB[1], RB[2], P, P + 1), T, 1)
    torch.cuda.synchronize()
    expect(k2, v2, TB[2], RB[1], n)
    cx.close()
