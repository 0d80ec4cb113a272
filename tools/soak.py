"""Soak run of the headline path: N decoupled C2 token steps to a 64-step pinned host ring, each
with its seq flag; after every 64 steps the consumer waits for the last flag and verifies EVERY
word of the 64 wires on the device against the writer's definition (dvt_verify), before the ring
is overwritten. Prints one JSON line: steps, bytes, mismatches (must be 0), GB/s including the
verification pauses.

  python tools/soak.py [--steps 100000]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
STEP = 2 * L * B * H * D * 2
RING = 64
SEED = 20240399


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100_000)
    ap.add_argument("--mode", default="token-host", choices=["token-host", "layer-hbm"],
                    help="token-host: decoupled token steps to pinned host (ticket / DMA + stream flag); "
                         "layer-hbm: one layer per call into an HBM ring with a gpu-scope release "
                         "(the 16-CTA cluster publish)")
    args = ap.parse_args()
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    cache = dv.cache(k, v)
    dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=SEED)
    ctx = dv.dv_create(0)
    hbm = args.mode == "layer-hbm"
    unit = STEP // L if hbm else STEP
    log = torch.empty(RING * unit // 2, dtype=torch.int16, device="cuda" if hbm else "cpu", pin_memory=not hbm)
    fl = torch.zeros(1, dtype=torch.int64, device="cuda" if hbm else "cpu", pin_memory=not hbm)
    ep = dv.endpoint_of(log, fl)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    pos = lambda t: P + (t - 1) % (S - P)  # noqa: E731
    lay = (lambda t: (t % L, t % L + 1)) if hbm else (lambda t: (0, L))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in range(1, args.steps + 1):
        q = pos(t)
        dv.dv_scatter(ctx, cache, lay(t) + (0, B, q, q + 1), ep, (t % RING) * unit, flag_slot=0, seq=t,
                      xfer=dv.DV_XFER_FUSED if hbm else dv.DV_XFER_DECOUPLED, stream=st)
        if t % RING == 0 or t == args.steps:
            dv.dv_wait(ctx, ep, 0, t, stream=st)            # the consumer: every step of the ring landed
            for tt in range(max(1, t - RING + 1), t + 1):
                w = log[(tt % RING) * unit // 2:(tt % RING + 1) * unit // 2]
                dv.dvt_verify(cache, cnt.data_ptr(), seed=SEED, reg=lay(tt) + (0, B, pos(tt), pos(tt) + 1),
                              wire_ptr=w.data_ptr(), stream=st)
            torch.cuda.current_stream().synchronize()      # the ring may now be overwritten
    dt = time.perf_counter() - t0
    print(json.dumps({"mode": args.mode, "steps": args.steps, "bytes": args.steps * unit,
                      "words_verified": args.steps * unit // 2,
                      "mismatches": int(cnt.item()), "flag": int(fl[0]), "seconds": round(dt, 2),
                      "gbs_incl_verification": round(args.steps * unit / dt / 1e9, 2)}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
