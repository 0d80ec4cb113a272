"""Soak of device plans (include/dv.h dv_dplan_*): the C2 per-layer token stream fused into the
producer for --steps token steps (40 producer launches per step, each storing one layer's new K/V
into the cache and straight into a pinned-host log, releasing that layer's flag), every --check
steps the whole log (40 layers) verified word by word on the device against the generator, and
every flag checked at its seq. Positions wrap inside S; plans are re-made (and the old ones freed)
at each wrap so flags stay monotone. Prints one JSON line."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20000)
ap.add_argument("--check", type=int, default=64)
args = ap.parse_args()

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
LAYER = 2 * B * H * D * 2
SEED = 20240312
k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
cache = dv.cache(k, v)
ctx = dv.dv_create(0)
log = torch.full((L * LAYER // 2,), -1, dtype=torch.int16, pin_memory=True)
fl = torch.zeros(L, dtype=torch.int64, pin_memory=True)
ep = dv.endpoint_of(log, fl)
st = torch.cuda.Stream()
sp = st.cuda_stream
WRAP = S - P
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
plans, base = [], 0
checks = words = 0
t0 = time.time()
for t in range(args.steps):
    kk = t % WRAP
    if kk == 0:   # (re)make the plans: seq base grows with every wrap
        st.synchronize()
        for pl in plans:
            dv.dv_dplan_free(ctx, pl)
        base = 1 + (t // WRAP) * WRAP
        plans = [dv.dv_dplan_scatter(ctx, cache, dv.region(l, l + 1, 0, B, P, P + 1), ep, l * LAYER, 0,
                                     flag_slot=l, seq=base, max_step=WRAP - 1) for l in range(L)]
    q = P + kk
    for l in range(L):
        dv.dvt_fill_rows(cache, SEED, dv.region(l, l + 1, 0, B, q, q + 1), plans[l], kk, stream=sp)
    if (t + 1) % args.check == 0 or t == args.steps - 1:
        st.synchronize()
        assert all(int(fl[l]) == base + kk for l in range(L)), "flag not at its seq"
        dv.dvt_verify(cache, cnt.data_ptr(), seed=SEED, reg=dv.region(0, L, 0, B, q, q + 1),
                      wire_ptr=log.data_ptr(), stream=sp)
        st.synchronize()
        checks += 1
        words += L * LAYER // 2
st.synchronize()
for pl in plans:
    dv.dv_dplan_free(ctx, pl)
print(json.dumps({"soak": "device plans: C2 per-layer token stream fused into the producer -> pinned host",
                  "steps": args.steps, "producer_launches": args.steps * L, "bytes_streamed": args.steps * L * LAYER,
                  "checks": checks, "words_checked": words, "mismatches": int(cnt.item()),
                  "wall_s": round(time.time() - t0, 1)}))
