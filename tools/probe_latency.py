"""Breakdown of the per-layer token-stream latency (SURVEY §8(d) "µs per token-stream per layer"):
%globaltimer stamps relative to the writer's end (dvt_fill of one layer's new position, C2 shape):
resident (first CTA before the PDL wait), past_wait (first CTA past it), stores_issued (last CTA
done issuing its stores), flag (the last CTA's st.release.sys of the seq flag returned).
Prints one JSON line per destination (pinned host, HBM) with p50 of each stamp in µs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
LAYER_BYTES = 2 * B * H * D * 2


def main():
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    cache = dv.cache(k, v)
    ctx = dv.dv_create(0)
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    log = torch.empty(LAYER_BYTES // 2 * L, dtype=torch.int16, pin_memory=True)
    fl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    dlog = torch.empty(LAYER_BYTES // 2 * L, dtype=torch.int16, device="cuda")
    dfl = torch.zeros(1, dtype=torch.int64, device="cuda")
    n = 400
    tag = os.environ.get("TAG", "")
    for name, ep in (("host", dv.endpoint_of(log, fl)), ("hbm", dv.endpoint_of(dlog, dfl))):
        te = torch.zeros(n, dtype=torch.int64, device="cuda")
        ts = torch.zeros((n, 4), dtype=torch.int64, device="cuda")
        ts[:, 1:3] = 2 ** 63 - 1
        for i in range(2 * L):   # warm: first-use costs must not eat the head start below
            reg = dv.region(i % L, i % L + 1, 0, B, P, P + 1)
            dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=20240305, reg=reg, stream=sp, t_end_ptr=te[0].data_ptr())
            dv.dv_scatter(ctx, cache, reg, ep, (i % L) * LAYER_BYTES, flag_slot=0, seq=10 ** 7 + i,
                          xfer=dv.DV_XFER_FUSED, stream=sp)
        torch.cuda.synchronize()
        dv.dvt_spin(20_000_000, 1, stream=sp)
        for i in range(n):
            q = P + 1 + i // L
            layer = i % L
            reg = dv.region(layer, layer + 1, 0, B, q, q + 1)
            dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=20240305, reg=reg, stream=sp, t_end_ptr=te[i].data_ptr())
            dv.dvt_trace(ctx, ts[i].data_ptr())
            dv.dv_scatter(ctx, cache, reg, ep, layer * LAYER_BYTES, flag_slot=0, seq=10 ** 8 + i,
                          xfer=dv.DV_XFER_FUSED, stream=sp)
        dv.dvt_trace(ctx, 0)
        torch.cuda.synchronize()
        rel = ((ts - te[:, None]).double() / 1e3)[L:]
        out = {"dst": name, "tag": tag, "n": rel.shape[0]}
        for j, key in ((1, "resident"), (2, "past_wait"), (3, "stores_issued"), (0, "flag")):
            col = rel[:, j].sort().values
            out[key + "_p50_us"] = round(float(col[len(col) // 2]), 3)
        out["flag_p99_us"] = round(float(rel[:, 0].sort().values[int(len(rel) * 0.99)]), 3)
        print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
