"""Soak of the credited ring with a HOST consumer: the GPU streams C2 token-layer chunks (160 KiB:
one layer, one position, b 8) into a 4-slot pinned-host ring whose credits are pinned host words;
a host thread checks every chunk word by word against the generator's precomputed words the
moment its flag appears, then releases the credit. Prints one JSON line.
  python tools/soak_ring.py --chunks 200000"""
import argparse
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402

L, H, D, B, S = 40, 40, 128, 8, 2048


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", type=int, default=200000)
    ap.add_argument("--slots", type=int, default=4)
    args = ap.parse_args()
    n, R = args.chunks, args.slots
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    c = dv.cache(k, v)
    seed = 99
    dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=seed)
    ctx = dv.dv_create(0)
    chunk = 2 * B * H * D * 2
    # the generator's words of the 64 (layer, position) chunks the soak cycles through, packed on
    # the device once and verified there (dvt_verify) before they serve as the expected words
    NE = 64
    expd = torch.empty(NE * chunk // 2, dtype=torch.int16, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for e in range(NE):
        lay, q = e % L, 1000 + e
        reg = dv.region(lay, lay + 1, 0, B, q, q + 1)
        w = expd[e * chunk // 2:(e + 1) * chunk // 2]
        dv.dv_scatter(ctx, c, reg, dv.endpoint_of(w), 0)
        dv.dvt_verify(c, cnt.data_ptr(), seed=seed, reg=reg, wire_ptr=w.data_ptr())
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    exp = expd.cpu().numpy().view(np.uint16).reshape(NE, -1)
    ring = torch.empty(R * chunk // 2, dtype=torch.int16, pin_memory=True)
    fl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    cr = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    ep = dv.endpoint_of(ring, fl, n_slots=R, slot_bytes=chunk, credits=cr)
    view = ring.numpy().view(np.uint16)
    flv, crv = fl.numpy(), cr.numpy()
    bad = [0]
    done = [0]

    def consumer():
        for s_ in range(1, n + 1):
            while flv[0] < s_:
                pass
            o = (s_ % R) * chunk // 2
            if not np.array_equal(view[o:o + chunk // 2], exp[(s_ - 1) % NE]):
                bad[0] += 1
            crv[0] = s_
            done[0] = s_
    sys.setswitchinterval(0.0002)   # the producer's enqueue and the consumer's poll share the GIL
    th = threading.Thread(target=consumer, daemon=True)
    t0 = time.time()
    th.start()
    st = torch.cuda.Stream()
    for s_ in range(1, n + 1):
        e = (s_ - 1) % NE
        lay, q = e % L, 1000 + e
        dv.dv_scatter(ctx, c, (lay, lay + 1, 0, B, q, q + 1), ep, 0, flag_slot=0, seq=s_, stream=st)
    st.synchronize()
    th.join(timeout=600)
    dt = time.time() - t0
    print(json.dumps({"soak": "credited ring, host consumer", "chunks": n, "slots": R, "chunk_bytes": chunk,
                      "bytes": n * chunk, "mismatched_chunks": bad[0], "consumed": done[0], "flag": int(fl[0]),
                      "credit": int(cr[0]), "wall_s": round(dt, 2),
                      "chunks_per_s": round(n / dt, 1)}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
