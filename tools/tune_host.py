"""Kernel-shape / transfer-mode sweep for the C2 host path (run under gpurun).

  python tools/tune_host.py            # spawns one child per variant (env DV_U / DV_VEC)
  python tools/tune_host.py --child    # one measurement set with the current env

Writes one JSON line per variant to stdout.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
STEP = 2 * L * B * H * D * 2
LAYER = STEP // L


def child():
    import torch
    import paper_2403_01876_b200 as dv
    ctx = dv.dv_create(0)
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    c = dv.cache(k, v)
    dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=1)
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    log = torch.empty(STEP * 8 // 2, dtype=torch.int16, pin_memory=True)
    fl = torch.zeros(2, dtype=torch.int64, pin_memory=True)
    dbuf = torch.empty(STEP * 8 // 2, dtype=torch.int16, device="cuda")
    dfl = torch.zeros(2, dtype=torch.int64, device="cuda")
    out = {"env": {k_: os.environ.get(k_) for k_ in ("DV_U", "DV_VEC", "DV_PDL", "DV_BULK", "DV_STM")}}
    cnt = [0]

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def loop(fn, n, per_event=False):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        evs = []
        a.record(st)
        for _ in range(n):
            if per_event:
                e0, e1 = ev(), ev()
                e0.record(st)
                fn()
                e1.record(st)
                evs.append((e0, e1))
            else:
                fn()
        b.record(st)
        torch.cuda.synchronize()
        tot = a.elapsed_time(b) / n * 1e3
        if per_event:
            ks = sorted(x.elapsed_time(y) * 1e3 for x, y in evs)
            return tot, ks[len(ks) // 2]
        return tot

    def tok(buf, flg, xf, layer=None):
        ep = dv.endpoint_of(buf, flg)

        def f():
            cnt[0] += 1
            q = P + cnt[0] % 1000
            if layer is None:
                reg = dv.region(0, L, 0, B, q, q + 1)
                off = (cnt[0] % 8) * STEP
            else:
                lay = cnt[0] % L
                reg = dv.region(lay, lay + 1, 0, B, q, q + 1)
                off = lay * LAYER
            dv.dv_scatter(ctx, c, reg, ep, off, flag_slot=0 if flg is not None else -1, seq=cnt[0],
                          xfer=xf, stream=sp)
        return f

    F, G = dv.DV_XFER_FUSED, dv.DV_XFER_STAGED
    if os.environ.get("DV_SWEEP_CTAS"):
        pb = torch.empty(LAYER * P // 2, dtype=torch.int16, pin_memory=True)
        pep = dv.endpoint_of(pb)
        for mc in (8, 16, 32, 64, 148, 296, 1184):
            cx = dv.dv_create(0, max_ctas=mc)
            def f(cx=cx):
                cnt[0] += 1
                q = P + cnt[0] % 1000
                dv.dv_scatter(cx, c, dv.region(0, L, 0, B, q, q + 1), dv.endpoint_of(log, fl), (cnt[0] % 8) * STEP,
                              flag_slot=0, seq=cnt[0], xfer=F, stream=sp)
            out[f"ctas{mc}_step_host_us"] = loop(f, 200)
            def g(cx=cx):
                cnt[0] += 1
                l_ = cnt[0] % L
                dv.dv_scatter(cx, c, dv.region(l_, l_ + 1, 0, B, 0, P), pep, 0, xfer=F, stream=sp)
            out[f"ctas{mc}_prompt_host_gbs"] = LAYER * P / loop(g, 5) / 1e3
            def h(cx=cx):
                cnt[0] += 1
                q = P + cnt[0] % 1000
                dv.dv_gather(cx, dv.endpoint_of(log, fl), (cnt[0] % 8) * STEP, c, dv.region(0, L, 0, B, q, q + 1),
                             xfer=F, stream=sp)
            out[f"ctas{mc}_gather_host_fused_us"] = loop(h, 200)
            cx.close()
        print(json.dumps(out), flush=True)
        return
    out["step_host_fused_noflag_us"] = loop(tok(log, None, F), 300)
    out["step_host_fused_flag_us"] = loop(tok(log, fl, F), 300)
    out["step_host_fused_flag_events_us"] = loop(tok(log, fl, F), 300, per_event=True)
    out["step_host_staged_flag_us"] = loop(tok(log, fl, G), 300)
    out["step_host_fused_streamop_us"] = loop(tok(log, fl, F | dv.DV_PUBLISH_STREAMOP), 300)
    out["step_hbm_flag_us"] = loop(tok(dbuf, dfl, F), 300)
    out["step_hbm_noflag_us"] = loop(tok(dbuf, None, F), 300)
    out["layer_host_fused_flag_us"] = loop(tok(log, fl, F, layer=True), 400, per_event=True)
    out["layer_host_fused_noflag_us"] = loop(tok(log, None, F, layer=True), 400, per_event=True)
    out["layer_hbm_flag_us"] = loop(tok(dbuf, dfl, F, layer=True), 400, per_event=True)
    out["layer_host_staged_flag_us"] = loop(tok(log, fl, G, layer=True), 400, per_event=True)
    out["empty_spin_us"] = loop(lambda: dv.dvt_spin(0, 1, stream=sp), 400, per_event=True)

    # writer -> flag latency with %globaltimer (no event between writer and stream-out: PDL works)
    def gt_lat(buf, flg, xf, n=400):
        ep = dv.endpoint_of(buf, flg)
        te = torch.zeros(n, dtype=torch.int64, device="cuda")
        ts = torch.zeros((n, 4), dtype=torch.int64, device="cuda")
        ts[:, 1:3] = 2 ** 63 - 1
        dv.dvt_spin(20_000_000, 1, stream=sp)   # head start: GPU runs behind the host
        for i in range(n):
            q = P + i % 1000
            lay = i % L
            reg = dv.region(lay, lay + 1, 0, B, q, q + 1)
            dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=1, reg=reg, stream=sp, t_end_ptr=te[i].data_ptr())
            dv.dvt_trace(ctx, ts[i].data_ptr())
            dv.dv_scatter(ctx, c, reg, ep, lay * LAYER, flag_slot=0, seq=10 ** 6 + i, xfer=xf, stream=sp)
        dv.dvt_trace(ctx, 0)
        torch.cuda.synchronize()
        res = {}
        for nm, col in (("flag", 0), ("resident", 1), ("past_wait", 2), ("stores_issued", 3)):
            d = sorted(((ts[:, col] - te).double() / 1e3).tolist()[20:])
            res[nm + "_p50"] = d[len(d) // 2]
            if col == 0:
                res["flag_p99"] = d[int(len(d) * 0.99)]
                res["flag_min"] = d[0]
        return res
    out["gt_layer_host_fused"] = gt_lat(log, fl, F)
    out["gt_layer_hbm_fused"] = gt_lat(dbuf, dfl, F)
    tres = torch.zeros(64, dtype=torch.int64, device="cuda")
    for i in range(64):
        dv.dvt_fill(c, dv.DVT_FILL_HASH, seed=1, reg=dv.region(0, 1, 0, 1, 5, 6), stream=sp, t_end_ptr=tres[i].data_ptr())
    torch.cuda.synchronize()
    out["globaltimer_samples_ns"] = sorted(set((tres % 1000).tolist()))[:16]
    # e2e: H2D of the token's K/V (side stream) -> cache, then stream-out (main stream)
    s_in = torch.cuda.Stream()
    dl = torch.empty(STEP * 8 // 2, dtype=torch.int16, pin_memory=True)
    dep_ = dv.endpoint_of(dl)
    evs = [torch.cuda.Event() for _ in range(8)]
    lep = dv.endpoint_of(log, fl)

    def e2e(gx, sx, n=200):
        def one(t):
            q = P + t % 1000
            dv.dv_gather(ctx, dep_, (t % 8) * STEP, c, dv.region(0, L, 0, B, q, q + 1), xfer=gx, stream=s_in)
            e = evs[t % 8]
            e.record(s_in)
            st.wait_event(e)
            dv.dv_scatter(ctx, c, dv.region(0, L, 0, B, q, q + 1), lep, (t % 8) * STEP, flag_slot=0, seq=t,
                          xfer=sx, stream=sp)
        for t in range(5):
            one(t)
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(st)
        s_in.wait_event(a)
        for t in range(n):
            one(t)
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e3
    for gn, gx in (("fused", F), ("staged", G)):
        for sn, sx in (("fused", F), ("staged", G)):
            out[f"e2e_gather_{gn}_scatter_{sn}_us"] = e2e(gx, sx)

    # prompt layer 163.8 MB
    pb = torch.empty(LAYER * P // 2, dtype=torch.int16, pin_memory=True)
    pd = torch.empty(LAYER * P // 2, dtype=torch.int16, device="cuda")
    lay = [0]

    def prm(buf, xf):
        ep = dv.endpoint_of(buf)

        def f():
            lay[0] = (lay[0] + 1) % L
            dv.dv_scatter(ctx, c, dv.region(lay[0], lay[0] + 1, 0, B, 0, P), ep, 0, xfer=xf, stream=sp)
        return f
    t = loop(prm(pb, F), 5)
    out["prompt_host_fused_gbs"] = LAYER * P / t / 1e3
    t = loop(prm(pb, G), 5)
    out["prompt_host_staged_gbs"] = LAYER * P / t / 1e3
    t = loop(prm(pd, F), 10)
    out["prompt_hbm_gbs_2R"] = 2 * LAYER * P / t / 1e3
    print(json.dumps(out), flush=True)


def main():
    variants = [{}, {"DV_STM": "1"}, {"DV_STM": "2"}, {"DV_VEC": "16"}, {"DV_VEC": "16", "DV_STM": "2"},
                {"DV_U": "8"}, {"DV_U": "2"}]
    for var in variants:
        env = dict(os.environ)
        env.update(var)
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True,
                           timeout=600)
        sys.stdout.write(r.stdout)
        if r.returncode:
            sys.stdout.write(json.dumps({"env": var, "error": r.stderr[-2000:]}) + "\n")
        sys.stdout.flush()


if __name__ == "__main__":
    if "--child" in sys.argv:
        child()
    else:
        main()
