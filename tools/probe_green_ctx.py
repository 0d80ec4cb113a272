"""Latency isolation by SM partitioning (green contexts): the per-layer token stream-out (C2 layer,
160 KiB, writer end -> flag) while a bf16 GEMM loop saturates the GPU, in three arrangements:

  priority   GEMM on a low-priority stream, writer + stream-out on a high-priority stream (all SMs
             shared; the round-2 default recommendation, NEXT-2);
  green      GEMM in a green context of the remaining SMs, writer + stream-out in a green context
             of 8 SMs (the minimum partition on sm_90+): the copy's CTAs never wait for GEMM CTAs
             to retire;
  green_copy GEMM on an ordinary stream (all SMs), stream-out in the 8-SM green context.

Also the price of the partition for the model's own work: the GEMM loop's TFLOP/s and an
HBM-bound step (a 2 GiB device copy) in the big green context vs on all SMs. One JSON line per
measurement. DST=host (default) or DST=hbm selects the destination."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from cuda.bindings import driver as cu  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if int(err) != 0:
        raise RuntimeError(f"CUDA driver error {err}")
    return r[1:] if isinstance(r, tuple) and len(r) > 2 else (r[1] if isinstance(r, tuple) and len(r) == 2 else None)


torch.cuda.init()
torch.empty(1, device="cuda")
ck(cu.cuInit(0))
dev = ck(cu.cuDeviceGet(0))
SMALL_SMS = int(os.environ.get("GREEN_SMS", "8"))
res = ck(cu.cuDeviceGetDevResource(dev, cu.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
SPLIT_FLAGS = int(os.environ.get("SPLIT_FLAGS", "0"))   # cuDevSmResourceSplitByCount useFlags (1 ignore co-scheduling, 2 max cluster)
groups, nb, rest = ck(cu.cuDevSmResourceSplitByCount(1, res, SPLIT_FLAGS, SMALL_SMS))
d_small = ck(cu.cuDevResourceGenerateDesc([groups[0]], 1))
d_big = ck(cu.cuDevResourceGenerateDesc([rest], 1))
flag = cu.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM
g_small = ck(cu.cuGreenCtxCreate(d_small, dev, flag))
g_big = ck(cu.cuGreenCtxCreate(d_big, dev, flag))
lo_pr, hi_pr = torch.cuda.Stream.priority_range()
NB = cu.CUstream_flags.CU_STREAM_NON_BLOCKING
s_small = torch.cuda.ExternalStream(int(ck(cu.cuGreenCtxStreamCreate(g_small, NB, hi_pr))))
s_big = torch.cuda.ExternalStream(int(ck(cu.cuGreenCtxStreamCreate(g_big, NB, 0))))
print(json.dumps({"sms_small": groups[0].sm.smCount, "sms_big": rest.sm.smCount, "split_flags": SPLIT_FLAGS}),
      flush=True)

L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
LAYER = 2 * B * H * D * 2
k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
cache = dv.cache(k, v)
ctx = dv.dv_create(0)
HOST = os.environ.get("DST", "host") == "host"
dlog = torch.empty(LAYER // 2 * L, dtype=torch.int16, device="cpu" if HOST else "cuda", pin_memory=HOST)
dfl = torch.zeros(1, dtype=torch.int64, device="cpu" if HOST else "cuda", pin_memory=HOST)
ep = dv.endpoint_of(dlog, dfl)
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
bm = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
big_src = torch.empty(1 << 30, dtype=torch.int16, device="cuda")
big_dst = torch.empty_like(big_src)
seqc = [10 ** 9]
N_GEMM = 60


def gemm_loop(stream, n=N_GEMM):
    with torch.cuda.stream(stream):
        for _ in range(n):
            torch.matmul(a, bm)


def timed(stream, fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def latency(copy_stream, gemm_stream, loaded, n=400):
    sp = copy_stream.cuda_stream
    for i in range(2 * L):   # warm the kernels on this stream
        reg = (i % L, i % L + 1, 0, B, P, P + 1)
        dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=1, reg=reg, stream=sp)
        seqc[0] += 1
        dv.dv_scatter(ctx, cache, reg, ep, (i % L) * LAYER, flag_slot=0, seq=seqc[0], stream=sp)
    te = torch.zeros(n, dtype=torch.int64, device="cuda")
    ts = torch.zeros((n, 4), dtype=torch.int64, device="cuda")
    ts[:, 1:3] = 2 ** 63 - 1
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if loaded:
        e0.record(gemm_stream)
        gemm_loop(gemm_stream)
        e1.record(gemm_stream)
    dv.dvt_spin(20_000_000, 1, stream=sp)
    for i in range(n):
        layer = i % L
        q = P + 1 + i // L
        reg = (layer, layer + 1, 0, B, q, q + 1)
        dv.dvt_fill(cache, dv.DVT_FILL_HASH, seed=1, reg=reg, stream=sp, t_end_ptr=te[i].data_ptr())
        dv.dvt_trace(ctx, ts[i].data_ptr())
        seqc[0] += 1
        dv.dv_scatter(ctx, cache, reg, ep, layer * LAYER, flag_slot=0, seq=seqc[0], stream=sp)
    dv.dvt_trace(ctx, 0)
    torch.cuda.synchronize()
    d = sorted(((ts[:, 0] - te).double() / 1e3).tolist()[L:])
    out = {"p50_us": round(d[len(d) // 2], 3), "p99_us": round(d[int(len(d) * 0.99)], 3), "n": len(d)}
    if loaded:
        out["gemm_tflops_during"] = round(N_GEMM * 2 * 8192 ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12, 1)
    return out


plain_lo = torch.cuda.Stream(priority=lo_pr)
plain_hi = torch.cuda.Stream(priority=hi_pr)
gemm_loop(plain_lo, 3)
gemm_loop(s_big, 3)
torch.cuda.synchronize()
def _copy(st):
    with torch.cuda.stream(st):
        for _ in range(10):
            big_dst.copy_(big_src)


import ctypes  # noqa: E402
_cublas = ctypes.CDLL("libcublas.so.12")


def sm_target(st, n):
    """cublasSetSmCountTarget on torch's cuBLAS handle for stream st (0 = the device's count)."""
    with torch.cuda.stream(st):
        h = torch.cuda.current_blas_handle()
        assert _cublas.cublasSetSmCountTarget(ctypes.c_void_p(h), ctypes.c_int(n)) == 0


for rep in range(2):
    for name, st, tgt in (("all_sms", plain_lo, 0), ("green_big", s_big, 0),
                          ("green_big_cublas_sm_target", s_big, rest.sm.smCount)):
        sm_target(st, tgt)
        ms = timed(st, lambda st=st: gemm_loop(st))
        ms_copy = timed(st, lambda st=st: _copy(st))
        print(json.dumps({"rep": rep, "compute_on": name,
                          "gemm_tflops": round(N_GEMM * 2 * 8192 ** 3 / (ms * 1e-3) / 1e12, 1),
                          "hbm_copy_gbs_2R": round(10 * 2 * big_src.numel() * 2 / (ms_copy * 1e-3) / 1e9, 1)}),
              flush=True)
        sm_target(st, 0)
    if os.environ.get("GEMM_ONLY"):
        continue
    for mode, cs, gs in (("priority", plain_hi, plain_lo), ("green", s_small, s_big), ("green_copy", s_small, plain_lo)):
        for loaded in (False, True):
            r = latency(cs, gs, loaded)
            print(json.dumps({"rep": rep, "dst": "host" if HOST else "hbm", "mode": mode, "loaded": loaded, **r}),
                  flush=True)
