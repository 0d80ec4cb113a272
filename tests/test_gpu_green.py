"""GPU parity of the streaming calls on a stream of a green context (an SM partition: DESIGN.md §6
"SM partitions"). An 8-SM partition cannot hold the 16-CTA cluster of the small gpu-scope publish,
so the library must fall back to the ticket form there instead of failing; every delivered word is
compared with the oracle, and flags are checked. The partition comes from the library's own
dv_partition_create (include/dv.h)."""
import numpy as np
import pytest
import torch

import kvgen
import paper_2403_01876_b200 as dv
from oracle import kvstream as ok

from gpu_util import ctx, flags, sentinel_like, to_dev, to_np

pytestmark = pytest.mark.gpu


_KEEP = []


def test_streaming_on_an_8_sm_green_context_stream():
    """C2-shaped layer (160 KiB: the size that takes the 16-CTA cluster publish into HBM), token
    steps to pinned host and into HBM with flags, a level-1 stream_out, a remap and a prompt-sized
    pack, all on the 8-SM partition's stream; == the oracle, flags at their seqs."""
    part = dv.dv_partition_create(0, 8)
    _KEEP.append(part)
    assert part.sms_streaming >= 8 and part.sms_compute >= 1
    assert part.sms_streaming + part.sms_compute <= torch.cuda.get_device_properties(0).multi_processor_count
    st = torch.cuda.ExternalStream(part.streaming)
    sp = st.cuda_stream
    L, B, H, S, D = 4, 8, 40, 96, 128
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=41)
    k, v = to_dev(K), to_dev(V)
    c = dv.cache(k, v)
    o = ok.Cache(K, V, 0, 0, H, S, D)
    cx = ctx()
    torch.cuda.synchronize()
    for dst_host in (False, True):
        reg = (1, 2, 0, B, 70, 71)               # one layer, one position: 160 KiB
        exp = ok.pack(o, reg)
        buf = sentinel_like((exp.size,), pinned=dst_host)
        fl = flags(1, pinned=dst_host)
        torch.cuda.synchronize()   # buffers made on torch's stream; the partition stream is non-blocking
        dv.dv_scatter(cx, c, dv.region(*reg), dv.endpoint_of(buf, fl), 0, flag_slot=0, seq=7, stream=sp)
        st.synchronize()
        assert np.array_equal(to_np(buf), exp) and int(fl[0]) == 7
    # level 1 into a device inbox, then a remap into another cache and a prompt-sized pack
    setup = dv.Setup([0, L], [0, B], S)
    reg = (0, L, 0, B, 10, 11)
    exp = ok.pack(o, reg)
    inbox = sentinel_like((exp.size,))
    ifl = flags(1)
    Ks, Vs = kvgen.sentinel_cache(L, B, H, S, D)
    dk, dvv = to_dev(Ks), to_dev(Vs)
    dc = dv.cache(dk, dvv)
    do = ok.Cache(Ks.copy(), Vs.copy(), 0, 0, H, S, D)
    rreg = (0, L, 0, B, 0, 64)
    pexp = ok.pack(o, rreg)
    pbuf = sentinel_like((pexp.size,))
    torch.cuda.synchronize()
    dv.dv_stream_out(cx, c, reg, setup, 0, 0, setup, dv.endpoint_array([dv.endpoint_of(inbox, ifl)]), seq=3,
                     stream=sp)
    dv.dv_remap(cx, c, dc, dv.region(*rreg), stream=sp)
    dv.dv_scatter(cx, c, dv.region(*rreg), dv.endpoint_of(pbuf), 0, stream=sp)
    st.synchronize()
    assert np.array_equal(to_np(inbox), exp) and int(ifl[0]) == 3
    ok.remap(o, do, rreg)
    assert np.array_equal(to_np(dk), do.K) and np.array_equal(to_np(dvv), do.V)
    assert np.array_equal(to_np(pbuf), pexp)


def test_partition_streams_run_concurrently_and_destroy():
    """A GEMM loop on the compute partition's stream and token steps on the streaming partition's
    stream at the same time: every streamed word == the oracle; the GEMM's result matches the same GEMM
    on the default stream; destroy after both finished; a second partition can then be made."""
    part = dv.dv_partition_create(0, 16)
    cs, gs = torch.cuda.ExternalStream(part.streaming), torch.cuda.ExternalStream(part.compute)
    a = torch.randn(2048, 2048, device="cuda", dtype=torch.bfloat16)
    ref = a @ a
    L, B, H, S, D = 2, 4, 8, 64, 128
    K, V = kvgen.kv5d_cache("hash", 0, L, 0, B, H, S, D, seed=5)
    c = dv.cache(to_dev(K), to_dev(V))
    o = ok.Cache(K, V, 0, 0, H, S, D)
    torch.cuda.synchronize()
    with torch.cuda.stream(gs):
        outs = [a @ a for _ in range(20)]
    bufs = []
    for q in range(20):
        reg = (0, L, 0, B, q, q + 1)
        buf = sentinel_like((ok.region_bytes(*reg, H, D, 2) // 2,), pinned=True)
        dv.dv_scatter(ctx(), c, dv.region(*reg), dv.endpoint_of(buf), 0, xfer=dv.DV_XFER_FUSED,
                      stream=cs.cuda_stream)
        bufs.append((reg, buf))
    cs.synchronize()
    gs.synchronize()
    for reg, buf in bufs:
        assert np.array_equal(to_np(buf), ok.pack(o, reg))
    assert all(torch.allclose(x.float(), ref.float(), rtol=1e-2, atol=1e-2) for x in outs)
    part.destroy()
    p2 = dv.dv_partition_create(0, 8)
    p2.destroy()
