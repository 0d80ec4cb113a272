"""The README usage example, run as a script (checks the docs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2403_01876_b200 as dv
ctx = dv.dv_create(0)
k = torch.empty((40, 8, 40, 2048, 128), dtype=torch.float16, device="cuda"); v = torch.empty_like(k)
cache = dv.cache(k, v)                                   # layers 0..39, requests 0..7
cache2 = dv.cache(torch.empty_like(k), torch.empty_like(v))
log = torch.empty(2 * 40 * 8 * 40 * 128, dtype=torch.float16, pin_memory=True)
flag = torch.zeros(1, dtype=torch.int64, pin_memory=True)
# stream the K/V of token position 1000 (all layers) to pinned host, publish seq 1 when landed
dv.dv_scatter(ctx, cache, dv.region(0, 40, 0, 8, 1000, 1001), dv.endpoint_of(log, flag), 0,
              flag_slot=0, seq=1)

# a 2-slot ring inbox with credits: step t lands in slot t % 2; the sender's copy waits (stream-
# ordered) until the receiver has consumed step t - 2; with DV_NOWAIT it returns DV_EBUSY instead
step = 2 * 40 * 8 * 40 * 128 * 2
ring = torch.empty(2 * step // 2, dtype=torch.float16, device="cuda")
fl, cr = (torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(2))
inbox = dv.endpoint_of(ring, fl, n_slots=2, slot_bytes=step, credits=cr)
stage = dv.Setup([0, 40], [0, 8], 2048)
for t in range(1, 5):
    reg = (0, 40, 0, 8, 1000 + t, 1001 + t)
    dv.dv_stream_out(ctx, cache, reg, stage, 0, 0, stage, [inbox], seq=t)    # sender
    dv.dv_stream_in(ctx, cache2, reg, stage, stage, 0, 0, inbox, t)           # receiver releases the credit
torch.cuda.synchronize()
assert int(flag[0]) == 1 and int(fl[0]) == 4 and int(cr[0]) == 4
print("readme example ok")
