"""One launch of each HBM-side kernel shape, for an ncu capture (tools/gpu_round.sh style):

  ncu --set full --clock-control none -k regex:"k_run_copy|k_packet_transpose" -o gpurun_out/hbm \
      python tools/ncu_hbm_kernels.py

Launch order (each preceded by one warm-up call that ncu also sees):
  1. C2 token step (6.55 MB, 25,600 runs of 256 B) packed into an HBM wire buffer
  2. C2 prompt layer (163.8 MB, 640 runs of 256 KB) packed into an HBM wire buffer
  3. C3 prompt layer remap, S 1024 -> 2048 (294.9 MB)
  4. FT6D prompt layer pack: K transpose + V run copy in one k_transpose_run launch
  5. one C2 token-layer (160 KiB) into HBM with a seq flag: k_copy_cluster (gpu-scope release)
  6. the same to pinned host with a seq flag: k_run_copy + system-scope release (PCIe stores)
  7. a C2-shaped 9-layer swap-in slice read from a pinned host log with the kernel's own loads
     (fused gather, 16 host CTAs): PCIe read bytes vs payload
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2403_01876_b200 as dv  # noqa: E402


def main():
    ctx = dv.dv_create(0)
    L, H, D, B, P, S = 40, 40, 128, 8, 1000, 2048
    k = torch.empty((L, B, H, S, D), dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    c = dv.cache(k, v)
    wire = torch.empty(2 * B * H * P * D, dtype=torch.int16, device="cuda")
    ep = dv.endpoint_of(wire)
    for _ in range(2):
        dv.dv_scatter(ctx, c, dv.region(0, L, 0, B, P, P + 1), ep, 0)
    for _ in range(2):
        dv.dv_scatter(ctx, c, dv.region(5, 6, 0, B, 0, P), ep, 0)
    torch.cuda.synchronize()
    del k, v
    H3 = 72
    pk = torch.empty((2, B, H3, 1024, D), dtype=torch.int16, device="cuda")
    pv = torch.empty_like(pk)
    tk = torch.empty((2, B, H3, 2048, D), dtype=torch.int16, device="cuda")
    tv = torch.empty_like(tk)
    for _ in range(2):
        dv.dv_remap(ctx, dv.cache(pk, pv), dv.cache(tk, tv), dv.region(0, 1, 0, B, 0, P))
    torch.cuda.synchronize()
    del pk, pv, tk, tv
    k6 = torch.empty((2, B, H, D // 8, S, 8), dtype=torch.int16, device="cuda")
    v6 = torch.empty((2, B, H, S, D), dtype=torch.int16, device="cuda")
    for _ in range(2):
        dv.dv_scatter(ctx, dv.cache(k6, v6), dv.region(0, 1, 0, B, 0, P), ep, 0)
    torch.cuda.synchronize()
    del k6, v6
    k5 = torch.empty((2, B, H, S, D), dtype=torch.int16, device="cuda")
    v5 = torch.empty_like(k5)
    c6 = dv.cache(k5, v5)
    dfl = torch.zeros(1, dtype=torch.int64, device="cuda")
    for i in range(2):
        dv.dv_scatter(ctx, c6, dv.region(1, 2, 0, B, P, P + 1), dv.endpoint_of(wire, dfl), 0, flag_slot=0,
                      seq=1 + i)
    host = torch.empty(2 * B * H * D, dtype=torch.int16, pin_memory=True)
    hfl = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    for i in range(2):
        dv.dv_scatter(ctx, c6, dv.region(1, 2, 0, B, P, P + 1), dv.endpoint_of(host, hfl), 0, flag_slot=0,
                      seq=1 + i)
    torch.cuda.synchronize()
    reg7 = (0, 2, 0, B, 1000, 1064)                       # 2 layers x 64 positions = 20.97 MB (K and V)
    nb7 = 2 * 2 * B * H * 64 * D * 2
    hlog = torch.zeros(nb7 // 2, dtype=torch.int16, pin_memory=True)
    for _ in range(2):
        dv.dv_gather(ctx, dv.endpoint_of(hlog), 0, c6, reg7, xfer=dv.DV_XFER_FUSED)
    torch.cuda.synchronize()
    ctx.close()


if __name__ == "__main__":
    main()
