"""Helpers for the GPU tests: move kvgen/oracle numpy arrays to and from torch memory.

Bit patterns travel as int16 views (torch has no arithmetic on them here), so nothing is ever
converted through a float type.
"""
import numpy as np
import torch

import paper_2403_01876_b200 as dv


def to_dev(a: np.ndarray, device="cuda:0") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(device)


def to_pinned(a: np.ndarray) -> torch.Tensor:
    t = torch.empty(a.shape, dtype=torch.int16, pin_memory=True)
    t.copy_(torch.from_numpy(np.ascontiguousarray(a).view(np.int16)))
    return t


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)


def sentinel_like(shape, device="cuda:0", pinned=False):
    if pinned:
        t = torch.empty(shape, dtype=torch.int16, pin_memory=True)
    else:
        t = torch.empty(shape, dtype=torch.int16, device=device)
    t.fill_(-1)  # 0xFFFF
    return t


def pinned_u16(n):
    t = torch.empty(n, dtype=torch.int16, pin_memory=True)
    t.fill_(-1)
    return t


def flags(n, device="cuda:0", pinned=False):
    if pinned:
        t = torch.zeros(n, dtype=torch.int64, pin_memory=True)
    else:
        t = torch.zeros(n, dtype=torch.int64, device=device)
    return t


def stream_ptr():
    return torch.cuda.current_stream().cuda_stream


_CTX = {}


def ctx(staging=0):
    key = staging
    if key not in _CTX:
        _CTX[key] = dv.dv_create(0, staging_bytes=staging)
    return _CTX[key]
