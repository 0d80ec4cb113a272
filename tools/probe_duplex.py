"""Probe: host memory bandwidth and concurrent H2D + D2H copy-engine throughput (is e2e bounded by
the PCIe link or by host DRAM?). Writes JSON to stdout."""
import json
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

out = {}
a = np.ones(1 << 30, np.uint8)
b = np.empty_like(a)
np.copyto(b, a)
t = time.perf_counter()
for _ in range(3):
    np.copyto(b, a)
out["host_memcpy_1thread_GBps_rw"] = 3 * 2 * a.nbytes / (time.perf_counter() - t) / 1e9
n = os.cpu_count()
chunks = np.array_split(np.arange(a.size), n)
def cp(ix):
    np.copyto(b[ix[0]:ix[-1] + 1], a[ix[0]:ix[-1] + 1])
with ThreadPoolExecutor(n) as ex:
    list(ex.map(cp, chunks))
    t = time.perf_counter()
    for _ in range(3):
        list(ex.map(cp, chunks))
out["host_memcpy_allthreads_GBps_rw"] = 3 * 2 * a.nbytes / (time.perf_counter() - t) / 1e9
N = 256 << 20
h1 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(N, dtype=torch.uint8, device="cuda")
d2 = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("d2h_only", lambda: h1.copy_(d1, non_blocking=True)),
                 ("h2d_only", lambda: d2.copy_(h2, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    out[name + "_GBps"] = 5 * N / (time.perf_counter() - t) / 1e9
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        h1.copy_(d1, non_blocking=True)
    with torch.cuda.stream(s2):
        d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t
out["duplex_total_GBps"] = 2 * 5 * N / dt / 1e9
out["duplex_per_direction_GBps"] = 5 * N / dt / 1e9
print(json.dumps(out))
