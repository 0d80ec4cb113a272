"""P0 probe: host/PCIe facts of the GPU box, written to gpurun_out/probe_host.json.
Uses torch only (plumbing); no product code."""
import json, os, subprocess, time, platform
import torch

out = {}
def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)
out["nproc"] = os.cpu_count()
out["sched_affinity"] = len(os.sched_getaffinity(0))
out["cpu_model"] = [l for l in open("/proc/cpuinfo") if "model name" in l][:1]
out["meminfo"] = sh("head -3 /proc/meminfo")
out["ulimit_l"] = sh("ulimit -l")
out["numa"] = sh("ls /sys/devices/system/node | grep node")
out["smi_pcie"] = sh("nvidia-smi -q | grep -A12 -i 'GPU Link Info'")
out["topo"] = sh("nvidia-smi topo -m")
out["gpu_count"] = torch.cuda.device_count()
dev = torch.device("cuda:0")
res = {}
for mb in [1, 16, 256, 1024]:
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
        for _ in range(3): fn()
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        reps = 10
        s.record()
        for _ in range(reps): fn()
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        res[f"{name}_{mb}MiB_GBps"] = n / ms / 1e6
    del h, d
out["pinned_copy"] = res
# large pinned allocation test
t0 = time.time()
try:
    big = torch.empty(32 << 30, dtype=torch.uint8, pin_memory=True)
    out["pin_32GiB_s"] = time.time() - t0
    del big
except Exception as ex:
    out["pin_32GiB_err"] = str(ex)[:300]
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_host.json", "w"), indent=1)
print(json.dumps(out, indent=1))
