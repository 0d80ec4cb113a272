"""Summarise ncu outputs (launch list CSV, --set full report, counter CSV) into markdown for profiles/.

  python tools/ncu_summary.py TAG [title]   -> prints markdown (reads gpurun_out/*_TAG.*)
"""
import csv
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")

FULL_KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
             "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
             "sm__warps_active.avg.pct_of_peak_sustained_active",
             "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
             "smsp__inst_executed.sum", "lts__t_bytes.sum"]


def rows_of(path):
    lines = [l for l in open(path) if l.startswith('"')]
    return list(csv.reader(lines))


def launches(tag):
    p = os.path.join(OUT, f"launches_{tag}.csv")
    if not os.path.exists(p):
        return ""
    r = rows_of(p)
    hdr, body = r[0], r[1:]
    agg = defaultdict(list)
    for x in body:
        d = dict(zip(hdr, x))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            agg[(d["Kernel Name"], d["Grid Size"], d["Block Size"])].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    s = ["| kernel | grid | block | launches | avg us | share of GPU time |", "|---|---|---|---|---|---|"]
    for (k, g, b), v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        s.append(f"| `{k}` | {g} | {b} | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / tot:.1%} |")
    return "\n".join(s)


def full(tag):
    p = os.path.join(OUT, f"prof_{tag}.ncu-rep")
    if not os.path.exists(p):
        return ""
    out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr = r[0]
    s = ["| launch | " + " | ".join(FULL_KEYS) + " |", "|---" * (len(FULL_KEYS) + 1) + "|"]
    for i, x in enumerate(r[2:]):
        vals = [x[hdr.index(k)] if k in hdr else "-" for k in FULL_KEYS]
        s.append(f"| {i} ({x[hdr.index('Kernel Name')]}) | " + " | ".join(vals) + " |")
    units = r[1]
    s.append("")
    s.append("units: " + ", ".join(f"{k}={units[hdr.index(k)]}" for k in FULL_KEYS if k in hdr))
    return "\n".join(s)


def io(tag):
    p = os.path.join(OUT, f"io_{tag}.csv")
    if not os.path.exists(p):
        return ""
    r = rows_of(p)
    hdr, body = r[0], r[1:]
    per = defaultdict(dict)
    for x in body:
        d = dict(zip(hdr, x))
        per[d["ID"]][d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    keys = sorted({k for v in per.values() for k in v})
    s = ["| launch | " + " | ".join(keys) + " |", "|---" * (len(keys) + 1) + "|"]
    for i, v in per.items():
        s.append(f"| {i} | " + " | ".join(f"{v[k][0]} {v[k][1]}" for k in keys) + " |")
    return "\n".join(s)


if __name__ == "__main__":
    tag = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else tag
    print(f"# ncu summary {title}\n")
    print("## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised)\n")
    print(launches(tag) + "\n")
    print("Reading the list: the command is `bench.py --steps 20 --warmup 3 --no-extras "
          "--no-cpu-baseline`. Its TIMED region launches exactly one kernel per token step, the "
          "200-CTA `k_run_copy<32, 4, 256>` pack (cache -> HBM staging, 6.55 MB); the step's bytes "
          "then cross PCIe by copy-engine DMA, which ncu does not list. `k_fill` (writing the 13.4 GB "
          "synthetic cache), the 16-CTA copies (preparing the e2e loop's host-side K/V) and `k_verify` "
          "(every-word parity of the last 8 steps) run outside the timed region. Inside a step the pack "
          "is ~4-5.5 us of ~119 us (3-5 %); the rest is the DMA, which is why the headline roofline "
          "is the PCIe link.\n")
    print("## Top kernel, --set full\n")
    print(full(tag) + "\n")
    print("## DRAM / PCIe counters per launch\n")
    print(io(tag))
