#!/usr/bin/env python
"""Summarise ncu outputs for profiles/.

  python tools/ncu_summary.py launches <launches.csv>         # per-kernel share of a launch list
  python tools/ncu_summary.py report <file.ncu-rep> [...]     # key --set full metrics per kernel
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("GPU Speed Of Light Throughput", "Memory Throughput"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "L2 Cache Throughput"),
    ("GPU Speed Of Light Throughput", "SM Active Cycles"),
    ("GPU Speed Of Light Throughput", "Elapsed Cycles"),
    ("Compute Workload Analysis", "Executed Ipc Active"),
    ("Compute Workload Analysis", "Issue Slots Busy"),
    ("Memory Workload Analysis", "Memory Throughput"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Occupancy", "Achieved Occupancy"),
    ("Occupancy", "Theoretical Occupancy"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Block Size"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_dmma.avg.pct_of_peak_sustained_active",
       "smsp__average_warp_latency_issue_stalled_barrier", "launch__registers_per_thread"]


def to_ms(v, unit):
    v = float(str(v).replace(",", ""))
    return {"ns": v / 1e6, "nsecond": v / 1e6, "us": v / 1e3, "usecond": v / 1e3, "ms": v, "msecond": v,
            "s": v * 1e3, "second": v * 1e3}.get(unit, v / 1e6)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg[k][0] += 1
        agg[k][1] += to_ms(d["Metric Value"], d["Metric Unit"])
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list: {path}  (cold-cache, serialised: compare shares)")
    print(f"{'kernel':64s} {'launches':>8s} {'total ms':>10s} {'avg us':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:64]:64s} {v[0]:8d} {v[1]:10.2f} {v[1] / v[0] * 1e3:9.1f} {v[1] / tot * 100:5.1f}%")
    print(f"{'TOTAL':64s} {sum(v[0] for v in agg.values()):8d} {tot:10.2f}")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        print("no data", path)
        return
    hdr = rows[0]
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        key = (d.get("ID"), d.get("Kernel Name", "")[:70])
        per.setdefault(key, {})[(d.get("Section Name"), d.get("Metric Name"))] = (d.get("Metric Value"), d.get("Metric Unit"))
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rawv = {}
    if len(rr) > 2:
        h = rr[0]
        units = rr[1]
        for row in rr[2:]:
            d = dict(zip(h, row))
            rawv[d.get("ID")] = {k: (d.get(k), units[h.index(k)] if k in h else "") for k in RAW if k in d}
    print(f"# ncu --set full summary: {path}")
    for (kid, name), m in per.items():
        print(f"\n## [{kid}] {name}")
        for sec, met in KEYS:
            if (sec, met) in m:
                v, u = m[(sec, met)]
                print(f"  {met:38s} {v} {u}")
        for k, (v, u) in rawv.get(kid, {}).items():
            print(f"  {k:38s} {v} {u}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        for p in sys.argv[2:]:
            report(p)
