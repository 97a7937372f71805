#!/usr/bin/env python
"""Summarise ncu outputs for profiles/.

  python tools/ncu_summary.py launches <launches.csv>         # per-kernel share of a launch list
  python tools/ncu_summary.py report <file.ncu-rep> [...]     # key --set full metrics per kernel
  python tools/ncu_summary.py traffic <CONFIG> <file.ncu-rep> [...]
        # dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged per kernel, merged into
        # profiles/ncu_traffic.json under CONFIG (the 'traffic' field of bench.py's roofline)
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


# bench.py kernel keys <- ncu kernel-name prefixes
TRAFFIC_KEYS = [("qrp_coop", "k_qrp_lazy"), ("pair_gram_f32", "k_pair_gram_tma"), ("pair_gram_f32", "k_pair_gram_tc"),
                ("pair_gram_f32", "k_pair_gram_sw"),
                ("pair_update_f32", "k_pair_update_tc"), ("pair_solve_f32", "k_pair_solve<float"),
                ("pair_gram_f64", "k_pair_gram_dmma"), ("pair_update_f64", "k_pair_update_dmma"),
                ("pair_solve_f64", "k_pair_solve<double")]


def traffic(config, paths):
    import json
    import os
    acc = collections.defaultdict(list)
    for path in paths:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(io.StringIO(raw)))
        if len(rr) < 3:
            continue
        h, units = rr[0], rr[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        for row in rr[2:]:
            d = dict(zip(h, row))
            name = d.get("Kernel Name", "").replace("void ", "").replace("mpj::", "")
            try:
                rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale.get(units[h.index("dram__bytes_read.sum")], 1)
                wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale.get(units[h.index("dram__bytes_write.sum")], 1)
            except (KeyError, ValueError):
                continue
            for key, pref in TRAFFIC_KEYS:
                if name.startswith(pref):
                    acc[key].append(rd + wr)
                    break
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    try:
        allv = json.load(open(out_path))
    except Exception:
        allv = {}
    if "_source" in allv and not isinstance(allv.get("_source"), dict):
        allv = {k: v for k, v in allv.items() if isinstance(v, dict)}     # round-1 flat layout: drop
    entry = {k: sum(v) / len(v) for k, v in acc.items()}
    entry["_source"] = ", ".join(paths) + " (ncu --set full; dram read + write bytes per launch, mean over captured launches)"
    entry["_launches"] = {k: len(v) for k, v in acc.items()}
    allv[config] = entry
    json.dump(allv, open(out_path, "w"), indent=1)
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3:])
    else:
        for p in sys.argv[2:]:
            report(p)
