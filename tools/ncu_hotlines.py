#!/usr/bin/env python
"""Per-source-line warp-stall samples of one kernel in an ncu report (needs -lineinfo builds):

    python tools/ncu_hotlines.py <file.ncu-rep> [kernel-substring] [top]
"""
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    args = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kern:
        args += ["-k", "regex:" + kern]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur = None
    hdr = None
    agg = {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0].isdigit():
            try:
                smp = int(r[4])
            except (ValueError, IndexError):
                continue
            key = (cur, int(r[0]))
            a = agg.setdefault(key, [0, r[1][:100]])
            a[0] += smp
    tot = sum(v[0] for v in agg.values()) or 1
    print(f"# warp-stall samples by source line: {path} {kern}  (total {tot})")
    for (f, ln), (smp, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{smp:9d} {100 * smp / tot:5.1f}%  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
