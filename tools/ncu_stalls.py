#!/usr/bin/env python
"""Per-source-line warp-stall reasons of one kernel in an ncu report (needs -lineinfo builds):

    python tools/ncu_stalls.py <file.ncu-rep> <kernel-substring> <file-substring> <line-lo> <line-hi>

Prints, for every source line of the file in [lo, hi] with samples, the total samples and the three largest
stall-reason columns of ncu's source page.
"""
import csv
import io
import subprocess
import sys


def main():
    path, kern, fsub, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
    args = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, hdr = None, None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not (hdr and r and r[0].isdigit() and cur and fsub in cur):
            continue
        ln = int(r[0])
        if ln < lo or ln > hi:
            continue
        vals = {}
        for h, v in zip(hdr, r):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    vals[h] = float(v)
                except ValueError:
                    pass
        tot = sum(vals.values())
        if tot <= 0:
            continue
        top = sorted(vals.items(), key=lambda kv: -kv[1])[:4]
        print(f"{ln:5d} {tot:10.0f}  {r[1].strip()[:70]:70s} " + "  ".join(f"{k[6:]}={v:.0f}" for k, v in top))


if __name__ == "__main__":
    main()
