"""Print the per-launch metrics of a tools/l2probe.sh capture: python tools/l2probe_parse.py gpurun_out/TAG/warm.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ik, im, iv, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault((r[iid], r[ik][:30]), {})[r[im]] = float(r[iv].replace(",", ""))
for (i, k), m in d.items():
    print(i, k, " ".join(f"{kk.split('__')[-1][:22]}={vv:.4g}" for kk, vv in m.items()))
