"""Mean duration per kernel name from an ncu --metrics gpu__time_duration.sum
--csv launch list:  python tools/launch_means.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[h + 1:]:
    agg.setdefault(r[ki][:70], []).append(float(r[vi].replace(",", "")))
for k, v in agg.items():
    print(f"{k:70s} n={len(v):3d} mean={sum(v) / len(v) / 1e6:8.3f} ms")
