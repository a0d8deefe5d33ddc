"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel name."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
for k, v in d.items():
    print(f"{k:70s} n={len(v):4d} mean={sum(v) / len(v) / 1000:9.1f} us  total={sum(v) / 1e6:9.3f} ms")
