"""Per-kernel mean duration from an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, d = None, collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h):
        d[r[h.index("Kernel Name")][:80]].append(float(r[h.index("Metric Value")].replace(",", "")))
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):5d} {sum(v) / len(v) / 1e3:9.2f} us  {k}")
