"""Per-kernel summary of an ncu --metrics launch list CSV (time, DRAM read/write), last N launches."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        hdr, start = r, i
        break
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d, names = defaultdict(dict), {}
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    d[r[ii]][r[mi]] = r[vi].replace(",", "")
    names[r[ii]] = r[ki][:60]
for k in list(d)[-n:]:
    m = d[k]
    print(f"{names[k]:60s} {float(m['gpu__time_duration.sum']) / 1e3:9.1f} us  "
          f"R {float(m.get('dram__bytes_read.sum', 0)) / 1e6:8.1f} MB  W {float(m.get('dram__bytes_write.sum', 0)) / 1e6:8.1f} MB")
