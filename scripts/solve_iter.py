"""Per-launch table of the last CG iteration from an ncu launch CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii, gi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Grid Size"))
L = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = L.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("samgb::", "").replace("<unnamed>::", "").replace("unnamed>::", ""), "grid": r[gi]})
    d[r[mi]] = float(r[vi].replace(",", ""))
items = list(L.values())
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
tot = 0
for d in items[-n:]:
    t = d.get("gpu__time_duration.sum", 0)
    b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tot += t
    print(f"{t/1e3:8.2f} us {b/1e6:8.2f} MB {b/t if t else 0:7.1f} GB/s grid {d['grid']:>12} {d['name'][:60]}")
print("sum us", round(tot / 1e3, 1))
