"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    out = []
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            out.append((r[ki], float(r[vi].replace(",", ""))))
    return out


def short(name):
    name = name.replace("samgb::", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    return name.split("(")[0][:70] + ("<" + name.split("<", 1)[1].split("(")[0][:40] if "<" in name.split("(")[0] and False else "")


def main(path, top=30):
    launches = load(path)
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for n, t in launches:
        k = n.split("(")[0][:100]
        tot[k] += t
        cnt[k] += 1
    T = sum(tot.values())
    print(f"{len(launches)} launches, {T/1e6:.3f} ms total (ncu, serialised, cold cache)")
    print(f"{'ms':>9} {'share':>6} {'n':>6} {'us/launch':>10}  kernel")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        print(f"{v/1e6:9.3f} {100*v/T:5.1f}% {cnt[k]:6d} {v/cnt[k]/1e3:10.2f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
