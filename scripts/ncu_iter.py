"""Per-kernel table of one CG iteration from an ncu --csv launch list
(gpu__time_duration / dram bytes; host-loop mode, SAMG_CG_GRAPH=0).

    python scripts/ncu_iter.py LAUNCHES.csv [--json OUT]
The last full iteration is the launches between the last two q = A p
(EpiDot) kernels."""
import argparse
import collections
import csv
import json

MULT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
        "msecond": 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--json")
    ap.add_argument("--peak", type=float, default=6547.2)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui, idi = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                                 "Metric Unit", "ID"))
    launch = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = launch.setdefault(r[idi], {"kernel": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", "")) * MULT.get(r[ui], 1)
    L = list(launch.values())
    idx = [i for i, d in enumerate(L) if "EpiDot" in d["kernel"]]
    it = L[idx[-2]:idx[-1]]
    out, tt, tb = [], 0.0, 0.0
    for d in it:
        t = d.get("gpu__time_duration.sum", 0.0)
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        tt += t
        tb += b
        name = d["kernel"].split("(")[0].replace("samgb::<unnamed>::", "").replace("void ", "")
        out.append({"kernel": name[:90], "us": round(t, 2), "dram_MB": round(b / 1e6, 2),
                    "TBps": round(b / t / 1e6, 2) if t else 0.0})
        print(f"{t:8.2f} us {b / 1e6:9.2f} MB {b / t / 1e6 if t else 0:6.2f} TB/s  {name[:90]}")
    print(f"total {tt:.1f} us, {tb / 1e9:.3f} GB DRAM, {tb / tt / 1e6:.2f} TB/s "
          f"= {tb / tt / 1e6 * 1e3 / a.peak:.3f} of {a.peak} GB/s")
    if a.json:
        json.dump({"kernels": out, "total_us": tt, "dram_GB": tb / 1e9,
                   "TBps": tb / tt / 1e6}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
