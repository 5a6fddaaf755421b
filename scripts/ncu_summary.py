"""Summarise an ncu --set full report (raw page) into JSON for profiles/.

    python scripts/ncu_summary.py REPORT.ncu-rep OUT.json [--algorithmic BYTES] [--config TEXT]

Writes the per-launch metrics that the roofline needs (duration, DRAM bytes,
DRAM throughput, occupancy, cache hit rates, shared-memory bank conflicts)
and, for the first launch, the bench-facing summary keys used by bench.py
(dram_bytes_per_launch = mean over launches of read + write).
"""
import argparse
import csv
import json
import re
import subprocess

KEEP = re.compile(r"^(gpu__time_duration|dram__bytes_(read|write)\.sum$|dram__bytes\.sum\.per_second"
                  r"|gpu__dram_throughput\.avg\.pct|launch__|sm__warps_active\.avg\.pct"
                  r"|sm__throughput\.avg\.pct|lts__t_sector_hit_rate\.pct|l1tex__t_sector_hit_rate\.pct"
                  r"|l1tex__data_bank_conflicts_pipe_lsu_mem_shared\.sum$|smsp__inst_executed\.sum$"
                  r"|sm__cycles_elapsed\.avg$|smsp__average_warp_latency_issue_stalled)")

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--algorithmic", type=float, default=None)
    ap.add_argument("--config", default="")
    a = ap.parse_args()
    if a.report.endswith(".csv"):  # the raw page already exported on the GPU box (ncu -i REP --page raw --csv)
        raw = open(a.report).read()
    else:
        raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    head, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"Kernel Name": r[head.index("Kernel Name")]}
        for k, u, v in zip(head, units, r):
            if KEEP.match(k):
                d[k] = f"{v} {u}".strip()
        launches.append(d)

    def bytes_of(d, k):
        v, u = d[k].split()
        return float(v.replace(",", "")) * UNIT[u]

    traffic = [bytes_of(d, "dram__bytes_read.sum") + bytes_of(d, "dram__bytes_write.sum")
               for d in launches]
    dur = [float(d["gpu__time_duration.sum"].split()[0]) for d in launches]
    summary = {"kernel": launches[0]["Kernel Name"], "config": a.config,
               "launches": len(launches),
               "dram_bytes_per_launch": sum(traffic) / len(traffic),
               "algorithmic_bytes_per_launch": a.algorithmic,
               "ncu_duration_us": sum(dur) / len(dur),
               "source": a.report.split("/")[-1] + " (ncu --set full --clock-control none)",
               "per_launch": launches}
    with open(a.out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "per_launch"}, indent=1))


if __name__ == "__main__":
    main()
