#!/usr/bin/env python
"""Summarise an ncu report (or a launch-list CSV) for profiles/.

    python scripts/ncu_summary.py report gpurun_out/prof.ncu-rep  [--bytes-per-launch B]
    python scripts/ncu_summary.py launches gpurun_out/launches.csv

`report` prints the key per-kernel metrics (duration, DRAM bytes/throughput,
occupancy, registers, top warp stalls) as JSON; `launches` prints each
kernel's share of the summed device time (ncu launch times are cold-cache and
serialised, so shares -- not absolutes -- are what compare with bench.py).
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct",
    "lts__t_sector_hit_rate.pct", "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__cycles_elapsed.avg.per_second",
]


def report(path, bytes_per_launch=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        stalls = {}
        for h, u, v in zip(hdr, units, r):
            if h in KEYS:
                d[h] = f"{v} {u}".strip()
            if h.startswith("smsp__average_warp_latency_issue_stalled_") or \
               (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")):
                try:
                    stalls[h.split("stalled_")[-1]] = float(v.replace(",", ""))
                except ValueError:
                    pass
        if stalls:
            top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
            d["top_stalls"] = top
        try:
            rd = float(d["dram__bytes_read.sum"].split()[0].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"].split()[0].replace(",", ""))
            unit = d["dram__bytes_read.sum"].split()[1]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d["dram_traffic_bytes"] = (rd + wr) * scale
            if bytes_per_launch:
                d["traffic_over_algorithmic"] = d["dram_traffic_bytes"] / bytes_per_launch
        except (KeyError, ValueError, IndexError):
            pass
        res.append(d)
    print(json.dumps(res, indent=1))


def launches(path):
    rows = list(csv.reader(open(path)))
    # find header row
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[i]
    kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = {}
    for r in rows[i + 1:]:
        if len(r) <= mv:
            continue
        name = r[kn].split("(")[0].replace("void ", "")
        try:
            ns = float(r[mv].replace(",", ""))
        except ValueError:
            continue
        n, t = tot.get(name, (0, 0.0))
        tot[name] = (n + 1, t + ns)
    all_ns = sum(t for _, t in tot.values())
    out = [{"kernel": k, "launches": n, "total_us": t / 1e3, "mean_us": t / n / 1e3,
            "share": t / all_ns} for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1])]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "report":
        b = None
        if "--bytes-per-launch" in sys.argv:
            b = float(sys.argv[sys.argv.index("--bytes-per-launch") + 1])
        report(sys.argv[2], b)
    else:
        launches(sys.argv[2])
