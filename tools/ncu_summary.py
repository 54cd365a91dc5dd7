"""Summarise ncu output for profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches.csv  > profiles/rNN_launches.txt
    python tools/ncu_summary.py kernels  gpurun_out/prof.ncu-rep  > profiles/rNN_<kernel>.txt

`launches`: per-kernel launch count, total and mean gpu__time_duration from a
`--metrics gpu__time_duration.sum` CSV log (cold-cache, serialised: compare
shares, not absolutes).  `kernels`: the metrics the roofline discussion cites
(DRAM bytes/throughput, L1/L2 hit rates and throughput, occupancy, issue
efficiency, top stall) from an `ncu --set full` report.
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

RAW = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(path: str) -> None:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ki, ni, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg: dict[str, list[float]] = collections.OrderedDict()
    for r in data:
        if r[ni] != "gpu__time_duration.sum":
            continue
        agg.setdefault(r[ki].split("(")[0][:80], []).append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    print(f"{'launches':>8} {'total_ms':>10} {'mean_us':>10} {'share':>7}  kernel")
    for name, v in agg.items():
        print(f"{len(v):8d} {sum(v) / 1e6:10.3f} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / total:7.2%}  {name}")
    print(f"{len(data):8d} {total / 1e6:10.3f}  (all launches)")


def kernels(path: str) -> None:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("-" * 100)
        print("kernel:", r[hdr.index("Kernel Name")])
        for m in RAW:
            if m in hdr:
                i = hdr.index(m)
                print(f"  {m:64s} {r[i]:>18s} {units[i]}")
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    for r in csv.reader(io.StringIO(det)):
        if len(r) > 15 and r[12] in ("Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
                                     "Issue Slots Busy", "Memory Throughput", "Achieved Occupancy"):
            print(f"  [{r[4][:40]}] {r[12]}: {r[14]} {r[13]}")
        if len(r) > 16 and r[15] == "CPIStall" and r[16] == "OPT":
            print(f"  [{r[4][:40]}] stall: {r[17][:260]}")


if __name__ == "__main__":
    {"launches": launches, "kernels": kernels}[sys.argv[1]](sys.argv[2])
