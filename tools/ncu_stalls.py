"""Per-kernel stall breakdown and key counters from an ncu raw CSV export
(ncu -i rep --page raw --csv):  python tools/ncu_stalls.py raw.csv [top]"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic"]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(d["Kernel Name"][:90])
        for k in KEYS:
            if k in d:
                print(f"   {k:60s} {d[k]} {units[hdr.index(k)]}")
        st = [(k, float(v.replace(",", ""))) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v not in ("", "n/a")]
        tot = sum(v for _, v in st) or 1.0
        print("   stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.1f}%"
                                      for k, v in sorted(st, key=lambda x: -x[1])[:top]))


if __name__ == "__main__":
    main()
