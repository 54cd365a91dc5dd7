"""DRAM traffic per hop launch from an `ncu --set full` report -> profiles/rNN_traffic_<config>.json.

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep "<how it was captured>" > profiles/r01_traffic_c3.json

Keys are "<kernel><FIN, FOUT>" (k_hop_bmt / k_hop); values average over the
captured launches: dram_bytes_per_launch (dram__bytes_read.sum +
dram__bytes_write.sum) and ncu_ms (gpu__time_duration.sum, cold-cache,
serialised).  bench.py reads the newest such file for the `traffic` field.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import re
import subprocess
import sys


def main() -> None:
    rep, source = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head = rows[0]
    ix = {k: head.index(k) for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
                                      "dram__bytes_write.sum")}
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    acc = collections.defaultdict(lambda: [0.0, 0.0, 0])
    for r in rows[2:]:
        name = r[ix["Kernel Name"]]
        m = re.search(r"(k_hop_bmt_nb|k_hop_bmt|k_hop)<(\d+), (\d+)", name)
        if not m:
            continue
        key = f"{m.group(1)}<{m.group(2)}, {m.group(3)}>"
        b = sum(float(r[ix[k]].replace(",", "")) * scale[units[ix[k]]]
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        t = float(r[ix["gpu__time_duration.sum"]].replace(",", "")) * tscale[units[ix["gpu__time_duration.sum"]]]
        a = acc[key]
        a[0] += b
        a[1] += t
        a[2] += 1
    out = {"source": source,
           "kernels": {k: {"dram_bytes_per_launch": round(v[0] / v[2]), "ncu_ms": round(v[1] / v[2], 6),
                           "launches": v[2]} for k, v in acc.items()}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
