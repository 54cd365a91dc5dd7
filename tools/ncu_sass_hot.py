"""Hot SASS lines of one kernel from an ncu source-page CSV export
(ncu -i rep --page source --csv --print-source sass):
    python tools/ncu_sass_hot.py sass.csv[.gz] KERNEL_SUBSTRING [min_share]"""
import csv
import gzip
import io
import sys


def main():
    path, pat = sys.argv[1], sys.argv[2]
    thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
    f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    rows = list(csv.reader(f))
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r]
            secs.append(cur)
        elif cur is not None:
            cur.append(r)
    num = lambda x: int(x.replace(",", "")) if x.replace(",", "").isdigit() else 0
    for s in secs:
        if pat not in s[0][1]:
            continue
        hdr = s[1]
        data = [r for r in s[2:] if len(r) > 5]
        ai, si = hdr.index("Address"), hdr.index("Source")
        ei, wi = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        tot, samp = sum(num(r[ei]) for r in data), sum(num(r[wi]) for r in data)
        print(s[0][1][:100], "inst", tot, "samples", samp)
        for r in data:
            if num(r[ei]) > tot * thr or num(r[wi]) > samp * thr:
                print(f"{r[ai][-5:]} {num(r[ei]) / 1e6:8.2f}M {100 * num(r[wi]) / samp:5.1f}%  {r[si].strip()[:80]}")
        break


if __name__ == "__main__":
    main()
