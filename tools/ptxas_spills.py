"""Registers / spills per kernel from `nvcc -Xptxas -v` output on stdin:
    nvcc ... -Xptxas -v -c x.cu 2>&1 | python tools/ptxas_spills.py [name-filter]"""
import re
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur and pat in cur:
        st, ld = m.groups()
        short = re.sub(r"_ZN4gift\w+?_GLOBAL__N__\w+?(\d+)(k_\w+?)I", r"\2<", cur)
        sys.stdout.write(f"{short[:60]:60s} spill st {st:>5} ld {ld:>5}\n")
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and pat in cur:
        sys.stdout.write(f"{'':60s} regs {m.group(1)}\n")
        cur = None
