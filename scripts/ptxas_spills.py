"""Registers and spills per kernel from `nvcc -Xptxas -v` output on stdin (dev aid).
usage: nvcc ... -Xptxas -v 2>&1 | python scripts/ptxas_spills.py [name-filter]"""
import re
import sys

flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
rows = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows.setdefault(cur, {})["spill"] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows.setdefault(cur, {})["reg"] = int(m.group(1))
for k, v in rows.items():
    if flt in k:
        print(f"{v.get('reg', '?'):>4} regs {v.get('spill', 0):>4} B spill  {k}")
