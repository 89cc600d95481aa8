"""Summarise a ptxas -v log: kernel (demangled-ish), registers, spills, smem."""
import re
import sys

cur = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = int(m.group(1)) + int(m.group(2))
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        pat = sys.argv[2] if len(sys.argv) > 2 else ""
        if pat in cur:
            print(f"regs={m.group(1):>4} spill={spill:>5}  {cur[:160]}")
        cur = None
