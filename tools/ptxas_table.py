"""Summarise `nvcc -Xptxas -v` output (stdin): correlate_kernel<KX,SH,RY,EDGE> -> registers, spills."""
import re
import sys

cur = None
rows = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        k = re.search(r"correlate_kernelILi(\d+)ELi(\d+)ELi(\d+)ELb(\d)E", m.group(1))
        cur = f"KX={k.group(1)} SH={k.group(2)} RY={k.group(3)} EDGE={k.group(4)}" if k else None
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows.setdefault(cur, {})["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
for k in sorted(rows, key=lambda s: [int(t.split("=")[1]) for t in s.split()]):
    r = rows[k]
    print(f"{k:28s} regs {r.get('regs')}  spill st/ld {r.get('spill')}")
