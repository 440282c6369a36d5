"""Aggregate an `ncu --page source --csv --print-source sass` export by opcode and by
loop region: python tools/ncu_src_regions.py src.csv [kernel-substring]"""
import collections
import csv
import io
import sys

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else None
text = open(path).read().split('"Kernel Name"')
for chunk in text[1:]:
    name, body = chunk.split("\n", 1)
    if want and want not in name:
        continue
    rows = list(csv.DictReader(io.StringIO(body)))
    tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    print(name[:110], "samples", tot)
    byop = collections.Counter()
    inst = collections.Counter()
    for r in rows:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        op = op.split(".")[0]
        byop[op] += int(r["Warp Stall Sampling (All Samples)"] or 0)
        inst[op] += int(r["Instructions Executed"] or 0)
    for op, v in byop.most_common(14):
        print(f"  {op:10s} {100 * v / tot:5.1f}% of samples  inst {inst[op]}")
    # contiguous windows of 64 instructions, sample share (find hot regions)
    win = 64
    shares = []
    for i in range(0, len(rows), win):
        s = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows[i:i + win])
        shares.append((i, s))
    print("  hot 64-instruction windows (index: share):",
          ", ".join(f"{i}:{100 * s / tot:.1f}%" for i, s in sorted(shares, key=lambda t: -t[1])[:12]))
