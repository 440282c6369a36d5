"""Instructions executed per source line and warp from an `ncu --set full --import-source on`
report: python tools/ncu_lines.py report.ncu-rep [block] [warps]  (block: 1-based function index;
warps: divide by the launch's warp count for per-warp figures).  Captures: tools/ncu_run_cfg.py."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
block = int(sys.argv[2]) if len(sys.argv) > 2 else 1
text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                      capture_output=True, text=True).stdout
parts = text.split('"File Path"')
blk = parts[block]
path = blk.split("\n", 1)[0].strip(',"')
fn = blk.split("\n", 2)[1]
body = blk.split("\n", 2)[2]
rows = list(csv.reader(io.StringIO(body)))
hdr = rows[0]
li, ii = hdr.index("Line No"), hdr.index("Instructions Executed")
per, ops, cur = collections.OrderedDict(), collections.defaultdict(collections.Counter), None
for r in rows[1:]:
    if len(r) <= ii:
        continue
    if r[li]:
        cur = int(r[li])
        continue
    if cur is None or r[2] in ("", "..."):
        continue
    try:
        n = int(r[ii])
    except ValueError:
        continue
    sp = r[3].split()
    op = sp[1] if sp and sp[0].startswith("@") else (sp[0] if sp else "?")
    per[cur] = per.get(cur, 0) + n
    ops[cur][op.split(".")[0]] += n
try:
    src = open(path).read().split("\n")
except OSError:
    src = []
tot = sum(per.values())
W = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
print(fn[:150])
print("total instructions", tot, "per warp", tot / W)
for ln, n in sorted(per.items()):
    if n > tot * 0.006:
        top = ", ".join(f"{o}:{c / W:.0f}" for o, c in ops[ln].most_common(5))
        line = src[ln - 1].strip()[:70] if ln - 1 < len(src) else ""
        print(f"{ln:4d} {n / W:7.1f}  {line:70s} | {top}")
