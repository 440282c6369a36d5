"""DRAM traffic per PG pass from an ncu launch list, for bench.py's roofline.traffic.

    python tools/ncu_traffic.py run cN                     # the profiled program
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file traffic_cN.csv python tools/ncu_traffic.py run cN
    python tools/ncu_traffic.py parse cN traffic_cN.csv counts_cN.json   # -> profiles/traffic.json

`run` builds the config's plan (zero inputs: traffic and FFMA time do not depend on
values), warms up one forward (PG residual epilogue) and one adjoint (PG epilogue) pass,
then runs one more of each and prints the launch counts of that last pair as JSON.
`parse` takes the last (forward + adjoint) correlation launches of the ncu CSV in
launch order, sums dram bytes read + written per pass, and records them with their
source in profiles/traffic.json.
"""
import csv
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {"c2": (16, (2048, 2048)), "c2s": (16, (2048, 2048)), "c3": (1, (128, 256, 256)),
          "c4": (1, (512, 1024, 1024)), "c5": (1, (256, 2048, 2048))}


def run(cfg):
    from paper_1711_11224_b200 import ndconv as nd, synth
    B, xs = SHAPES[cfg]
    h = synth.psf_for(cfg)
    ys = tuple(s + k - 1 for s, k in zip(xs, h.shape))
    p = nd.Plan(xs, h, batch=B)
    p.set_observation(np.zeros((B,) + ys, np.float32))
    p.forward()
    p.adjoint()
    p.reset_stats()
    p.forward()
    p.adjoint()
    nf, _ = p.stats(0)
    na, _ = p.stats(1)
    p.close()
    print(json.dumps({"config": cfg, "forward_launches": nf, "adjoint_launches": na}))


def parse(cfg, csv_path, counts_path):
    counts = json.load(open(counts_path))
    rows = list(csv.reader(l for l in open(csv_path) if not l.startswith("==")))
    head = rows[0]
    ki, ni, vi, idi = head.index("Kernel Name"), head.index("Metric Name"), head.index("Metric Value"), head.index("ID")
    per = {}
    for r in rows[1:]:
        if len(r) <= max(ki, ni, vi) or "correlate" not in r[ki]:  # correlate_kernel, correlate_pair_kernel
            continue
        d = per.setdefault(int(r[idi]), {})
        d[r[ni]] = float(r[vi].replace(",", ""))
    ids = sorted(per)
    nf, na = counts["forward_launches"], counts["adjoint_launches"]
    last = ids[-(nf + na):]
    fwd, adj = last[:nf], last[nf:]

    def tot(group, key):
        return sum(per[i].get(key, 0.0) for i in group)

    out = {}
    for name, g in (("forward", fwd), ("adjoint", adj)):
        out[name] = int(tot(g, "dram__bytes_read.sum") + tot(g, "dram__bytes_write.sum"))
        out[name + "_read"] = int(tot(g, "dram__bytes_read.sum"))
        out[name + "_write"] = int(tot(g, "dram__bytes_write.sum"))
        out[name + "_ncu_ms"] = tot(g, "gpu__time_duration.sum") / 1e6
        out[name + "_launches"] = len(g)
    head_commit = subprocess.run(["git", "rev-parse", "--short", "HEAD"], cwd=ROOT, capture_output=True,
                                 text=True).stdout.strip()
    out["source"] = (f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (per launch, summed per pass) "
                     f"over tools/ncu_traffic.py run {cfg} at {head_commit or 'HEAD'}: {os.path.basename(csv_path)}")
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    data = json.load(open(tf)) if os.path.exists(tf) else {}
    data[cfg] = out
    data["_source"] = "tools/ncu_traffic.py: DRAM bytes read + written per pass (all launches of the pass)"
    json.dump(data, open(tf, "w"), indent=1)
    print(json.dumps({cfg: out}))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        parse(sys.argv[2], sys.argv[3], sys.argv[4])
