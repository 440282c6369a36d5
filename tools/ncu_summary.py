"""Summarise ncu outputs into profiles/ (committed evidence).

    python tools/ncu_summary.py launches gpurun_out/launches_r01.csv profiles/r01_launches.md
    python tools/ncu_summary.py full gpurun_out/prof_r01.ncu-rep profiles/r01_correlate_full.md
    python tools/ncu_summary.py full gpurun_out/prof_r01_raw.csv profiles/r01_correlate_full.md

`launches`: per-kernel launch counts, total / mean device time and share (the ncu
per-launch times are cold-cache and serialised -- compare shares, not absolutes).
`full`: the headline counters of a --set full capture (duration, DRAM bytes, SM /
FMA-pipe / issue utilisation, occupancy, registers) per profiled launch.
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys


def launches(path: str, out: str):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "second": 1e3, "s": 1e3}
        ms = v * scale.get(unit, 1e-6)
        rows.append((short, ms))
    agg = collections.OrderedDict()
    for k, ms in rows:
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + ms)
    total = sum(t for _, t in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list: {path}\n\n")
        f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` over the whole command "
                "(setup + warm-up + timed steps); per-launch times are cold-cache and serialised.\n\n")
        f.write("| kernel | launches | total ms | mean ms | share |\n|---|---|---|---|---|\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| `{k}` | {n} | {t:.3f} | {t / n:.4f} | {t / total:.1%} |\n")
    print(open(out).read())


METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "smsp__inst_executed.sum",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__average_warp_latency_issue_stalled_barrier",
]


def full(path: str, out: str):
    # a .ncu-rep, or its `--page raw --csv` export (exported on the GPU box when the
    # report itself is too large to bring back)
    if path.endswith(".csv"):
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rdr = list(csv.reader(io.StringIO(raw)))
    if len(rdr) < 3:
        raise SystemExit("no data in " + path)
    hdr, units, data = rdr[0], rdr[1], rdr[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    with open(out, "w") as f:
        f.write(f"# ncu --set full: {path}\n\n")
        for row in data:
            f.write(f"## {row[idx['Kernel Name']][:120]}\n\n| metric | value | unit |\n|---|---|---|\n")
            for m in METRICS:
                if m in idx:
                    f.write(f"| {m} | {row[idx[m]]} | {units[idx[m]]} |\n")
            f.write("\n")
    print(open(out).read())


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
