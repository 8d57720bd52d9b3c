#!/usr/bin/env python3
"""Summarise ncu captures for profiles/: key metrics of each `--set full` report and the
per-kernel share of a `gpu__time_duration.sum` launch list.

    python scripts/ncu_summary.py OUT.md report1.ncu-rep ... [--launches launches.csv]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "lts__t_bytes.sum",
]


def report_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        res.append((d.get("Kernel Name", "?"), {k: (d[k], u.get(k, "")) for k in KEYS if k in d}))
    return res


def launches(path):
    per = defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(lines)))
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
        name = r["Kernel Name"].split("(")[0]
        per[name][0] += 1
        per[name][1] += v * scale
    return per


def main():
    args = sys.argv[1:]
    out = args[0]
    lpath = None
    if "--launches" in args:
        i = args.index("--launches")
        lpath = args[i + 1]
        args = args[:i] + args[i + 2:]
    lines = []
    for rep in args[1:]:
        lines.append(f"## {rep}\n")
        for name, m in report_rows(rep):
            lines.append(f"### `{name[:120]}`\n")
            lines.append("| metric | value | unit |\n|---|---|---|")
            for k, (v, u) in m.items():
                lines.append(f"| {k} | {v} | {u} |")
            lines.append("")
    if lpath:
        per = launches(lpath)
        tot = sum(v[1] for v in per.values())
        lines.append(f"## launch list {lpath} (ncu, serialised, cold-cache: compare shares)\n")
        lines.append("| kernel | launches | total us | share |\n|---|---|---|---|")
        for name, (n, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| {name} | {n} | {us:.1f} | {us / tot:.3f} |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
