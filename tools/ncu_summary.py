#!/usr/bin/env python
"""Summarise ncu output (run here, on the CPU box) for profiles/.

usage:
  python tools/ncu_summary.py launches <launches.csv>          per-kernel launch times and shares
  python tools/ncu_summary.py full <report.ncu-rep> [algo_bytes_per_launch]
  python tools/ncu_summary.py traffic <report.ncu-rep> <n_hexes> <out.json>
      DRAM bytes per hex of the first kernel in the capture (bench.py's roofline.traffic)
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread",
    "launch__block_size",
    "launch__grid_size",
    "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "lts__t_sector_hit_rate.pct",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_wait_per_warp_active.pct",
    "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
    "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_no_instruction_per_warp_active.pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def to_bytes(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return x * scale


def to_ns(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    return x * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)


def launches(path: str) -> None:
    with open(path) as fh:
        text = fh.read()
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if "Kernel Name" in l)
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg: "OrderedDict[str, list]" = OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        agg.setdefault(name, []).append(to_ns(r[vi], r[ui]))
    total = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | total us | share |")
    print("|---|---:|---:|---:|---:|")
    for k, v in agg.items():
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / 1e3:.1f} | {sum(v) / total:.1%} |")


def traffic(path: str, n: int, out_json: str) -> None:
    import json
    import os
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, r = rows[0], rows[1], rows[2]
    rd = to_bytes(r[h.index("dram__bytes_read.sum")], u[h.index("dram__bytes_read.sum")])
    wr = to_bytes(r[h.index("dram__bytes_write.sum")], u[h.index("dram__bytes_write.sum")])
    name = r[h.index("Kernel Name")].split("(")[0] if "Kernel Name" in h else "?"
    rec = {"dram_bytes_per_hex": round((rd + wr) / n, 4),
           "source": f"{os.path.relpath(path)}: dram__bytes_read.sum {rd / 1e9:.6f} GB + dram__bytes_write.sum "
                     f"{wr / 1e6:.4f} MB for one {name} launch over {n} hexes"}
    with open(out_json, "w") as fh:
        json.dump(rec, fh)
    print(json.dumps(rec))


def full(path: str, algo: float | None) -> None:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"### {name.split('(')[0]}")
        vals = {}
        for i, k in enumerate(h):
            if k in KEYS:
                vals[k] = (r[i], u[i])
                print(f"* {k} = {r[i]} {u[i]}")
        if "dram__bytes_read.sum" in vals and "gpu__time_duration.sum" in vals:
            rd = to_bytes(*vals["dram__bytes_read.sum"])
            wr = to_bytes(*vals["dram__bytes_write.sum"])
            t = to_ns(*vals["gpu__time_duration.sum"])
            print(f"* traffic (read+write) = {rd + wr:.6e} B; achieved under ncu = {(rd + wr) / t:.1f} GB/s")
            if algo:
                print(f"* traffic / algorithmic bytes = {(rd + wr) / algo:.4f}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "traffic":
        traffic(sys.argv[2], int(sys.argv[3]), sys.argv[4])
    else:
        full(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None)
