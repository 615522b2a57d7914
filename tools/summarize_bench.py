#!/usr/bin/env python
"""Markdown table of bench.py JSON lines (tooling for profiles/).  usage: summarize_bench.py LOG..."""
from __future__ import annotations

import json
import os
import sys


def rows(path):
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            yield json.loads(line)


def main(paths):
    print("| log | op / config | value | ms/step | roofline (achieved / peak) | frac | notes |")
    print("|---|---|---:|---:|---|---:|---|")
    for p in paths:
        for d in rows(p):
            r = d.get("roofline") or {}
            op = d.get("op", "check")
            cfg = (d.get("config") or {}).get("workload", "")[:40]
            notes = []
            ph = r.get("kernel_us_cupti") or {}
            if any(isinstance(v, float) for v in ph.values()):
                notes.append("kernels us: " + ", ".join(f"{k} {v:.1f}" for k, v in ph.items() if isinstance(v, float)))
            elif op == "check":
                ph = r.get("phase_ms_per_step", {})
                notes.append("phases us: " + ", ".join(f"{k} {v * 1e3:.1f}" for k, v in ph.items()))
            if op == "check":
                sub = d.get("subdivision") or {}
                if sub.get("nodes_per_s"):
                    notes.append(f"{sub['nodes_per_step']:.3g} nodes, {sub['nodes_per_s'] / 1e9:.2f} G nodes/s")
                if d.get("e2e"):
                    notes.append(f"e2e {d['e2e']['value'] / 1e6:.0f} M/s")
                if d.get("cpu_baseline"):
                    notes.append(f"oracle {d['cpu_baseline']['value'] / 1e6:.2f} M/s on {d['cpu_baseline']['cores']} cores")
            for k in ("nodes_per_step", "capped", "n_valid", "rel_tol"):
                if k in d:
                    notes.append(f"{k} {d[k]}")
            clk = d.get("clocks") or {}
            if clk.get("sm_mhz"):
                notes.append(f"SM {clk['sm_mhz']} MHz {','.join(clk.get('reasons', [])) or 'no throttle'}")
            print(f"| {os.path.basename(p)} | {op} / {cfg} | {d['value'] / 1e9:.3f} G/s | {d['ms_per_step']:.4f} | "
                  f"{r.get('achieved', 0):.0f} / {r.get('peak', 0):.0f} {r.get('unit', '')} | {r.get('frac', 0):.3f} | "
                  f"{'; '.join(notes)} |")


if __name__ == "__main__":
    main(sys.argv[1:])
