#!/usr/bin/env python
"""Digest of a round's final run (tooling for DESIGN.md 6b): reads the bench JSON
lines under profiles/<round>/final/ and prints a markdown table of the headline
figures, so the numbers quoted in DESIGN.md can be regenerated from the logs.

usage: python tools/report.py [profiles/r01/final]
"""
from __future__ import annotations

import json
import os
import sys


def lines(path):
    if not os.path.exists(path):
        return []
    return [json.loads(l) for l in open(path) if l.strip().startswith("{")]


def kern(d, name):
    k = (d.get("roofline") or {}).get("kernel_us_cupti") or {}
    return next((v for n, v in k.items() if name in n and isinstance(v, float)), None)


def main(folder):
    rows = []
    for fname, label in [("bench.log", "config 1 (headline)"), ("bench_c0.log", "config 0"),
                         ("bench_c2.log", "config 2"), ("bench_c3.log", "config 3"), ("bench_c4.log", "config 4")]:
        for d in lines(os.path.join(folder, fname)):
            r = d["roofline"]
            p1 = r.get("pass1_us")
            sub = kern(d, "subdiv_kernel")
            note = []
            if d.get("e2e"):
                note.append(f"e2e {d['e2e']['value'] / 1e6:.0f} M/s ({d['e2e'].get('frac_of_link', 0):.2f} of link)")
            if d.get("graph"):
                note.append(f"graph {d['graph']['ms_per_step'] * 1e3:.1f} us/call")
            if d.get("cpu_baseline"):
                note.append(f"oracle {d['cpu_baseline']['value'] / 1e6:.2f} M/s on {d['cpu_baseline']['cores']} cores")
            s = d.get("subdivision") or {}
            if s.get("nodes_per_s") and s.get("nodes_per_step", 0) > 1e6:
                note.append(f"{s['nodes_per_step']:.3g} nodes at {s['nodes_per_s'] / 1e9:.1f} G nodes/s")
            rows.append((label, d["value"], d["ms_per_step"] * 1e3, p1, r.get("frac"), sub, d.get("clocks", {}), "; ".join(note)))
    print("| workload | value (hex/s) | step (us) | pass 1 (us) | frac of copy peak | subdiv (us) | SM MHz | notes |")
    print("|---|---:|---:|---:|---:|---:|---:|---|")
    for label, v, ms, p1, fr, sub, clk, note in rows:
        print(f"| {label} | {v / 1e9:.2f} G | {ms:.1f} | {p1 or 0:.1f} | {fr or 0:.3f} | {sub or 0:.1f} | "
              f"{clk.get('sm_mhz')} | {note} |")
    for fname in ("quality_c1.log", "quality_c3.log", "screen_c1.log", "screen_c3.log", "bounds_c1.log",
                  "bounds_c3.log", "bounds_c4.log", "select_c3.log", "quads.log"):
        for d in lines(os.path.join(folder, fname)):
            print(f"| {d.get('op')} {fname.split('.')[0].split('_')[-1]} | {d['value'] / 1e9:.2f} G | "
                  f"{d['ms_per_step'] * 1e3:.1f} | | {d['roofline']['frac']:.3f} | | {d.get('clocks', {}).get('sm_mhz')} | |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join("profiles", "r01", "final"))
