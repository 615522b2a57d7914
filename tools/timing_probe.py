#!/usr/bin/env python
"""Where does a check call's step time go?  (tooling for profiles/; GPU only)

Runs the config-1 workload through hexval_check_soa four ways and prints one
JSON object:
  clean      K back-to-back calls bracketed by two CUDA events (the headline)
  profiled   the same with the library's per-kernel events (hexval_profile)
  per_call   a pair of CUDA events around every call
  cupti      torch.profiler (CUPTI activity records) kernel durations and the
             gaps between consecutive GPU activities of the clean loop
usage: python tools/timing_probe.py [--config 1] [--steps 50]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    import torch
    import bench
    import paper_1706_01613_b200 as hv

    layout, n, host = bench.make_inputs(a.config, 0)
    dev = [torch.from_numpy(x).cuda() for x in host]
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()

    def step(profile=None):
        if layout == "soa":
            hv.check_soa(dev[0], flags=flags, profile=profile)
        else:
            hv.check_indexed(dev[0], dev[1], flags=flags, profile=profile)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    out = {"config": a.config, "n": n, "steps": a.steps}

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.steps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    out["clean_us_per_step"] = e0.elapsed_time(e1) * 1e3 / a.steps

    prof = hv.Profile()
    prof.read()
    e0.record(s)
    for _ in range(a.steps):
        step(profile=prof)
    e1.record(s)
    torch.cuda.synchronize()
    out["profiled_us_per_step"] = e0.elapsed_time(e1) * 1e3 / a.steps
    out["profiled_phases_us"] = {k: v["ms"] * 1e3 / max(1, v["launches"]) for k, v in prof.read().items()}

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    for b, e in evs:
        b.record(s)
        step()
        e.record(s)
    torch.cuda.synchronize()
    out["per_call_event_us"] = sum(b.elapsed_time(e) for b, e in evs) * 1e3 / a.steps

    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        for _ in range(a.steps):
            step()
        torch.cuda.synchronize()
    acts = []
    for ev in p.events():
        if ev.device_type.name == "CUDA":
            acts.append((ev.time_range.start, ev.time_range.end, ev.name))
    acts.sort()
    per = {}
    for t0, t1, name in acts:
        key = name.split("<")[0].split("::")[-1].strip()[-40:]
        d = per.setdefault(key, [0, 0.0])
        d[0] += 1
        d[1] += t1 - t0
    out["cupti_kernels_us"] = {k: {"count": c, "mean_us": tot / c} for k, (c, tot) in per.items()}
    gaps = [acts[i + 1][0] - acts[i][1] for i in range(len(acts) - 1)]
    if acts:
        out["cupti_span_us_per_step"] = (acts[-1][1] - acts[0][0]) / a.steps
        out["cupti_gap_us_mean"] = sum(gaps) / max(1, len(gaps))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
