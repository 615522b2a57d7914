#!/usr/bin/env python
"""Host-side cost of one small call (config 0, 10k hexes): the Python binding, a
direct ctypes call with cached pointers, and the bare device time (tooling for
profiles/; GPU only).  Prints one JSON object (microseconds per call)."""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def per_call(fn, reps=2000):
    import torch
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t_host = (time.perf_counter() - t0) / reps
    torch.cuda.synchronize()
    t_all = (time.perf_counter() - t0) / reps
    return t_host * 1e6, t_all * 1e6


def main():
    import torch
    import bench
    import paper_1706_01613_b200 as hv
    _, n, host = bench.make_inputs(0, 0)
    dev = torch.from_numpy(host[0]).cuda()
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    L = hv.lib()
    cp, fp = dev.data_ptr(), flags.data_ptr()
    s = torch.cuda.current_stream().cuda_stream
    out = {"n": n}
    out["binding_enqueue_us"], out["binding_total_us"] = per_call(lambda: hv.check_soa(dev, flags=flags))
    out["ctypes_enqueue_us"], out["ctypes_total_us"] = per_call(lambda: L.hexval_check_soa(cp, n, fp, None, s))
    out["current_stream_us"], _ = per_call(lambda: torch.cuda.current_stream().cuda_stream)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
