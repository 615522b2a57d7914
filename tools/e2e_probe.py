#!/usr/bin/env python
"""End-to-end (host buffers) rate of hexval_check_soa_host against the PCIe link
(tooling for profiles/; GPU only): the plain pinned->device copy rate of the
same bytes, and the e2e rate for several chunk sizes.  Prints one JSON object."""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    import paper_1706_01613_b200 as hv

    _, n, host = bench.make_inputs(1, 0)
    pin = torch.from_numpy(host[0]).pin_memory()
    fl = torch.empty(n, dtype=torch.uint8).pin_memory()
    dev = torch.empty(pin.shape, dtype=pin.dtype, device="cuda")
    out = {"n": n, "bytes": pin.numel() * 8}
    rates = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(pin, non_blocking=True)
        torch.cuda.synchronize()
        rates.append(pin.numel() * 8 / (time.perf_counter() - t0) / 1e9)
    out["link_h2d_gbs_one_copy"] = max(rates)
    del dev
    torch.cuda.empty_cache()
    for chunk in (1 << 19, 1 << 20, 1 << 21, 1 << 22, 1 << 23):
        hv.check_soa_host(pin, fl, chunk_hexes=chunk)
        t0 = time.perf_counter()
        for _ in range(3):
            hv.check_soa_host(pin, fl, chunk_hexes=chunk)
        dt = (time.perf_counter() - t0) / 3
        out[f"chunk_{chunk}"] = {"hex_per_s": n / dt, "h2d_gbs": pin.numel() * 8 / dt / 1e9}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
