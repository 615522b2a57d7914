#!/usr/bin/env python
"""Validate a hexahedral mesh on the GPU: validity flags, Ushakova's Test 1 and the
minimum corner scaled Jacobian in one pass, plus certified bounds on min det J for
the elements that are not valid.

  python examples/check_mesh.py                       # a jittered 100^3 structured mesh
  python examples/check_mesh.py mesh.npz              # arrays `vertices` (nv, 3) float64,
                                                      # `hex_idx` (n, 8) int32, Fig. 3 node order
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def jittered_grid(m: int = 100, jitter: float = 0.3, seed: int = 0):
    rng = np.random.default_rng(seed)
    g = np.stack(np.meshgrid(np.arange(m + 1), np.arange(m + 1), np.arange(m + 1), indexing="ij"), -1)
    verts = (g.reshape(-1, 3)[:, ::-1] + rng.uniform(-jitter, jitter, ((m + 1) ** 3, 3))).astype(np.float64)
    i, j, k = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    vid = lambda a, b, c: a + (m + 1) * (b + (m + 1) * c)                    # noqa: E731
    idx = np.stack([vid(i, j, k), vid(i + 1, j, k), vid(i + 1, j + 1, k), vid(i, j + 1, k),
                    vid(i, j, k + 1), vid(i + 1, j, k + 1), vid(i + 1, j + 1, k + 1), vid(i, j + 1, k + 1)], 1)
    return verts, idx.astype(np.int32)


def main(argv):
    import torch
    import paper_1706_01613_b200 as hv

    if len(argv) > 1:
        z = np.load(argv[1])
        verts, idx = np.ascontiguousarray(z["vertices"], np.float64), np.ascontiguousarray(z["hex_idx"], np.int32)
    else:
        verts, idx = jittered_grid()
    v, x = torch.from_numpy(verts).cuda(), torch.from_numpy(idx).cuda()
    hv.check_screen_indexed(v, x)                                          # warm-up (device setup)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    flags, sj, t1 = hv.check_screen_indexed(v, x)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    verdict = (flags & 3).cpu().numpy()
    names = {hv.INVALID: "invalid", hv.VALID: "valid", hv.UNDETERMINED: "undetermined", hv.NONFINITE: "nonfinite"}
    n = idx.shape[0]
    print(f"{n} hexahedra in {dt * 1e3:.2f} ms ({n / dt / 1e9:.2f} G hex/s)")
    for code, name in names.items():
        print(f"  {name:13s} {int((verdict == code).sum())}")
    print(f"  subdivided    {int(((flags & hv.FLAG_SUBDIVIDED) > 0).sum().item())}")
    t1_fail_valid = int(((t1 == 0) & ((flags & 3) == hv.VALID)).sum().item())
    print(f"  Test 1 fails on {int((t1 == 0).sum().item())} (on valid ones: {t1_fail_valid}, must be 0)")
    ok = (flags & 3) == hv.VALID
    if ok.any():
        print(f"  min corner scaled Jacobian over valid hexes: {float(sj[ok].min()):.4g}")
    bad = torch.nonzero((flags & 3) != hv.VALID).flatten()
    if bad.numel():
        sub = x[bad.to(torch.int64)].contiguous()
        lo, up, _ = hv.min_detj_bounds_indexed(v, sub, 1e-3)
        torch.cuda.synchronize()
        k = int(torch.argmin(up).item())
        print(f"  most negative element {int(bad[k])}: min det J in [{float(lo[k]):.4g}, {float(up[k]):.4g}]")
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv))
