#!/usr/bin/env python
"""Write tests/golden/config4_oracle.npz: the CPU oracle's verdicts on all 4M hexes of config 4.

Calls only oracle/ (and the shared seeded generator hexgen/): nothing here comes from the
CUDA path.  Stored per hex: the whole flags byte, the near-boundary bit (reading G14), and
the subdivision node count (uint32; compared only for VALID hexes, reading G4).  The GPU
test tests/test_gpu_parity.py::test_config4_every_hex_against_the_oracle compares the whole
flags byte of every hex against this file.  Run time: ~13 min on 8 cores.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import hexgen  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "config4_oracle.npz")


def main():
    n = hexgen.config_size(4)
    coords, _ = hexgen.adversarial_config(n, 4)
    t0 = time.time()
    r = oracle.check_soa(coords)
    dt = time.time() - t0
    np.savez_compressed(OUT, flags=r["flags"], near=r["near"], nodes=r["nodes"].astype(np.uint32),
                        n=np.int64(n), seed=np.int64(4))
    print(f"config 4: {n} hexes in {dt:.0f} s on {oracle.num_threads(0)} threads; "
          f"flags {np.bincount(r['flags'], minlength=8).tolist()}, near {int(r['near'].sum())}, "
          f"nodes {int(r['nodes'].sum())} -> {OUT} ({os.path.getsize(OUT)} B)")


if __name__ == "__main__":
    main()
