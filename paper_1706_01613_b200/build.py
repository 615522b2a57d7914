"""Build libhexval.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "hexval.cu")
SRC_DIAG = os.path.join(HERE, "csrc", "diag.cu")      # roofline probes (not the hot path)
DEPS = [SRC, SRC_DIAG, os.path.join(HERE, "csrc", "hexval_device.cuh"), os.path.join(HERE, "csrc", "scratch.cuh"),
        os.path.join(ROOT, "include", "hexval.h")]
LIB = os.path.join(HERE, "libhexval.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-fmad=false",                 # every FMA is explicit (__fma_rn): bit-identical recomputation
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-O2",
    "-shared", "-cudart", "static",
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libhexval.so (or, for A/B measurements, a variant with extra -D defines at `out`)."""
    target = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-o", target, SRC, SRC_DIAG]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode}); see {log}")
    if verbose:
        sys.stdout.write(res.stderr)
    return target


DEBUG_LIB = os.path.join(HERE, "libhexval_debug.so")


# invariant traps + the smallest practical K4 stack capacity: the capacity-adaptive pop size runs in
# its one-node mode on inputs the default capacity never throttles (tests/test_gpu_parity.py)
SMALLCAP_LIB = os.path.join(HERE, "libhexval_smallcap.so")


def build_all(force: bool = False) -> list[str]:
    """The product library and its test variants (used by the GPU tests): HEXVAL_DEBUG invariant
    traps, and the same with a 416-slot K4 stack."""
    out = [build(force=force)]
    for lib, defines in ((DEBUG_LIB, ("HEXVAL_DEBUG",)), (SMALLCAP_LIB, ("HEXVAL_DEBUG", "HEXVAL_K4_CAP=416"))):
        if force or not os.path.exists(lib) or any(os.path.getmtime(d) > os.path.getmtime(lib) for d in DEPS):
            out.append(build(out=lib, defines=defines))
        else:
            out.append(lib)
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--out", default=None, help="variant library path (A/B builds)")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=True, out=a.out, defines=a.defines))
