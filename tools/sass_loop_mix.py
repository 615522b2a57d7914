#!/usr/bin/env python
"""Static instruction mix of a kernel's hot loop (tooling): the span of the backward
branch that encloses a marker instruction (default: the K4 stack pop, a 256-bit LDG).
Usage: python tools/sass_loop_mix.py LIB.so KERNEL_SUBSTRING [MARKER_REGEX]"""
import collections
import re
import subprocess
import sys


def main():
    lib, kname = sys.argv[1], sys.argv[2]
    marker = re.compile(sys.argv[3] if len(sys.argv) > 3 else r"LDG\.E.*\.256")
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = out.split("Function : ")
    body = next(f for f in funcs[1:] if kname in f.splitlines()[0])
    ins = []
    for line in body.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    mark = next(a for a, t in ins if marker.search(t))
    best = None
    for a, t in ins:
        m = re.search(r"BRA\s+(?:`\()?0x([0-9a-f]+)", t)
        if m:
            tgt = int(m.group(1), 16)
            if tgt <= mark <= a and (best is None or a - tgt > best[1] - best[0]):
                best = (tgt, a)
    lo, hi = best
    cnt = collections.Counter()
    for a, t in ins:
        if lo <= a <= hi:
            op = t.split()[0]
            if op.startswith("@"):
                op = t.split()[1]
            cnt[op.split(".")[0]] += 1
    tot = sum(cnt.values())
    print(f"loop 0x{lo:x}..0x{hi:x}: {tot} instructions")
    for k, v in cnt.most_common(25):
        print(f"  {k:10s} {v}")


if __name__ == "__main__":
    main()
