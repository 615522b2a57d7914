"""Bit-exact CPU emulation of the CUDA path's root arithmetic (test infrastructure only).

The CUDA kernels evaluate the 20 tetrahedron determinants, the Step-2 rounding
bound and the 27 Bezier coefficients with explicit round-to-nearest intrinsics
(``__dadd_rn``, ``__dmul_rn``, ``__fma_rn``) and ``-fmad=false``
(``paper_1706_01613_b200/csrc/hexval_device.cuh``: ``samples20``,
``step2_tau``, ``transform``, ``root_coeffs``).  This module repeats those
operations in the same order with IEEE doubles: Python's float ``+ - *`` are
correctly rounded binary64 operations, and the fused multiply-add is an exact
rational sum rounded once (CPython's int true division is correctly rounded).

It exists so that the rounding-error bound the GPU relies on (tau2 of Step 2)
can be pinned against exact arithmetic on the CPU (tests/test_tau_bounds.py);
``tests/test_gpu_parity.py::test_root_emulation_is_bit_exact`` checks on the
GPU that the emulation and the kernels agree bit for bit.  Nothing here is
imported by the product path or by the oracle.
"""
from __future__ import annotations

import math
import struct

U = 2.0 ** -53


def fma(a: float, b: float, c: float) -> float:
    """round(a*b + c) with a single rounding (IEEE fusedMultiplyAdd, round to nearest even)."""
    an, ad = a.as_integer_ratio()
    bn, bd = b.as_integer_ratio()
    cn, cd = c.as_integer_ratio()
    num = an * bn * cd + cn * ad * bd
    den = ad * bd * cd
    if num == 0:
        # exact zero: +0 under round-to-nearest unless a*b and c are both -0
        prod_neg_zero = (a == 0 or b == 0) and (math.copysign(1.0, a) * math.copysign(1.0, b) < 0)
        return -0.0 if (prod_neg_zero and math.copysign(1.0, c) < 0) else 0.0
    return num / den


def hiword(x: float) -> int:
    """High 32 bits of a double as a signed int (hexval_device.cuh key())."""
    return struct.unpack("<q", struct.pack("<d", x))[0] >> 32


def abskey(x: float) -> int:
    return hiword(x) & 0x7FFFFFFF


def from_words(hi: int, lo: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", ((hi & 0xFFFFFFFF) << 32) | (lo & 0xFFFFFFFF)))[0]


def _sub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def _add(a, b):
    return (a[0] + b[0], a[1] + b[1], a[2] + b[2])


def det3(a, b, c) -> float:
    """hexval_device.cuh det3: a . (b x c) with three FMAs per cross component order."""
    wx = fma(b[1], c[2], -(b[2] * c[1]))
    wy = fma(b[2], c[0], -(b[0] * c[2]))
    wz = fma(b[0], c[1], -(b[1] * c[0]))
    return fma(a[2], wz, fma(a[1], wy, a[0] * wx))


def edge_vectors(X):
    """The 12 edge vectors in samples20 order: v12 v43 v56 v87 v14 v23 v58 v67 v15 v26 v48 v37."""
    n = [tuple(float(v) for v in X[k]) for k in range(8)]
    pairs = [(1, 0), (2, 3), (5, 4), (6, 7), (3, 0), (2, 1), (7, 4), (6, 5), (4, 0), (5, 1), (7, 3), (6, 2)]
    return [_sub(n[j], n[i]) for j, i in pairs]


def samples20(X):
    """(c[8], d[12], ekey): corner dets, 4 x edge-midpoint dets, hi word of max |edge component|."""
    v12, v43, v56, v87, v14, v23, v58, v67, v15, v26, v48, v37 = edge_vectors(X)
    e = 0
    for v in (v12, v43, v56, v87, v14, v23, v58, v67, v15, v26, v48, v37):
        for x in v:
            e = max(e, abskey(x))
    c = [det3(v12, v14, v15), det3(v12, v23, v26), det3(v43, v23, v37), det3(v43, v14, v48),
         det3(v56, v58, v15), det3(v56, v67, v26), det3(v87, v67, v37), det3(v87, v58, v48)]
    Se0, Se1 = _add(v14, v23), _add(v58, v67)
    Sz0, Sz1 = _add(v15, v26), _add(v48, v37)
    Tx0, Tx1 = _add(v12, v43), _add(v56, v87)
    Tz0, Tz1 = _add(v15, v48), _add(v26, v37)
    Ux0, Ux1 = _add(v12, v56), _add(v43, v87)
    Ue0, Ue1 = _add(v14, v58), _add(v23, v67)
    d = [det3(v12, Se0, Sz0), det3(Tx0, v23, Tz1), det3(v43, Se0, Sz1), det3(Tx0, v14, Tz0),
         det3(Ux0, Ue0, v15), det3(Ux0, Ue1, v26), det3(Ux1, Ue1, v37), det3(Ux1, Ue0, v48),
         det3(v56, Se1, Sz0), det3(Tx1, v67, Tz1), det3(v87, Se1, Sz1), det3(Tx1, v58, Tz0)]
    return c, d, e


def step2_tau(ekey: int) -> float:
    """hexval_device.cuh step2_tau: 512 u E^3 with E an upper key of max |edge component| + underflow term."""
    E = from_words(ekey, 0xFFFFFFFF)
    E2 = E * E
    t = ((512.0 * U) * E2) * E
    return fma(8.7e-317, 1.0 + E2, t)


def transform(c, d):
    """hexval_device.cuh transform: (e2[12], f4[6], z8) = (2 b_edge, 4 b_face, 8 b_centre)."""
    ends = [(0, 1), (1, 2), (2, 3), (0, 3), (0, 4), (1, 5), (2, 6), (3, 7), (4, 5), (5, 6), (6, 7), (4, 7)]
    e2 = [(d[k] - c[a]) - c[b] for k, (a, b) in enumerate(ends)]
    p01, p23, p45, p67 = c[0] + c[1], c[2] + c[3], c[4] + c[5], c[6] + c[7]
    C21, C26 = p01 + p23, p45 + p67
    C22, C24 = p01 + p45, p23 + p67
    C23 = (c[1] + c[2]) + (c[5] + c[6])
    C25 = (c[0] + c[3]) + (c[4] + c[7])
    s45, s67 = d[4] + d[5], d[6] + d[7]
    D21 = (d[0] + d[1]) + (d[2] + d[3])
    D26 = (d[8] + d[9]) + (d[10] + d[11])
    D22 = (d[0] + d[8]) + s45
    D24 = (d[2] + d[10]) + s67
    D23 = (d[1] + d[9]) + (d[5] + d[6])
    D25 = (d[3] + d[11]) + (d[4] + d[7])
    f4 = [fma(-3.0, C21, D21), fma(-3.0, C22, D22), fma(-3.0, C23, D23),
          fma(-3.0, C24, D24), fma(-3.0, C25, D25), fma(-3.0, C26, D26)]
    Dall = (D21 + D26) + (s45 + s67)
    Call = C21 + C26
    z8 = fma(-5.0, Call, Dall)
    return e2, f4, z8


def root_coeffs(X):
    """The 27 root Bezier coefficients in Fig. 3 order as the CUDA path computes them
    (the values hexval_check_* writes to coeffs_out)."""
    c, d, _ = samples20(X)
    e2, f4, z8 = transform(c, d)
    return list(c) + [0.5 * v for v in e2] + [0.25 * v for v in f4] + [0.125 * z8]
