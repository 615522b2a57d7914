"""Pins of the fp64 rounding-error bounds tau against exact rational arithmetic (-m "not gpu").

The paper is silent on floating point.  Every
near-boundary exclusion and every exact-sign fallback rests on three bounds:

* ``oracle_sample_tau`` (oracle.c ``sample_tau``): the oracle re-decides a Step-2
  sample exactly when ``|c| <= tau_c`` (reading G8), so tau_c must bound the
  oracle's own error on det J at the 27 nodes;
* ``oracle_tau_depth(E, Mb, d)``: a decision with ``|value| <= tau(d)`` marks the
  hex near-boundary (reading G14).  It is the *combined* bound: the oracle and
  the CUDA path each stay within tau/2 of the exact value, so a decision outside
  tau is the same on both sides;
* the CUDA path's Step-2 filter ``step2_tau`` (hexval_device.cuh): pass 1 treats
  a sample with ``|fl| > tau2`` as robustly signed, so tau2 must bound the
  kernel's error on the 8 corner and 12 edge-midpoint determinants.

Reference values are exact: the coordinates are dyadic rationals, so det J at
the 27 nodes (Lagrange gradients, App. A), the Bezier coefficients (Table 1 =
exact inverse of the Bernstein collocation matrix) and the de Casteljau
children are integers over a known power of two.  The CUDA path's values come
from the bit-exact emulation in tests/gpu_emulation.py (checked against the
kernels on the GPU).  Hex sets: random perturbed cubes, degenerate ones
(duplicate nodes, dyadic coplanar layers), 2^+-200-scaled ones and config-4
near-boundary hexes.
"""
from __future__ import annotations

import random

import numpy as np
import pytest

import hexgen
import oracle
from tests import gpu_emulation as gemu
from tests import pins

KAPPA = pins.KAPPA
XI2 = pins.XI2

# 8 * Table 1 as integers (exact inverse of the Bernstein collocation matrix)
_TB8 = [[int(8 * v) for v in row] for row in pins.invert_exact(pins.collocation_matrix_exact())]
assert all(8 * v == int(8 * v) for row in pins.invert_exact(pins.collocation_matrix_exact()) for v in row)
_TB8_SPARSE = [[(t, v) for t, v in enumerate(row) if v] for row in _TB8]
# 4 * dL_k/dxi_a at node sigma as integers: s_a * (2 lin_b)(2 lin_c)
_G4 = []
for _s in range(27):
    g = []
    for _k in range(8):
        two_lin = [int(XI2[_s][a]) if KAPPA[_k][a] == 1 else 2 - int(XI2[_s][a]) for a in range(3)]
        row = []
        for a in range(3):
            sg = 1 if KAPPA[_k][a] == 1 else -1
            o = [b for b in range(3) if b != a]
            row.append(sg * two_lin[o[0]] * two_lin[o[1]])
        g.append(row)
    _G4.append(g)
# layout of a node's coefficients on the (3,3,3) grid: slot i + 3j + 9k for (i, j, k) = XI2[sigma]
_SLOT = [int(XI2[s][0] + 3 * XI2[s][1] + 9 * XI2[s][2]) for s in range(27)]


def _ints(X):
    """Integer coordinates Xi and D with X = Xi / D exactly (D a power of two)."""
    fr = [[float(v).as_integer_ratio() for v in row] for row in X]
    D = max(d for row in fr for _, d in row)
    return [[n * (D // d) for n, d in row] for row in fr], D


def exact_samples(Xi):
    """det(4 J) at the 27 nodes (ints): det J(xi_sigma) = value / (64 D^3)."""
    out = []
    for s in range(27):
        J = [[sum(Xi[k][i] * _G4[s][k][a] for k in range(8)) for a in range(3)] for i in range(3)]
        out.append(J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1])
                   - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0])
                   + J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]))
    return out


def exact_bezier(C):
    """8 * Table 1 * C (ints): b_sigma = value / (512 D^3)."""
    return [sum(v * C[t] for t, v in row) for row in _TB8_SPARSE]


def exact_child(B, o):
    """Child o (Fig. 3 corner order) by de Casteljau at 1/2 per axis, xi then eta then zeta,
    on integer coefficients in Fig. 3 order; the result is scaled by 4 per axis (64 per level)."""
    G = [0] * 27
    for s in range(27):
        G[_SLOT[s]] = B[s]
    kap = [int(v) // 2 for v in XI2[o]]
    for axis in range(3):
        stride = (1, 3, 9)[axis]
        H = [0] * 27
        for base in range(27):
            if (base // stride) % 3 != 0:
                continue
            p0, p1, p2 = G[base], G[base + stride], G[base + 2 * stride]
            if kap[axis] == 0:
                q = (4 * p0, 2 * (p0 + p1), p0 + 2 * p1 + p2)
            else:
                q = (p0 + 2 * p1 + p2, 2 * (p1 + p2), 4 * p2)
            for t in range(3):
                H[base + t * stride] = q[t]
        G = H
    return [G[_SLOT[s]] for s in range(27)]


def _err(v: float, N: int, Q: int) -> float:
    """|v - N/Q| as a float (exact difference, one rounding)."""
    vn, vd = float(v).as_integer_ratio()
    return abs(vn * Q - N * vd) / (vd * Q)


# ---------------------------------------------------------------------------
# hex sets
# ---------------------------------------------------------------------------
def _random_hexes(m, amp, seed, scale=1.0):
    coords = hexgen.soa_config(m, amp, seed)
    X = hexgen.soa_to_nodes(coords)
    rng = np.random.default_rng(seed)
    off = rng.uniform(-8, 8, size=(m, 1, 3))
    return [np.ldexp(X[i] + off[i], 0) * scale for i in range(m)]


def _degenerate_hexes(m, seed):
    """Duplicate face-neighbour nodes and dyadic coordinates on coarse grids (coplanar layers):
    samples that are exactly 0 and samples within a few ulps of 0."""
    rng = random.Random(seed)
    out = []
    for q in range(m):
        X = hexgen.UNIT_CUBE.astype(np.float64).copy()
        if q % 3 == 0:
            X = X + np.array([[rng.choice([-0.25, 0, 0.25, 0.5]) for _ in range(3)] for _ in range(8)])
        elif q % 3 == 1:
            X = X + np.array([[rng.uniform(-0.3, 0.3) for _ in range(3)] for _ in range(8)])
            a = rng.randrange(8)
            b = [(1, 3, 4), (0, 2, 5), (1, 3, 6), (0, 2, 7), (0, 5, 7), (1, 4, 6), (2, 5, 7), (3, 4, 6)][a][rng.randrange(3)]
            X[b] = X[a]
        else:
            X = X + np.array([[rng.randrange(-2, 3) / 8.0 for _ in range(3)] for _ in range(8)])
            X[:, 2] = np.where(X[:, 2] > 0.5, X[:, 2], rng.choice([0.0, 0.125]))
        out.append(X)
    return out


def _config4_hexes(m):
    coords, _ = hexgen.adversarial_config(m, 4, start=1_000_000)
    X = hexgen.soa_to_nodes(coords)
    return [X[i] for i in range(m)]


@pytest.fixture(scope="module")
def hex_sets():
    return {
        "random": _random_hexes(4000, 0.35, 101),
        "random_wide": _random_hexes(1500, 0.5, 102),
        "degenerate": _degenerate_hexes(1500, 103),
        "scaled_2^+200": _random_hexes(1500, 0.4, 104, scale=2.0 ** 200),
        "scaled_2^-200": _random_hexes(1500, 0.4, 105, scale=2.0 ** -200),
        "config4": _config4_hexes(1500),
    }


# ---------------------------------------------------------------------------
# the pins
# ---------------------------------------------------------------------------
def test_tau_depth_is_cubic_in_the_edge_scale_and_linear_in_depth():
    """Dimensional check of oracle_tau_depth: det J is a cubic form of the coordinates, so
    its rounding error bound must scale as E^3 (an E-for-E^3 slip fails here), and the
    de Casteljau term grows linearly with depth times max|b|."""
    for E in (2.0 ** -200, 1e-3, 1.0, 3.7, 2.0 ** 200):
        t1, t2 = oracle.tau_depth(E, 0.0, 0), oracle.tau_depth(2 * E, 0.0, 0)
        assert t2 == pytest.approx(8 * t1, rel=1e-12)
        for d in (1, 7, 20):
            Mb = 5.0 * E ** 3
            inc = oracle.tau_depth(E, Mb, d) - oracle.tau_depth(E, Mb, 0)
            assert inc == pytest.approx(d * (oracle.tau_depth(E, Mb, 1) - oracle.tau_depth(E, Mb, 0)), rel=1e-9)
            assert inc > 0


def test_rounding_bounds_hold_against_exact_arithmetic(hex_sets):
    """|fp - exact| <= tau for every bound the parity rests on, on every hex of every set,
    with the worst observed ratio reported per set; and each bound is not vacuous (the
    worst ratio is above 1e-6 on every set, so a bound off by a power of E fails too)."""
    rng = random.Random(7)
    report = {}
    for name, hexes in hex_sets.items():
        worst = {"tau_c": 0.0, "tau2_gpu": 0.0, "root_oracle": 0.0, "root_gpu": 0.0, "child": 0.0}
        n_child = 0
        for q, X in enumerate(hexes):
            Xi, D = _ints(X)
            C = exact_samples(Xi)
            Qc = 64 * D ** 3
            r = oracle.check_hex(X)
            if r["verdict"] == oracle.NONFINITE:
                continue
            # (1) oracle samples vs tau_c (Step-2 exact fallback threshold)
            for s in range(27):
                tc = oracle.sample_tau(X, s)
                e = _err(r["c"][s], C[s], Qc)
                assert e <= tc, (name, q, s, e, tc)
                if tc > 0:
                    worst["tau_c"] = max(worst["tau_c"], e / tc)
            # (2) CUDA path's 20 samples vs its Step-2 filter bound tau2
            c, d, ekey = gemu.samples20(X)
            tau2 = gemu.step2_tau(ekey)
            for k in range(8):
                e = _err(c[k], C[k], Qc)
                assert e <= tau2, (name, q, k, e, tau2)
                worst["tau2_gpu"] = max(worst["tau2_gpu"], e / tau2)
            for k in range(12):
                e = _err(d[k], 4 * C[8 + k], Qc)            # d = 4 c_edge
                assert e <= tau2, (name, q, 8 + k, e, tau2)
                worst["tau2_gpu"] = max(worst["tau2_gpu"], e / tau2)
            # (3) root coefficients of both implementations vs tau_depth(0) / 2
            B = exact_bezier(C)
            Qb = 512 * D ** 3
            Mb = float(np.max(np.abs(r["b"])))
            t0 = oracle.tau_depth(r["E"], Mb, 0)
            bg = gemu.root_coeffs(X)
            for s in range(27):
                eo, eg = _err(r["b"][s], B[s], Qb), _err(bg[s], B[s], Qb)
                assert eo <= t0 / 2 and eg <= t0 / 2, (name, q, s, eo, eg, t0)
                worst["root_oracle"] = max(worst["root_oracle"], 2 * eo / t0)
                worst["root_gpu"] = max(worst["root_gpu"], 2 * eg / t0)
            # (4) children of the first three levels (one random path per hex, from both roots;
            # the CUDA path's de Casteljau is the oracle's up to exact power-of-two scalings)
            if q % 2 == 0:
                Bx, Q = B, Qb
                fo, fg = np.array(r["b"]), np.array(bg)
                for depth in (1, 2, 3):
                    o = rng.randrange(8)
                    Bx, Q = exact_child(Bx, o), Q * 64
                    fo, fg = oracle.subdivide(fo, o), oracle.subdivide(fg, o)
                    td = oracle.tau_depth(r["E"], Mb, depth)
                    for s in range(27):
                        eo, eg = _err(fo[s], Bx[s], Q), _err(fg[s], Bx[s], Q)
                        assert eo <= td / 2 and eg <= td / 2, (name, q, depth, s, eo, eg, td)
                        worst["child"] = max(worst["child"], 2 * max(eo, eg) / td)
                    n_child += 1
        report[name] = worst
    print("\nworst |fp - exact| / bound per hex set:")
    for name, w in report.items():
        print(f"  {name:>14}: " + ", ".join(f"{k} {v:.3g}" for k, v in w.items()))
    for name, w in report.items():
        if name == "degenerate":
            continue                        # dyadic inputs: most values are exact
        for k, v in w.items():
            assert v > 1e-6, (name, k, v)
