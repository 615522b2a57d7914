"""Independent reference computations used by the tests to pin the oracle.

Nothing here is imported by the oracle or by the CUDA path.  Each function is
written from the paper's definitions with a different formulation from the
oracle's where one exists:

* the trilinear map through its Lagrange shape functions (App. A,
  PAPER.md:1360-1378) and their gradients, det J via numpy's determinant
  (the oracle uses the section 5 edge-vector derivatives and a Leibniz sum);
* Bernstein polynomials straight from PAPER.md:461-470;
* exact rationals with ``fractions.Fraction`` (the oracle uses a C bigint).
"""
from __future__ import annotations

import os
from fractions import Fraction
from math import comb

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# Fig. 3 node / coefficient order as 2*xi
XI2 = np.array([
    (0, 0, 0), (2, 0, 0), (2, 2, 0), (0, 2, 0), (0, 0, 2), (2, 0, 2), (2, 2, 2), (0, 2, 2),
    (1, 0, 0), (2, 1, 0), (1, 2, 0), (0, 1, 0), (0, 0, 1), (2, 0, 1), (2, 2, 1), (0, 2, 1),
    (1, 0, 2), (2, 1, 2), (1, 2, 2), (0, 1, 2),
    (1, 1, 0), (1, 0, 1), (2, 1, 1), (1, 2, 1), (0, 1, 1), (1, 1, 2), (1, 1, 1)], dtype=np.int64)
KAPPA = XI2[:8] // 2          # reference corners of nodes 1..8


def load_golden(name: str):
    """Return (X (8,3), expect dict) from tests/golden/<name>.txt."""
    path = os.path.join(GOLDEN_DIR, name + ".txt")
    rows, expect = [], {}
    with open(path) as fh:
        for line in fh:
            line = line.strip()
            if line.startswith("# expect:"):
                for tok in line[len("# expect:"):].split():
                    k, v = tok.split("=")
                    expect[k] = v
                continue
            if not line or line.startswith("#"):
                continue
            rows.append([float(t) for t in line.split()])
    X = np.array(rows, dtype=np.float64)
    assert X.shape == (8, 3)
    return X, expect


# ---------------------------------------------------------------------------
# trilinear map via shape functions (App. A) -> Jacobian matrix -> det
# ---------------------------------------------------------------------------

def shape_gradients(xi: np.ndarray) -> np.ndarray:
    """dL_k/dxi_a for the 8 App. A shape functions at points xi (..., 3) -> (..., 8, 3)."""
    xi = np.asarray(xi, dtype=np.float64)
    lin = np.where(KAPPA[None, :, :] == 1, xi[..., None, :], 1.0 - xi[..., None, :])  # (...,8,3)
    sgn = np.where(KAPPA == 1, 1.0, -1.0)                                             # (8,3)
    g = np.empty(lin.shape)
    for a in range(3):
        others = [b for b in range(3) if b != a]
        g[..., a] = sgn[:, a] * lin[..., others[0]] * lin[..., others[1]]
    return g


def jacobian(X: np.ndarray, xi: np.ndarray) -> np.ndarray:
    """J_ij = dx_i/dxi_j at points xi (..., 3) -> (..., 3, 3)."""
    g = shape_gradients(xi)
    return np.einsum("ki,...kj->...ij", X, g)


def detj(X: np.ndarray, xi: np.ndarray) -> np.ndarray:
    return np.linalg.det(jacobian(X, xi))


def grid_points(m: int) -> np.ndarray:
    t = np.linspace(0.0, 1.0, m + 1)
    P = np.stack(np.meshgrid(t, t, t, indexing="ij"), axis=-1)
    return P.reshape(-1, 3)


# ---------------------------------------------------------------------------
# Bernstein basis
# ---------------------------------------------------------------------------

def bernstein(n: int, k: int, t):
    return comb(n, k) * t ** k * (1 - t) ** (n - k)


def bezier_eval(b: np.ndarray, xi: np.ndarray) -> np.ndarray:
    xi = np.atleast_2d(xi)
    out = np.zeros(xi.shape[0])
    for s in range(27):
        i, j, k = XI2[s]
        out += b[s] * bernstein(2, i, xi[:, 0]) * bernstein(2, j, xi[:, 1]) * bernstein(2, k, xi[:, 2])
    return out


def collocation_matrix_exact():
    """A[sigma][tau] = B_tau(xi_sigma) in exact rationals."""
    A = []
    for s in range(27):
        xs = [Fraction(int(v), 2) for v in XI2[s]]
        row = []
        for t in range(27):
            i, j, k = (int(v) for v in XI2[t])
            row.append(bernstein(2, i, xs[0]) * bernstein(2, j, xs[1]) * bernstein(2, k, xs[2]))
        A.append(row)
    return A


def invert_exact(A):
    """Gauss-Jordan over Fractions."""
    n = len(A)
    M = [list(map(Fraction, row)) + [Fraction(int(i == j)) for j in range(n)] for i, row in enumerate(A)]
    for col in range(n):
        piv = next(r for r in range(col, n) if M[r][col] != 0)
        M[col], M[piv] = M[piv], M[col]
        p = M[col][col]
        M[col] = [v / p for v in M[col]]
        for r in range(n):
            if r != col and M[r][col] != 0:
                f = M[r][col]
                M[r] = [a - f * b for a, b in zip(M[r], M[col])]
    return [row[n:] for row in M]


# ---------------------------------------------------------------------------
# exact det J at a node (Fractions; Lagrange gradients)
# ---------------------------------------------------------------------------

def detj_exact(X: np.ndarray, sigma: int) -> Fraction:
    xi = [Fraction(int(v), 2) for v in XI2[sigma]]
    J = [[Fraction(0)] * 3 for _ in range(3)]
    for k in range(8):
        kap = KAPPA[k]
        lin = [xi[a] if kap[a] == 1 else 1 - xi[a] for a in range(3)]
        for a in range(3):
            s = 1 if kap[a] == 1 else -1
            others = [b for b in range(3) if b != a]
            g = s * lin[others[0]] * lin[others[1]]
            for i in range(3):
                J[i][a] += Fraction(float(X[k, i])) * g
    return (J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1])
            - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0])
            + J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]))


# ---------------------------------------------------------------------------
# Table 3 and Table 2 transcribed
# ---------------------------------------------------------------------------

EDGES = [(1, 2), (2, 3), (3, 4), (1, 4), (1, 5), (2, 6), (3, 7), (4, 8), (5, 6), (6, 7), (7, 8), (5, 8)]
FACE_CORNERS = [(1, 2, 3, 4), (1, 2, 5, 6), (2, 3, 6, 7), (3, 4, 7, 8), (1, 4, 5, 8), (5, 6, 7, 8)]
FACE_EDGES = [(9, 10, 11, 12), (9, 13, 14, 17), (10, 14, 15, 18), (11, 15, 16, 19), (12, 13, 16, 20),
              (17, 18, 19, 20)]


def table3_exact():
    """T-tilde (27x20) as printed in Table 3."""
    T = [[Fraction(0)] * 20 for _ in range(27)]
    for k in range(8):
        T[k][k] = Fraction(1)
    for e, (a, b) in enumerate(EDGES):
        T[8 + e][a - 1] = Fraction(-1, 2)
        T[8 + e][b - 1] = Fraction(-1, 2)
        T[8 + e][8 + e] = Fraction(2)
    for f in range(6):
        for q in range(4):
            T[20 + f][FACE_CORNERS[f][q] - 1] = Fraction(-3, 4)
            T[20 + f][FACE_EDGES[f][q] - 1] = Fraction(1)
    for k in range(8):
        T[26][k] = Fraction(-5, 8)
    for e in range(8, 20):
        T[26][e] = Fraction(1, 2)
    return T


def table2_printed_exact():
    """The 7x20 block of Table 2 exactly as printed (b_21..27 from b_1..20)."""
    T = [[Fraction(0)] * 20 for _ in range(7)]
    for f in range(6):
        for q in range(4):
            T[f][FACE_CORNERS[f][q] - 1] = Fraction(1, 4)
            T[f][FACE_EDGES[f][q] - 1] = Fraction(-1, 2)
    for k in range(8):
        T[6][k] = Fraction(1, 4)
    for e in range(8, 20):
        T[6][e] = Fraction(-1, 4)
    return T


def corner_scaled_jacobian(X: np.ndarray) -> float:
    """min over corners of det(e1,e2,e3)/(|e1||e2||e3|) with the 3 corner edges."""
    vals = []
    for k in range(8):
        kap = KAPPA[k]
        edges = []
        for a in range(3):
            nb = kap.copy()
            nb[a] = 1 - nb[a]
            j = int(np.nonzero((KAPPA == nb).all(axis=1))[0][0])
            e = X[j] - X[k]
            edges.append(e if kap[a] == 0 else -e)
        M = np.array(edges).T
        vals.append(np.linalg.det(M) / np.prod([np.linalg.norm(e) for e in edges]))
    return float(min(vals))


def tet_det(p0, p1, p2, p3) -> float:
    """det(p1-p0, p2-p0, p3-p0) = 6 * signed volume."""
    return float(np.linalg.det(np.array([p1 - p0, p2 - p0, p3 - p0]).T))


# Two 5-tet decompositions of the hexahedron (1-based nodes).
TETS_A = [(3, 1, 6, 8), (1, 2, 3, 6), (4, 1, 3, 8), (1, 5, 6, 8), (7, 3, 6, 8)]
TETS_B = [(2, 4, 5, 7), (1, 2, 4, 5), (2, 3, 4, 7), (6, 2, 5, 7), (4, 8, 5, 7)]


def volume_10_tets(X: np.ndarray) -> float:
    va = sum(tet_det(*(X[i - 1] for i in t)) for t in TETS_A) / 6.0
    vb = sum(tet_det(*(X[i - 1] for i in t)) for t in TETS_B) / 6.0
    return 0.5 * (va + vb)


def volume_quadrature(X: np.ndarray, order: int = 4) -> float:
    """Gauss-Legendre quadrature of det J over [0,1]^3 (exact for triquadratics with order >= 2)."""
    x, w = np.polynomial.legendre.leggauss(order)
    x = 0.5 * (x + 1.0)
    w = 0.5 * w
    P = np.stack(np.meshgrid(x, x, x, indexing="ij"), axis=-1).reshape(-1, 3)
    W = np.einsum("i,j,k->ijk", w, w, w).ravel()
    return float(np.sum(W * detj(X, P)))


def random_hexes(n: int, amp: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    U = KAPPA.astype(np.float64)
    return U[None] + rng.uniform(-amp, amp, size=(n, 8, 3))
