"""CPU oracle for the robust validity of linear hexahedra (section 6).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
this package.  The product path (``paper_1706_01613_b200``) never imports or
calls it, and the two share no code: see ``oracle.c`` for what is computed and
DESIGN.md for the readings of the paper it follows.

This module is ctypes marshalling only; every step of the algorithm runs in
``liboracle.so`` (plain C, built by :func:`build`).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.c")

INVALID, VALID, UNDETERMINED, NONFINITE = 0, 1, 2, 3
FLAG_SUBDIVIDED = 4
MAX_DEPTH = 20


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -ffp-contract=off, OpenMP)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-Wall",
               "-shared", "-fPIC", SRC, "-o", LIB_PATH, "-lm"]
        subprocess.run(cmd, check=True)
    return LIB_PATH


class OracleResult(ctypes.Structure):
    _fields_ = [
        ("verdict", ctypes.c_int),
        ("subdivided", ctypes.c_int),
        ("flags", ctypes.c_int),
        ("exact_used", ctypes.c_int),
        ("near_boundary", ctypes.c_int),
        ("max_depth", ctypes.c_int),
        ("nodes", ctypes.c_int64),
        ("margin_ratio", ctypes.c_double),
        ("E", ctypes.c_double),
        ("c", ctypes.c_double * 27),
        ("b", ctypes.c_double * 27),
        ("witness", ctypes.c_double * 3),
        ("witness_value", ctypes.c_double),
    ]

    def as_dict(self):
        return {
            "verdict": self.verdict, "subdivided": self.subdivided, "flags": self.flags,
            "exact_used": self.exact_used, "near_boundary": self.near_boundary,
            "max_depth": self.max_depth, "nodes": self.nodes,
            "margin_ratio": self.margin_ratio, "E": self.E,
            "c": np.array(self.c[:]), "b": np.array(self.b[:]),
            "witness": np.array(self.witness[:]), "witness_value": self.witness_value,
        }


class OracleBounds(ctypes.Structure):
    _fields_ = [("lower", ctypes.c_double), ("upper", ctypes.c_double), ("tol", ctypes.c_double),
                ("capped", ctypes.c_int), ("nodes", ctypes.c_int64)]


_lib = None
_D = ctypes.POINTER(ctypes.c_double)


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_check_hex.argtypes = [_D, ctypes.POINTER(OracleResult)]
        L.oracle_check_hex.restype = ctypes.c_int
        L.oracle_check_soa.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_check_soa.restype = None
        L.oracle_check_indexed.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_int]
        L.oracle_check_indexed.restype = None
        L.oracle_detj.argtypes = [_D, _D]
        L.oracle_detj.restype = ctypes.c_double
        L.oracle_samples27.argtypes = [_D, _D]
        L.oracle_bezier_from_samples.argtypes = [_D, _D]
        L.oracle_tb_matrix.argtypes = [_D]
        L.oracle_bezier_eval.argtypes = [_D, _D]
        L.oracle_bezier_eval.restype = ctypes.c_double
        L.oracle_subdivide.argtypes = [_D, ctypes.c_int, _D]
        L.oracle_exact_sign.argtypes = [_D, ctypes.c_int]
        L.oracle_exact_sign.restype = ctypes.c_int
        L.oracle_node_xi.argtypes = [ctypes.c_int, _D]
        L.oracle_classify_coeffs.argtypes = [_D, ctypes.c_double, ctypes.POINTER(OracleResult)]
        L.oracle_classify_coeffs.restype = ctypes.c_int
        L.oracle_corner_quality.argtypes = [_D, _D, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        L.oracle_corner_quality.restype = None
        L.oracle_corner_quality_soa.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_int]
        L.oracle_corner_quality_soa.restype = None
        L.oracle_corner_quality_indexed.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_corner_quality_indexed.restype = None
        L.oracle_min_detj_bounds.argtypes = [_D, ctypes.c_double, ctypes.POINTER(OracleBounds)]
        L.oracle_min_detj_bounds.restype = None
        L.oracle_min_detj_bounds_soa.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p,
                                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_min_detj_bounds_soa.restype = None
        L.oracle_check_quad.argtypes = [_D, _D, ctypes.POINTER(ctypes.c_int)]
        L.oracle_check_quad.restype = ctypes.c_int
        L.oracle_exact_orient2d.argtypes = [_D, _D, _D]
        L.oracle_exact_orient2d.restype = ctypes.c_int
        L.oracle_check_quad_soa.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_int]
        L.oracle_check_quad_soa.restype = None
        L.oracle_sample_tau.argtypes = [_D, ctypes.c_int]
        L.oracle_sample_tau.restype = ctypes.c_double
        L.oracle_tau_depth.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int]
        L.oracle_tau_depth.restype = ctypes.c_double
        L.oracle_num_threads.argtypes = [ctypes.c_int]
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _hex(X) -> np.ndarray:
    X = np.ascontiguousarray(np.asarray(X, dtype=np.float64).reshape(8, 3))
    return X


def check_hex(X) -> dict:
    """Run the whole algorithm on one hex (8x3 nodes in Fig. 3 order)."""
    X = _hex(X)
    r = OracleResult()
    lib().oracle_check_hex(_dptr(X), ctypes.byref(r))
    return r.as_dict()


def detj(X, xi) -> float:
    X = _hex(X)
    xi = np.ascontiguousarray(np.asarray(xi, dtype=np.float64))
    return lib().oracle_detj(_dptr(X), _dptr(xi))


def samples27(X) -> np.ndarray:
    X = _hex(X)
    c = np.zeros(27)
    lib().oracle_samples27(_dptr(X), _dptr(c))
    return c


def bezier_from_samples(c) -> np.ndarray:
    c = np.ascontiguousarray(np.asarray(c, dtype=np.float64))
    b = np.zeros(27)
    lib().oracle_bezier_from_samples(_dptr(c), _dptr(b))
    return b


def tb_matrix() -> np.ndarray:
    T = np.zeros((27, 27))
    lib().oracle_tb_matrix(_dptr(T))
    return T


def bezier_eval(b, xi) -> float:
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    xi = np.ascontiguousarray(np.asarray(xi, dtype=np.float64))
    return lib().oracle_bezier_eval(_dptr(b), _dptr(xi))


def subdivide(b, child: int) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    out = np.zeros(27)
    lib().oracle_subdivide(_dptr(b), int(child), _dptr(out))
    return out


def exact_sign(X, sigma: int) -> int:
    X = _hex(X)
    return lib().oracle_exact_sign(_dptr(X), int(sigma))


def node_xi(sigma: int) -> np.ndarray:
    xi = np.zeros(3)
    lib().oracle_node_xi(int(sigma), _dptr(xi))
    return xi


def classify_coeffs(b, E: float = 1.0) -> dict:
    """Steps 4-5 of the algorithm on an arbitrary 27-coefficient vector."""
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    r = OracleResult()
    lib().oracle_classify_coeffs(_dptr(b), float(E), ctypes.byref(r))
    return r.as_dict()


def sample_tau(X, sigma: int) -> float:
    """Bound on the rounding error of samples27(X)[sigma] (the Step-2 exact-fallback threshold)."""
    X = _hex(X)
    return lib().oracle_sample_tau(_dptr(X), int(sigma))


def tau_depth(E: float, Mb: float, depth: int) -> float:
    """Near-boundary bound on a Bezier value at subdivision depth `depth` (reading G14)."""
    return lib().oracle_tau_depth(float(E), float(Mb), int(depth))


def num_threads(nthreads: int = 0) -> int:
    return lib().oracle_num_threads(int(nthreads))


def check_soa(coords: np.ndarray, want_coeffs: bool = False, nthreads: int = 0):
    """Batch over a (24, n) SoA array.  Returns dict of flags / near / nodes / exact (/ coeffs)."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    n = coords.shape[1]
    flags = np.zeros(n, np.uint8)
    near = np.zeros(n, np.uint8)
    nodes = np.zeros(n, np.int64)
    exact = np.zeros(n, np.uint8)
    coeffs = np.zeros((27, n)) if want_coeffs else None
    lib().oracle_check_soa(coords.ctypes.data, n, flags.ctypes.data,
                           coeffs.ctypes.data if coeffs is not None else None,
                           near.ctypes.data, nodes.ctypes.data, exact.ctypes.data, int(nthreads))
    out = {"flags": flags, "near": near, "nodes": nodes, "exact": exact}
    if coeffs is not None:
        out["coeffs"] = coeffs
    return out


def check_indexed(vertices: np.ndarray, hex_idx: np.ndarray, want_coeffs: bool = False, nthreads: int = 0):
    vertices = np.ascontiguousarray(vertices, dtype=np.float64)
    hex_idx = np.ascontiguousarray(hex_idx, dtype=np.int32)
    n = hex_idx.shape[0]
    flags = np.zeros(n, np.uint8)
    near = np.zeros(n, np.uint8)
    nodes = np.zeros(n, np.int64)
    exact = np.zeros(n, np.uint8)
    coeffs = np.zeros((27, n)) if want_coeffs else None
    lib().oracle_check_indexed(vertices.ctypes.data, hex_idx.ctypes.data, n, flags.ctypes.data,
                               coeffs.ctypes.data if coeffs is not None else None,
                               near.ctypes.data, nodes.ctypes.data, exact.ctypes.data, int(nthreads))
    out = {"flags": flags, "near": near, "nodes": nodes, "exact": exact}
    if coeffs is not None:
        out["coeffs"] = coeffs
    return out


def corner_quality(X) -> dict:
    """NEXT-2: min corner scaled Jacobian, Ushakova Test 1 (exact signs), near-zero flag."""
    X = _hex(X)
    sj = ctypes.c_double()
    t1, nr = ctypes.c_int(), ctypes.c_int()
    lib().oracle_corner_quality(_dptr(X), ctypes.byref(sj), ctypes.byref(t1), ctypes.byref(nr))
    return {"sj_min": sj.value, "test1": t1.value, "near": nr.value}


def corner_quality_soa(coords: np.ndarray, nthreads: int = 0) -> dict:
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    n = coords.shape[1]
    sj = np.zeros(n)
    t1 = np.zeros(n, np.uint8)
    nr = np.zeros(n, np.uint8)
    lib().oracle_corner_quality_soa(coords.ctypes.data, n, sj.ctypes.data, t1.ctypes.data, nr.ctypes.data,
                                    int(nthreads))
    return {"sj_min": sj, "test1": t1, "near": nr}


def corner_quality_indexed(vertices: np.ndarray, hex_idx: np.ndarray, nthreads: int = 0) -> dict:
    vertices = np.ascontiguousarray(vertices, dtype=np.float64)
    hex_idx = np.ascontiguousarray(hex_idx, dtype=np.int32)
    n = hex_idx.shape[0]
    sj = np.zeros(n)
    t1 = np.zeros(n, np.uint8)
    nr = np.zeros(n, np.uint8)
    lib().oracle_corner_quality_indexed(vertices.ctypes.data, hex_idx.ctypes.data, n, sj.ctypes.data,
                                        t1.ctypes.data, nr.ctypes.data, int(nthreads))
    return {"sj_min": sj, "test1": t1, "near": nr}


def min_detj_bounds(X, rel_tol: float) -> dict:
    """NEXT-1: certified [lower, upper] on min det J with upper - lower <= rel_tol * max|b| (or capped)."""
    X = _hex(X)
    r = OracleBounds()
    lib().oracle_min_detj_bounds(_dptr(X), float(rel_tol), ctypes.byref(r))
    return {"lower": r.lower, "upper": r.upper, "tol": r.tol, "capped": r.capped, "nodes": r.nodes}


def min_detj_bounds_soa(coords: np.ndarray, rel_tol: float, nthreads: int = 0) -> dict:
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    n = coords.shape[1]
    lo, up, cap = np.zeros(n), np.zeros(n), np.zeros(n, np.uint8)
    lib().oracle_min_detj_bounds_soa(coords.ctypes.data, n, float(rel_tol), lo.ctypes.data, up.ctypes.data,
                                     cap.ctypes.data, int(nthreads))
    return {"lower": lo, "upper": up, "capped": cap}


def select_valid(flags: np.ndarray, group: np.ndarray | None = None, n_groups: int = 0):
    """NEXT-3: ids of the VALID candidates in increasing order,
    and the number of VALID candidates per group.  Plain definition (numpy)."""
    flags = np.asarray(flags, dtype=np.uint8)
    valid = (flags & 3) == VALID
    ids = np.flatnonzero(valid).astype(np.int32)
    counts = None
    if group is not None:
        counts = np.bincount(np.asarray(group)[valid], minlength=n_groups).astype(np.int32)
    return ids, counts


def check_quad(Q) -> dict:
    """NEXT-4: validity of a linear quadrangle (4x2 nodes, counter-clockwise)."""
    Q = np.ascontiguousarray(np.asarray(Q, dtype=np.float64).reshape(4, 2))
    J = np.zeros(4)
    nr = ctypes.c_int()
    f = lib().oracle_check_quad(_dptr(Q), _dptr(J), ctypes.byref(nr))
    return {"flags": f, "J": J, "near": nr.value}


def exact_orient2d(a, b, c) -> int:
    a, b, c = (np.ascontiguousarray(np.asarray(v, dtype=np.float64)) for v in (a, b, c))
    return lib().oracle_exact_orient2d(_dptr(a), _dptr(b), _dptr(c))


def check_quad_soa(coords: np.ndarray, nthreads: int = 0) -> dict:
    """Batch over a (8, n) SoA array: plane 2k + a = axis a of node k."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    n = coords.shape[1]
    flags, near = np.zeros(n, np.uint8), np.zeros(n, np.uint8)
    J = np.zeros((4, n))
    lib().oracle_check_quad_soa(coords.ctypes.data, n, flags.ctypes.data, J.ctypes.data, near.ctypes.data,
                                int(nthreads))
    return {"flags": flags, "J": J, "near": near}
