"""Seeded synthetic inputs for the hexahedron-validity hot path (configs 0-4).

This module is shared by the CUDA path's tests / bench and by the CPU oracle's
tests.  It holds NONE of the method's arithmetic: no Jacobian determinants, no
Bezier transforms, no sign classification.  It only places points in space.

Layouts:

* SoA:     ``coords`` float64 of shape (24, n), C-contiguous; plane
           ``p = 3*k + a`` holds axis ``a`` of node ``k`` (Fig. 3 node order,
           PAPER.md:530-633; shape functions PAPER.md:1360-1378), i.e. element
           ``i`` of plane ``p`` is ``coords.ravel()[p*n + i]``.
* indexed: ``vertices`` float64 (nv, 3) AoS xyz and ``hex_idx`` int32 (n, 8),
           row-major, Fig. 3 node order (bottom face counter-clockwise, then
           the top face).

Random numbers: a counter-based SplitMix64 (Steele, Lea, Flood 2014).  Stream
``(seed, stream)`` has key ``K = mix(seed*G + stream*H + 1)`` and its value at
counter ``c`` is ``mix(K + (c+1)*G)``; uniforms are the top 53 bits times
2**-53.  Every draw is addressed by (seed, stream, counter), so any sub-range of
a configuration can be regenerated without generating the rest (the bench's CPU
baseline and the full-size parity samples rely on this).

Configurations follow BASELINE.json ``configs`` and SURVEY.md section 8(d).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "UNIT_CUBE", "splitmix64", "uniform", "soa_config", "indexed_config",
    "adversarial_config", "CONFIGS", "config_size", "make", "soa_to_nodes",
    "nodes_to_soa", "indexed_to_soa", "ragged_soa", "quad_soa", "UNIT_SQUARE",
]

_G = np.uint64(0x9E3779B97F4A7C15)
_H = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# Fig. 3 corner order: reference coordinates of nodes 1..8.
UNIT_CUBE = np.array(
    [[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
     [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]], dtype=np.float64)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 output finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64).copy()
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def _key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k = np.uint64(seed) * _G + np.uint64(stream) * _H + np.uint64(1)
    return splitmix64(np.array([k], dtype=np.uint64))[0]


def uniform(seed: int, stream: int, counter) -> np.ndarray:
    """Uniform doubles in [0, 1) at the given counters of stream (seed, stream)."""
    c = np.asarray(counter, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = splitmix64(_key(seed, stream) + (c + np.uint64(1)) * _G)
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


# --------------------------------------------------------------------------
# configs 0 / 1: perturbed unit cubes, SoA
# --------------------------------------------------------------------------

def soa_config(n: int, amp: float, seed: int, start: int = 0) -> np.ndarray:
    """Hexes ``start .. start+n-1`` of the perturbed-unit-cube family.

    Node k of hex i is ``UNIT_CUBE[k] + amp*(2*r - 1)`` per axis, r uniform,
    drawn at (seed, stream=p, counter=i) for plane p = 3k+a (SURVEY.md 8(d),
    configs 0 and 1).  Returns the (24, n) SoA block.
    """
    idx = np.arange(start, start + n, dtype=np.uint64)
    out = np.empty((24, n), dtype=np.float64)
    for p in range(24):
        k, a = divmod(p, 3)
        r = uniform(seed, p, idx)
        out[p] = UNIT_CUBE[k, a] + amp * (2.0 * r - 1.0)
    return out


# --------------------------------------------------------------------------
# configs 2 / 3: jittered structured grid + connectivity
# --------------------------------------------------------------------------

def grid_vertices(m: int, jitter: float, seed: int, k0: int = 0) -> np.ndarray:
    """(m^3, 3) vertices; id = i + m*(j + m*k) sits at (i, j, k + k0) + U[-jitter, jitter]^3.

    ``k0`` shifts the block along k (weak-scaling shards of config 2: rank r takes the
    k-slab starting at plane 200 r of a 200 x 200 x 200N grid); the jitter is drawn at the
    vertex's global id, so neighbouring slabs share their boundary plane exactly."""
    nv = m ** 3
    ids = np.arange(nv, dtype=np.uint64)
    i = (ids % np.uint64(m)).astype(np.float64)
    j = ((ids // np.uint64(m)) % np.uint64(m)).astype(np.float64)
    kk = ids // np.uint64(m * m) + np.uint64(k0)
    gid = ids + np.uint64(k0 * m * m)
    v = np.empty((nv, 3), dtype=np.float64)
    for a, base in enumerate((i, j, kk.astype(np.float64))):
        v[:, a] = base + jitter * (2.0 * uniform(seed, 1000 + a, gid) - 1.0)
    return v


# Fig. 3 corner offsets in (i, j, k)
_CORNER_OFF = UNIT_CUBE.astype(np.int64)


def cell_connectivity(m: int, cells: np.ndarray) -> np.ndarray:
    """int64 (len(cells), 8): the 8 vertex ids of grid cells (cells of an (m-1)^3 grid)."""
    mc = m - 1
    ci = cells % mc
    cj = (cells // mc) % mc
    ck = cells // (mc * mc)
    out = np.empty((cells.size, 8), dtype=np.int64)
    for k in range(8):
        di, dj, dk = _CORNER_OFF[k]
        out[:, k] = (ci + di) + m * ((cj + dj) + m * (ck + dk))
    return out


# 26 neighbour offsets (all of {-1,0,1}^3 except 0)
_NEIGH26 = np.array([(a, b, c) for c in (-1, 0, 1) for b in (-1, 0, 1) for a in (-1, 0, 1)
                     if (a, b, c) != (0, 0, 0)], dtype=np.int64)


def candidate_connectivity(m: int, n: int, p_swap: float, seed: int, start: int = 0) -> np.ndarray:
    """Config 3 candidates ``start .. start+n-1`` (SURVEY.md 8(d) cfg 3).

    Candidate h uses cell h mod (m-1)^3; each of its 8 indices is replaced with
    probability p_swap by a uniform in-range 26-neighbour of that vertex
    (redrawn while out of range, up to 64 attempts, else kept).  Duplicates
    allowed.  Returns int32 (n, 8).
    """
    h = np.arange(start, start + n, dtype=np.int64)
    cells = h % ((m - 1) ** 3)
    conn = cell_connectivity(m, cells)
    hu = h.astype(np.uint64)
    for k in range(8):
        swap = uniform(seed, 100 + k, hu) < p_swap
        sel = np.nonzero(swap)[0]
        if sel.size == 0:
            continue
        vid = conn[sel, k]
        vi, vj, vk = vid % m, (vid // m) % m, vid // (m * m)
        new = vid.copy()
        pending = np.ones(sel.size, dtype=bool)
        for attempt in range(64):
            if not pending.any():
                break
            r = uniform(seed, 200 + 8 * attempt + k, hu[sel])
            d = np.minimum((r * 26.0).astype(np.int64), 25)
            off = _NEIGH26[d]
            ni, nj, nk = vi + off[:, 0], vj + off[:, 1], vk + off[:, 2]
            ok = pending & (ni >= 0) & (ni < m) & (nj >= 0) & (nj < m) & (nk >= 0) & (nk < m)
            new[ok] = (ni + m * (nj + m * nk))[ok]
            pending &= ~ok
        conn[sel, k] = new
    return conn.astype(np.int32)


def indexed_config(cfg: int, start: int = 0, count: int | None = None, slab: int = 0, workers: int = 1):
    """(vertices, hex_idx) for config 2 (structured 200^3) or 3 (40M candidates).

    ``slab`` (config 2): the k-slab ``slab`` of a grid stacked along k (see grid_vertices).
    ``workers`` > 1 generates config 3's connectivity in parallel chunks (identical result:
    every draw is addressed by the candidate id)."""
    if cfg == 2:
        m, jit, seed, n_total = 201, 0.3, 2, 200 ** 3
        verts = grid_vertices(m, jit, seed, k0=200 * slab)
        n = n_total - start if count is None else count
        cells = np.arange(start, start + n, dtype=np.int64)
        return verts, cell_connectivity(m, cells).astype(np.int32)
    if cfg == 3:
        m, jit, seed, n_total = 100, 0.2, 3, 40_000_000
        verts = grid_vertices(m, jit, seed)
        n = n_total - start if count is None else count
        return verts, _chunked(lambda a, c: candidate_connectivity(m, c, 0.1, seed, a), start, n, workers, axis=0)
    raise ValueError(cfg)


def _chunked(fn, start: int, n: int, workers: int, axis: int):
    """fn(start, count) over ``workers`` contiguous chunks in forked processes, concatenated."""
    if workers <= 1 or n < 2_000_000:
        return fn(start, n)
    import multiprocessing as mp
    global _FORK_FN
    step = -(-n // workers)
    parts = [(a, min(step, start + n - a)) for a in range(start, start + n, step)]
    _FORK_FN = fn                                   # inherited by the forked workers
    try:
        with mp.get_context("fork").Pool(len(parts)) as pool:
            out = pool.map(_fork_call, parts)
    finally:
        _FORK_FN = None
    return np.ascontiguousarray(np.concatenate(out, axis=axis))


_FORK_FN = None


def _fork_call(ac):
    return _FORK_FN(*ac)


# --------------------------------------------------------------------------
# config 4: adversarial near-boundary families (closed-form verdicts)
# --------------------------------------------------------------------------

def _rotations24() -> np.ndarray:
    """The 24 proper rotations of the reference cube as 3x3 signed permutation matrices."""
    mats = []
    for perm in ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)):
        for sx in (1, -1):
            for sy in (1, -1):
                for sz in (1, -1):
                    R = np.zeros((3, 3))
                    for r, (c, s) in enumerate(zip(perm, (sx, sy, sz))):
                        R[r, c] = s
                    if round(np.linalg.det(R)) == 1:
                        mats.append(R)
    return np.array(mats)


_ROT24 = _rotations24()


def _corner_index(kappa: np.ndarray) -> np.ndarray:
    """Fig. 3 index of reference corners kappa (..., 3) in {0,1}^3."""
    table = {tuple(c): i for i, c in enumerate(_CORNER_OFF.tolist())}
    flat = kappa.reshape(-1, 3)
    return np.array([table[tuple(x)] for x in flat.tolist()]).reshape(kappa.shape[:-1])


# _RELABEL[q, k] = old node index that becomes new node k under cube rotation q
_RELABEL = np.stack([
    _corner_index(np.rint((R @ (UNIT_CUBE - 0.5).T).T + 0.5).astype(np.int64)) for R in _ROT24])


def _affine(seed: int, ids: np.ndarray, stream0: int):
    """Random affine maps A = rotation * diag(U[0.5,2]^3) * unit-shear(U[-1/2,1/2]) and translations."""
    u = [uniform(seed, stream0 + s, ids) for s in range(12)]
    # uniform random rotation from a unit quaternion (Shoemake)
    u1, u2, u3 = u[0], u[1], u[2]
    q0 = np.sqrt(1 - u1) * np.sin(2 * math.pi * u2)
    q1 = np.sqrt(1 - u1) * np.cos(2 * math.pi * u2)
    q2 = np.sqrt(u1) * np.sin(2 * math.pi * u3)
    q3 = np.sqrt(u1) * np.cos(2 * math.pi * u3)
    w, x, y, z = q0, q1, q2, q3
    R = np.empty((ids.size, 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z); R[:, 0, 1] = 2 * (x * y - z * w); R[:, 0, 2] = 2 * (x * z + y * w)
    R[:, 1, 0] = 2 * (x * y + z * w); R[:, 1, 1] = 1 - 2 * (x * x + z * z); R[:, 1, 2] = 2 * (y * z - x * w)
    R[:, 2, 0] = 2 * (x * z - y * w); R[:, 2, 1] = 2 * (y * z + x * w); R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    D = np.zeros((ids.size, 3, 3))
    for a in range(3):
        D[:, a, a] = 0.5 + 1.5 * u[3 + a]
    S = np.zeros((ids.size, 3, 3))
    S[:, 0, 0] = S[:, 1, 1] = S[:, 2, 2] = 1.0
    S[:, 0, 1] = u[6] - 0.5
    S[:, 0, 2] = u[7] - 0.5
    S[:, 1, 2] = u[8] - 0.5
    A = R @ D @ S
    t = np.stack([8.0 * u[9] - 4.0, 8.0 * u[10] - 4.0, 8.0 * u[11] - 4.0], axis=-1)
    return A, t


def _pushed_corner(seed: int, ids: np.ndarray):
    """Parallelepiped x = A xi + t with corner k pushed along reference axis a.

    With push u = (t_p - 1) s_a e_a in reference coordinates (s_a = +1 if corner
    k has reference coordinate 1 on axis a, else -1) the map is
    x = A(xi + L_k(xi) u) + t; its min Jacobian / volume is r = 4 t_p / (3 + t_p)
    (derivation in DESIGN.md "Input recipe").  Target r ~ U[-1e-3, 1e-3].
    """
    r = 2e-3 * uniform(seed, 10, ids) - 1e-3
    tp = 3.0 * r / (4.0 - r)
    k = np.minimum((uniform(seed, 11, ids) * 8).astype(np.int64), 7)
    a = np.minimum((uniform(seed, 12, ids) * 3).astype(np.int64), 2)
    kappa = _CORNER_OFF[k]                                # (m, 3)
    s_a = np.where(kappa[np.arange(ids.size), a] == 1, 1.0, -1.0)
    ref = np.broadcast_to(UNIT_CUBE, (ids.size, 8, 3)).copy()
    ref[np.arange(ids.size), k, a] += (tp - 1.0) * s_a
    A, t = _affine(seed, ids, 20)
    X = np.einsum("mij,mkj->mki", A, ref) + t[:, None, :]
    return X, r


def _twisted_prism(seed: int, ids: np.ndarray):
    """Twisted prism: bottom (+-1/2, +-1/2, 0), top (S p, 1); det J = q(zeta) = 1+(T-2)z+(1-T+D)z^2.

    Minimum q* at zeta* ~ U[0.2, 0.8]; |r| = q*/mean(q) ~ U[1e-5, 1e-3] with a
    random sign.  A random cube rotation relabels
    the nodes and a random affine map + translation is applied.
    """
    mag = 1e-5 + (1e-3 - 1e-5) * uniform(seed, 40, ids)
    sgn = np.where(uniform(seed, 41, ids) < 0.5, -1.0, 1.0)
    r = sgn * mag
    zs = 0.2 + 0.6 * uniform(seed, 42, ids)
    K = ((1 - zs) ** 3 + zs ** 3) / 3.0
    qs = (r * K / zs ** 2) / (1.0 - r + r * K / zs ** 2)
    c2 = (1.0 - qs) / zs ** 2
    T = 2.0 - 2.0 * c2 * zs
    D = c2 - 1.0 + T
    disc = T * T / 4.0 - D
    m = ids.size
    Smat = np.zeros((m, 2, 2))
    real = disc >= 0
    sq = np.sqrt(np.abs(disc))
    Smat[real, 0, 0] = T[real] / 2 + sq[real]
    Smat[real, 1, 1] = T[real] / 2 - sq[real]
    Smat[~real, 0, 0] = T[~real] / 2
    Smat[~real, 1, 1] = T[~real] / 2
    Smat[~real, 0, 1] = -sq[~real]
    Smat[~real, 1, 0] = sq[~real]
    bottom = UNIT_CUBE[:4, :2] - 0.5                       # (4, 2)
    X = np.zeros((m, 8, 3))
    X[:, :4, :2] = bottom
    X[:, 4:, :2] = np.einsum("mij,kj->mki", Smat, bottom)
    X[:, 4:, 2] = 1.0
    q = np.minimum((uniform(seed, 43, ids) * 24).astype(np.int64), 23)
    X = X[np.arange(m)[:, None], _RELABEL[q]]
    A, t = _affine(seed, ids, 60)
    X = np.einsum("mij,mkj->mki", A, X) + t[:, None, :]
    return X, r


def adversarial_config(n: int, seed: int = 4, start: int = 0):
    """Config 4 hexes start..start+n-1: (coords (24, n) SoA, r (n,)).

    Even ids: pushed-corner parallelepipeds, odd ids: twisted prisms.  The
    exact-geometry verdict is VALID iff r > 0 (closed form; rounding of the
    generated coordinates moves min det J by O(1e-16) relative).
    """
    ids = np.arange(start, start + n, dtype=np.uint64)
    even = (ids % np.uint64(2)) == 0
    X = np.empty((n, 8, 3))
    r = np.empty(n)
    if even.any():
        X[even], r[even] = _pushed_corner(seed, ids[even])
    if (~even).any():
        X[~even], r[~even] = _twisted_prism(seed, ids[~even])
    return nodes_to_soa(X), r


# --------------------------------------------------------------------------
# helpers
# --------------------------------------------------------------------------

def nodes_to_soa(X: np.ndarray) -> np.ndarray:
    """(n, 8, 3) node array -> (24, n) SoA."""
    n = X.shape[0]
    return np.ascontiguousarray(X.reshape(n, 24).T)


def soa_to_nodes(coords: np.ndarray) -> np.ndarray:
    """(24, n) SoA -> (n, 8, 3) node array."""
    return np.ascontiguousarray(coords.T.reshape(-1, 8, 3))


def indexed_to_soa(vertices: np.ndarray, hex_idx: np.ndarray) -> np.ndarray:
    return nodes_to_soa(vertices[hex_idx.astype(np.int64)])


UNIT_SQUARE = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=np.float64)


def quad_soa(n: int, amp: float, seed: int, start: int = 0) -> np.ndarray:
    """Linear quadrangles (NEXT-4): unit-square corner k + amp*(2r-1) per axis, r drawn at
    (seed, stream=500+p, counter=i) for plane p = 2k + a.  Returns the (8, n) SoA block."""
    idx = np.arange(start, start + n, dtype=np.uint64)
    out = np.empty((8, n), dtype=np.float64)
    for p in range(8):
        k, a = divmod(p, 2)
        out[p] = UNIT_SQUARE[k, a] + amp * (2.0 * uniform(seed, 500 + p, idx) - 1.0)
    return out


def ragged_soa(n: int, seed: int = 11, amp: float = 0.35) -> np.ndarray:
    """Small perturbed-cube SoA set of arbitrary size (used for ragged-tail tests)."""
    return soa_config(n, amp, seed)


@dataclass(frozen=True)
class ConfigInfo:
    cfg: int
    layout: str
    n: int
    description: str


CONFIGS = {
    0: ConfigInfo(0, "soa", 10_000, "10k perturbed unit cubes, noise U[-0.25,0.25]^3, seed 0"),
    1: ConfigInfo(1, "soa", 10_000_000, "10M perturbed unit cubes, noise U[-0.35,0.35]^3, seed 1"),
    2: ConfigInfo(2, "indexed", 8_000_000, "200^3 structured grid, 201^3 vertices jitter +-0.3, seed 2"),
    3: ConfigInfo(3, "indexed", 40_000_000, "40M candidates on a 100^3 jittered grid (+-0.2), p_swap 0.1, seed 3"),
    4: ConfigInfo(4, "soa", 4_000_000, "4M adversarial: pushed-corner parallelepipeds + twisted prisms, seed 4"),
}


def config_size(cfg: int) -> int:
    return CONFIGS[cfg].n


def make(cfg: int, start: int = 0, count: int | None = None, workers: int = 1, slab: int = 0):
    """Generate (part of) a configuration.

    Returns ``("soa", coords)`` / ``("soa", coords, r)`` for configs 0, 1, 4 and
    ``("indexed", vertices, hex_idx)`` for configs 2, 3.  ``workers`` > 1 generates large
    configurations in parallel chunks (bit-identical to the serial result).
    """
    info = CONFIGS[cfg]
    n = info.n - start if count is None else count
    if cfg == 0:
        return ("soa", soa_config(n, 0.25, 0, start))
    if cfg == 1:
        return ("soa", _chunked(lambda a, c: soa_config(c, 0.35, 1, a), start, n, workers, axis=1))
    if cfg == 4:
        both = _chunked(lambda a, c: np.vstack(adversarial_config(c, 4, a)), start, n, workers, axis=1)
        return ("soa", np.ascontiguousarray(both[:24]), np.ascontiguousarray(both[24]))
    verts, idx = indexed_config(cfg, start, n, slab=slab, workers=workers)
    return ("indexed", verts, idx)
