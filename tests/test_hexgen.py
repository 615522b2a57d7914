"""Input generators: determinism, sub-range addressing, layouts, workload statistics."""
import numpy as np

import hexgen
from tests import pins


def test_uniform_is_counter_based_and_in_range():
    a = hexgen.uniform(5, 7, np.arange(1000))
    b = hexgen.uniform(5, 7, np.arange(500, 1000))
    assert np.array_equal(a[500:], b)
    assert a.min() >= 0.0 and a.max() < 1.0
    assert abs(a.mean() - 0.5) < 0.03
    assert not np.array_equal(a, hexgen.uniform(5, 8, np.arange(1000)))
    assert not np.array_equal(a, hexgen.uniform(6, 7, np.arange(1000)))


def test_soa_subrange_matches_full():
    full = hexgen.soa_config(2000, 0.35, 1)
    part = hexgen.soa_config(300, 0.35, 1, start=1234)
    assert np.array_equal(full[:, 1234:1534], part)
    assert full.shape == (24, 2000) and full.flags["C_CONTIGUOUS"]
    # node k = unit-cube corner + noise in [-amp, amp]
    X = hexgen.soa_to_nodes(full)
    d = X - pins.KAPPA[None]
    assert np.all(np.abs(d) <= 0.35)


def test_structured_grid_connectivity():
    verts, idx = hexgen.indexed_config(2, start=0, count=1000)
    assert verts.shape == (201 ** 3, 3) and idx.dtype == np.int32 and idx.shape == (1000, 8)
    # hex 0 is the cell at the origin, Fig. 3 order
    m = 201
    exp = [0, 1, 1 + m, m, m * m, 1 + m * m, 1 + m + m * m, m + m * m]
    assert idx[0].tolist() == exp
    base = np.rint(verts[idx[5]]).astype(int)
    assert np.array_equal(base - base[0], pins.KAPPA)


def test_candidate_set_statistics():
    verts, idx = hexgen.indexed_config(3, start=0, count=200_000)
    assert verts.shape == (10 ** 6, 3)
    assert idx.min() >= 0 and idx.max() < 10 ** 6
    dup = np.array([len(set(r)) < 8 for r in idx[:20000].tolist()])
    assert 0.10 < dup.mean() < 0.30            # ~18% have a duplicate vertex
    # sub-range addressing
    _, idx2 = hexgen.indexed_config(3, start=150_000, count=1000)
    assert np.array_equal(idx[150_000:151_000], idx2)


def test_adversarial_closed_form_minimum():
    """Pushed-corner family: min det J / volume = r (independent sampling of det J)."""
    coords, r = hexgen.adversarial_config(40, seed=4)
    X = hexgen.soa_to_nodes(coords)
    P = pins.grid_points(8)
    for x, rr in zip(X[0::2], r[0::2]):
        dj = pins.detj(x, P)
        vol = pins.volume_quadrature(x)
        assert abs(dj.min() / vol - rr) < 1e-9
    # twisted prisms: min over a fine zeta grid matches r within the grid error
    t = np.linspace(0, 1, 2001)
    for x, rr in zip(X[1::2], r[1::2]):
        vol = pins.volume_quadrature(x)
        G = np.stack(np.meshgrid([0.0, 0.5, 1.0], [0.0, 0.5, 1.0], t, indexing="ij"), -1).reshape(-1, 3)
        best = None
        for perm in ([0, 1, 2], [0, 2, 1], [2, 1, 0]):    # the min plane may be along any axis
            m = pins.detj(x, G[:, perm]).min() / vol
            best = m if best is None else min(best, m)
        assert abs(best - rr) < 2e-6


def test_verdict_mix_matches_the_survey_recipe():
    """The synthetic configs reproduce SURVEY.md 8(d)'s first-pass mix (App. B.1), checked
    with the oracle on prefix samples: config 1 ~4.9% INVALID, config 3 ~35.6% INVALID."""
    import oracle
    c1 = hexgen.soa_config(40_000, 0.35, 1)
    f1 = oracle.check_soa(c1)["flags"] & 3
    assert 0.040 < np.mean(f1 == oracle.INVALID) < 0.060
    assert np.mean(f1 == oracle.VALID) > 0.94
    verts, idx = hexgen.indexed_config(3, start=0, count=40_000)
    f3 = oracle.check_indexed(verts, idx)["flags"] & 3
    assert 0.32 < np.mean(f3 == oracle.INVALID) < 0.40
