"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the passage it checks.  None of them compares the oracle with
itself: the references are exact rational matrices built from the Bernstein
definition, an independent shape-function evaluation of det J, closed forms,
the paper's printed examples, brute-force sampling and Python exact rationals.
"""
from fractions import Fraction

import numpy as np
import pytest

import hexgen
import oracle
from tests import pins

U = pins.KAPPA.astype(np.float64)


# --------------------------------------------------------------------------
# constants: Table 1, Table 2, Table 3
# --------------------------------------------------------------------------

def test_table1_is_inverse_of_bernstein_collocation():
    """T_b = A^-1 with A_{sigma tau} = B_tau(xi_sigma) (Table 1)."""
    Ainv = pins.invert_exact(pins.collocation_matrix_exact())
    T = oracle.tb_matrix()
    for s in range(27):
        for t in range(27):
            assert Fraction(float(T[s, t])) == Ainv[s][t], (s, t)


def test_table1_rows_sum_to_one():
    """Constant functions have constant Bezier coefficients."""
    T = oracle.tb_matrix()
    assert np.all(T.sum(axis=1) == 1.0)


def test_table3_equals_D_times_Tsub_with_corrected_table2():
    """Table 3 = D * T_sub; Table 2 as printed has the opposite sign (reading G1)."""
    Tb = pins.invert_exact(pins.collocation_matrix_exact())
    Tsub = [row[:20] for row in Tb[:20]]
    printed = pins.table2_printed_exact()
    # printed rows sum to -1, which cannot preserve constants
    assert all(sum(r) == -1 for r in printed)
    corrected = [[-v for v in r] for r in printed]
    D = [[Fraction(int(i == j)) for j in range(20)] for i in range(20)] + corrected
    DT = [[sum(D[i][k] * Tsub[k][j] for k in range(20)) for j in range(20)] for i in range(27)]
    T3 = pins.table3_exact()
    assert DT == T3
    # and with the printed sign the product does not reproduce Table 3
    Dp = [[Fraction(int(i == j)) for j in range(20)] for i in range(20)] + printed
    DTp = [[sum(Dp[i][k] * Tsub[k][j] for k in range(20)) for j in range(20)] for i in range(27)]
    assert DTp != T3


def test_oracle_coefficients_match_table3_route():
    """b = T_b c_27 (oracle) equals T-tilde c_20 (Table 3) on random hexes (Cor. 1)."""
    T3 = np.array([[float(v) for v in r] for r in pins.table3_exact()])
    for X in pins.random_hexes(300, 0.45, 1):
        r = oracle.check_hex(X)
        b3 = T3 @ r["c"][:20]
        scale = np.max(np.abs(r["b"]))
        assert np.max(np.abs(b3 - r["b"])) <= 1e-13 * scale


def test_corollary1_seven_monomials_vanish():
    """m_220 = m_202 = m_022 = m_221 = m_212 = m_122 = m_222 = 0 (Cor. 1)."""
    t = np.array([0.0, 0.5, 1.0])
    V1 = np.vander(t, 3, increasing=True)            # 1D Vandermonde on {0,1/2,1}
    Vi = np.linalg.inv(V1)
    for X in pins.random_hexes(200, 0.45, 2):
        c = oracle.samples27(X)
        C = np.zeros((3, 3, 3))
        for s in range(27):
            i, j, k = pins.XI2[s]
            C[i, j, k] = c[s]
        M = np.einsum("ai,bj,ck,ijk->abc", Vi, Vi, Vi, C)   # monomial coefficients m_abc
        scale = np.max(np.abs(M))
        for (a, b, cc) in [(2, 2, 0), (2, 0, 2), (0, 2, 2), (2, 2, 1), (2, 1, 2), (1, 2, 2), (2, 2, 2)]:
            assert abs(M[a, b, cc]) <= 1e-12 * scale


# --------------------------------------------------------------------------
# samples and the Bezier expansion
# --------------------------------------------------------------------------

def test_samples_are_detj_at_nodes():
    """c_sigma = det J(xi_sigma), vs an independent shape-function evaluation."""
    nodes = pins.XI2 / 2.0
    for X in pins.random_hexes(200, 0.45, 3):
        c = oracle.samples27(X)
        ref = pins.detj(X, nodes)
        assert np.max(np.abs(c - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_bezier_expansion_reproduces_detj():
    """sum_sigma b_sigma B_sigma(xi) = det J(xi) everywhere (Eq. e:bezExpansion)."""
    rng = np.random.default_rng(4)
    for X in pins.random_hexes(200, 0.45, 4):
        b = oracle.check_hex(X)["b"]
        P = rng.uniform(0, 1, size=(50, 3))
        ref = pins.detj(X, P)
        got = pins.bezier_eval(b, P)
        assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(b))
        # and the oracle's own evaluator agrees with the independent one
        for p in P[:5]:
            assert abs(oracle.bezier_eval(b, p) - pins.bezier_eval(b, p[None])[0]) <= 1e-14 * np.max(np.abs(b))


def test_corner_coefficients_are_corner_tet_determinants():
    """b_1..8 = det J at corners = 6 vol(corner tet)."""
    for X in pins.random_hexes(100, 0.4, 5):
        b = oracle.check_hex(X)["b"]
        for k in range(8):
            kap = pins.KAPPA[k]
            nbrs = []
            for a in range(3):
                nb = kap.copy()
                nb[a] = 1 - nb[a]
                nbrs.append(int(np.nonzero((pins.KAPPA == nb).all(axis=1))[0][0]))
            d = pins.tet_det(X[k], X[nbrs[0]], X[nbrs[1]], X[nbrs[2]])
            flips = int(np.sum(kap))                  # each flipped axis reverses one edge
            assert abs(b[k] - (-1) ** flips * d) <= 1e-13 * max(1.0, abs(d))


def test_mean_coefficient_is_volume():
    """mean(b) = integral of det J = hex volume (10 tets; quadrature)."""
    for X in pins.random_hexes(100, 0.4, 6):
        b = oracle.check_hex(X)["b"]
        v10 = pins.volume_10_tets(X)
        vq = pins.volume_quadrature(X)
        assert abs(b.mean() - v10) <= 1e-13 * np.max(np.abs(b))
        assert abs(b.mean() - vq) <= 1e-12 * np.max(np.abs(b))


# --------------------------------------------------------------------------
# closed forms
# --------------------------------------------------------------------------

def test_unit_cube_valid_no_subdivision():
    r = oracle.check_hex(U)
    assert r["flags"] == oracle.VALID and r["nodes"] == 0
    assert np.all(r["b"] == 1.0)


def test_mirrored_cube_invalid():
    X = U.copy()
    X[:, 0] *= -1.0
    r = oracle.check_hex(X)
    assert r["flags"] == oracle.INVALID
    assert np.all(r["b"] == -1.0)


def test_parallelepiped_all_coefficients_equal():
    """Affine map => det J constant => all 27 b equal det A."""
    rng = np.random.default_rng(7)
    for _ in range(200):
        A = rng.normal(size=(3, 3))
        x0 = rng.normal(size=3)
        X = U @ A.T + x0
        r = oracle.check_hex(X)
        d = np.linalg.det(A)
        assert np.max(np.abs(r["b"] - d)) <= 1e-13 * max(1.0, np.max(np.abs(A)) ** 3)
        assert (r["flags"] & 3) == (oracle.VALID if d > 0 else oracle.INVALID)
        assert r["nodes"] == 0


def test_power_of_two_scaling_is_exact():
    """Scaling by 2^k scales every det J value by 8^k exactly; the verdict is unchanged."""
    for X in pins.random_hexes(100, 0.45, 8):
        r0 = oracle.check_hex(X)
        r1 = oracle.check_hex(X * 4.0)
        assert r1["flags"] == r0["flags"]
        assert np.array_equal(r1["b"], r0["b"] * 64.0)


# --------------------------------------------------------------------------
# subdivision
# --------------------------------------------------------------------------

def test_subdivision_is_exact_reparameterisation():
    rng = np.random.default_rng(9)
    for _ in range(100):
        b = rng.normal(size=27)
        for o in range(8):
            child = oracle.subdivide(b, o)
            kap = pins.KAPPA[o]
            loc = rng.uniform(0, 1, size=(20, 3))
            glob = 0.5 * (kap[None, :] + loc)
            assert np.max(np.abs(pins.bezier_eval(child, loc) - pins.bezier_eval(b, glob))) <= 1e-14 * np.max(np.abs(b))


def test_subdivision_children_lie_in_the_parent_hull():
    """De Casteljau children are convex combinations of the parent's coefficients: every
    child coefficient lies in [min b, max b] and the spread max - min never grows
    (SPEC.md's subdivision-convergence property; the basis of the bounds)."""
    rng = np.random.default_rng(12)
    for _ in range(200):
        b = rng.normal(size=27) * rng.uniform(0.1, 10.0)
        lo, hi = b.min(), b.max()
        eps = 4e-16 * np.max(np.abs(b))
        for o in range(8):
            c = oracle.subdivide(b, o)
            assert c.min() >= lo - eps and c.max() <= hi + eps
            assert c.max() - c.min() <= hi - lo + 2 * eps


def test_subdivision_children_corners_are_values():
    """Child corner coefficients are actual values of the polynomial."""
    rng = np.random.default_rng(10)
    b = rng.normal(size=27)
    for o in range(8):
        child = oracle.subdivide(b, o)
        kap = pins.KAPPA[o]
        for k in range(8):
            pt = 0.5 * (kap + pins.KAPPA[k])
            assert abs(child[k] - pins.bezier_eval(b, pt[None])[0]) <= 1e-14 * np.max(np.abs(b))


def test_depth_cap_gives_undetermined():
    """A polynomial >= 0 with a zero at a non-dyadic point never decides: depth cap -> UNDETERMINED."""
    a = 1.0 / 3.0
    q = np.array([a * a, a * (a - 1.0), (1.0 - a) ** 2])     # Bernstein coefficients of (t-a)^2
    b = np.array([q[i] + q[j] + q[k] for i, j, k in pins.XI2])
    r = oracle.classify_coeffs(b, 1.0)
    assert r["flags"] == (oracle.UNDETERMINED | oracle.FLAG_SUBDIVIDED)
    assert r["max_depth"] == oracle.MAX_DEPTH
    # shifted upwards by a margin, the same polynomial is VALID after subdivision
    r2 = oracle.classify_coeffs(b + 1e-3, 1.0)
    assert r2["flags"] == (oracle.VALID | oracle.FLAG_SUBDIVIDED)


def test_invalid_dominates_undetermined():
    """A negative child corner anywhere gives INVALID even if another branch caps (reading G4)."""
    a = 1.0 / 3.0
    q = np.array([a * a, a * (a - 1.0), (1.0 - a) ** 2])
    b = np.array([q[i] + q[j] + q[k] for i, j, k in pins.XI2])
    b[26] = -5.0          # centre coefficient very negative: det < 0 near the centre
    r = oracle.classify_coeffs(b, 1.0)
    assert (r["flags"] & 3) == oracle.INVALID
    assert pins.bezier_eval(b, r["witness"][None])[0] <= 0.0


# --------------------------------------------------------------------------
# the paper's examples (Figs. 5-7)
# --------------------------------------------------------------------------

def test_fig5_invalid_with_27_positive_samples(golden_hexes):
    X, exp = golden_hexes["fig5_invalid"]
    r = oracle.check_hex(X)
    assert (r["flags"] & 3) == oracle.INVALID and exp["verdict"] == "INVALID"
    assert np.all(pins.detj(X, pins.XI2 / 2.0) > 0)          # caption: positive at the 27 nodes
    assert np.all(r["c"] > 0)
    assert r["subdivided"] == 1                                # decided by recursive_subdivision
    assert pins.detj(X, r["witness"][None])[0] <= 0.0          # witness really is non-positive


def test_fig6_valid(golden_hexes):
    X, exp = golden_hexes["fig6_valid"]
    r = oracle.check_hex(X)
    assert exp["verdict"] == "VALID"
    assert (r["flags"] & 3) == oracle.VALID
    assert r["subdivided"] == 1 and np.min(r["b"]) < 0        # needs subdivision to prove validity
    P = pins.grid_points(40)
    assert np.min(pins.detj(X, P)) > 0


def test_fig7_invalid_at_step2_with_high_corner_quality(golden_hexes):
    X, exp = golden_hexes["fig7_invalid"]
    r = oracle.check_hex(X)
    assert exp["verdict"] == "INVALID"
    assert r["flags"] == oracle.INVALID                        # Step 2, not subdivided
    assert np.all(r["c"][:8] > 0) and np.min(r["c"][8:20]) < 0
    assert abs(pins.corner_scaled_jacobian(X) - float(exp["corner_scaled_jacobian"])) <= 0.01


# --------------------------------------------------------------------------
# brute force and exactness
# --------------------------------------------------------------------------

def test_brute_force_never_contradicts():
    """Dense sampling of det J never contradicts a verdict (SURVEY.md 4 pin 8)."""
    P = pins.grid_points(16)
    adv, _ = hexgen.adversarial_config(200, seed=4, start=5000)
    Xs = np.concatenate([pins.random_hexes(150, 0.5, 11), pins.random_hexes(150, 0.6, 12),
                         hexgen.soa_to_nodes(adv)])
    seen = set()
    for X in Xs:
        r = oracle.check_hex(X)
        v = r["flags"] & 3
        seen.add((v, r["subdivided"]))
        E3 = r["E"] ** 3
        if v == oracle.VALID:
            assert np.min(pins.detj(X, P)) > -1e-12 * E3
        elif v == oracle.INVALID:
            assert pins.detj(X, r["witness"][None])[0] <= 1e-12 * E3
    assert (oracle.VALID, 1) in seen and (oracle.INVALID, 1) in seen and (oracle.INVALID, 0) in seen


def _degenerate_hexes(rng, n):
    """Hexes with duplicated or coplanar vertices: det J values exactly 0 at some nodes."""
    out = []
    for _ in range(n):
        X = U + rng.uniform(-0.3, 0.3, size=(8, 3))
        kind = rng.integers(0, 3)
        i, j = rng.choice(8, size=2, replace=False)
        if kind == 0:
            X[j] = X[i]                                  # duplicate vertex
        elif kind == 1:
            X[j] = X[i] + 0.5 * (X[(i + 1) % 8] - X[i])  # point on a segment (rounded)
        else:
            X[:, 2] = np.round(X[:, 2] * 8) / 8          # many coplanar dyadic points
            X[j, 2] = X[i, 2]
        out.append(X)
    return out


def test_exact_sign_matches_rational_arithmetic():
    """The oracle's bigint sign of det J(xi_sigma) equals Python exact rationals."""
    rng = np.random.default_rng(13)
    hexes = _degenerate_hexes(rng, 60) + list(pins.random_hexes(20, 0.4, 14))
    zeros = 0
    for X in hexes:
        for s in range(27):
            ex = pins.detj_exact(X, s)
            sg = (ex > 0) - (ex < 0)
            zeros += sg == 0
            assert oracle.exact_sign(X, s) == sg, (s, X)
    assert zeros > 20


def test_exact_zero_sample_is_invalid():
    """A sample exactly 0 (diagonal duplicate) is decided INVALID although fp gives +-tiny (reading G2/G8)."""
    rng = np.random.default_rng(15)
    hits = 0
    for _ in range(200):
        X = U + rng.uniform(-0.3, 0.3, size=(8, 3))
        X[2] = X[0]                       # nodes 1 and 3 coincide: det J = 0 at corner 2
        r = oracle.check_hex(X)
        assert pins.detj_exact(X, 1) == 0
        assert (r["flags"] & 3) == oracle.INVALID
        if r["c"][1] != 0.0:
            hits += 1
            assert r["exact_used"] >= 1
    assert hits > 0


def test_nonfinite_and_out_of_range():
    for bad in (np.nan, np.inf, -np.inf, 2.0 ** 301):
        X = U.copy()
        X[5, 1] = bad
        assert oracle.check_hex(X)["flags"] == oracle.NONFINITE
    X = U * 2.0 ** 299
    assert oracle.check_hex(X)["flags"] == oracle.VALID


# --------------------------------------------------------------------------
# closed-form families (config 4) and batch driver
# --------------------------------------------------------------------------

def test_adversarial_families_closed_form_verdicts():
    """Pushed-corner and twisted-prism families: VALID iff r > 0 (DESIGN.md input recipe)."""
    coords, r = hexgen.adversarial_config(600, seed=4, start=0)
    o = oracle.check_soa(coords, nthreads=0)
    v = o["flags"] & 3
    assert np.array_equal(v, np.where(r > 0, oracle.VALID, oracle.INVALID))
    even = np.arange(600) % 2 == 0
    assert not np.any(o["flags"][even] & oracle.FLAG_SUBDIVIDED)    # multilinear: never subdivides
    assert np.mean((o["flags"][~even] & oracle.FLAG_SUBDIVIDED) > 0) > 0.9
    assert not np.any(o["near"])


def test_twisted_valid_node_count_is_order_independent():
    """For VALID hexes the subdivision tree is fully explored: node count equals that of a
    breadth-first count done here."""
    coords, r = hexgen.adversarial_config(40, seed=4, start=1001)
    nodes = hexgen.soa_to_nodes(coords)
    for X, rr in zip(nodes[0::2], r[0::2]):          # start is odd: even positions are twisted prisms
        res = oracle.check_hex(X)
        if (res["flags"] & 3) != oracle.VALID or not res["subdivided"]:
            continue
        count, frontier = 0, [(res["b"], 0)]
        while frontier:
            nxt = []
            for b, d in frontier:
                count += 1
                for o in range(8):
                    ch = oracle.subdivide(b, o)
                    assert np.min(ch[:8]) > 0
                    if np.min(ch[8:]) > 0:
                        continue
                    assert d + 1 < oracle.MAX_DEPTH
                    nxt.append((ch, d + 1))
            frontier = nxt
        assert count == res["nodes"]
        if count > 50:
            return
    pytest.fail("no large valid twisted hex in the sample")


def test_batch_equals_single():
    coords = hexgen.soa_config(500, 0.4, 99)
    o = oracle.check_soa(coords, want_coeffs=True, nthreads=4)
    X = hexgen.soa_to_nodes(coords)
    for i in range(0, 500, 7):
        r = oracle.check_hex(X[i])
        assert o["flags"][i] == r["flags"]
        assert np.array_equal(o["coeffs"][:, i], r["b"])


def test_config0_has_no_near_boundary_hexes():
    _, coords = hexgen.make(0)
    o = oracle.check_soa(coords)
    assert o["near"].sum() == 0
    f = o["flags"]
    assert np.all((f & 3) != oracle.UNDETERMINED)


# --------------------------------------------------------------------------
# NEXT-2: corner screening quantities
# --------------------------------------------------------------------------

def test_corner_quality_closed_forms():
    """Unit cube: scaled Jacobian 1; shear x += s*y: every corner frame has det 1 and one
    edge of length sqrt(1+s^2), so the min is 1/sqrt(1+s^2); mirrored cube: -1, Test 1 fails."""
    assert oracle.corner_quality(U) == {"sj_min": 1.0, "test1": 1, "near": 0}
    for s in (0.25, 0.5, 2.0):
        X = U.copy()
        X[:, 0] += s * X[:, 1]
        r = oracle.corner_quality(X)
        assert abs(r["sj_min"] - 1.0 / np.sqrt(1.0 + s * s)) <= 1e-15 and r["test1"] == 1
    M = U * np.array([-1.0, 1.0, 1.0])
    r = oracle.corner_quality(M)
    assert r["sj_min"] == -1.0 and r["test1"] == 0


def test_corner_quality_fig7_and_fig5(golden_hexes):
    """Fig. 7 caption: corner scaled Jacobian "0.64" (0.6471 truncated, reading G10);
    Fig. 5: all corner tets positive (Test 1 passes) although the hex is invalid."""
    r7 = oracle.corner_quality(golden_hexes["fig7_invalid"][0])
    assert abs(r7["sj_min"] - 0.64) < 0.01 and abs(r7["sj_min"] - 0.6471) < 5e-5
    r5 = oracle.corner_quality(golden_hexes["fig5_invalid"][0])
    assert r5["test1"] == 1
    assert (oracle.check_hex(golden_hexes["fig5_invalid"][0])["flags"] & 3) == oracle.INVALID


def test_corner_quality_invariances_and_test1_definition():
    """Invariant under rotation, translation and positive scaling; Test 1 == all corner
    samples > 0 (independent exact rational evaluation); Test 1 is necessary for validity."""
    rng = np.random.default_rng(21)
    for X in pins.random_hexes(200, 0.45, 22):
        r = oracle.corner_quality(X)
        Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        if np.linalg.det(Q) < 0:
            Q[:, 0] *= -1
        Y = (X @ Q.T) * 3.7 + rng.normal(size=3)
        r2 = oracle.corner_quality(Y)
        assert abs(r["sj_min"] - r2["sj_min"]) <= 1e-12
        exact_pos = all(pins.detj_exact(X, k) > 0 for k in range(8))
        assert r["test1"] == int(exact_pos)
        if (oracle.check_hex(X)["flags"] & 3) == oracle.VALID:
            assert r["test1"] == 1
    X = U.copy()
    X[1] = X[0]                                  # zero-length corner edge: undefined metric
    assert np.isnan(oracle.corner_quality(X)["sj_min"])


# --------------------------------------------------------------------------
# NEXT-1: bounds on min det J
# --------------------------------------------------------------------------

def test_bounds_parallelepiped_and_cube():
    """Affine map: det J constant, every coefficient equals det A, so lower = upper = det A."""
    assert oracle.min_detj_bounds(U, 0.0) == {"lower": 1.0, "upper": 1.0, "tol": 0.0, "capped": 0, "nodes": 0}
    rng = np.random.default_rng(31)
    for _ in range(50):
        A = rng.normal(size=(3, 3))
        X = U @ A.T + rng.normal(size=3)
        d = np.linalg.det(A)
        r = oracle.min_detj_bounds(X, 1e-9)
        assert abs(r["lower"] - d) <= 1e-12 * max(1, abs(d)) and abs(r["upper"] - d) <= 1e-12 * max(1, abs(d))


@pytest.mark.parametrize("rel_tol,family", [(1e-2, "both"), (1e-4, "both"), (1e-9, "pushed")])
def test_bounds_closed_form_families(rel_tol, family):
    """Pushed-corner and twisted-prism families (DESIGN.md input recipe): min det J = r * V
    in closed form, V = mean(b) = volume; the bounds must bracket it within tol.  (The
    twisted prisms attain their minimum on a plane, so their tree grows like 1/tol.)"""
    coords, r = hexgen.adversarial_config(120, seed=4, start=9000)
    X = hexgen.soa_to_nodes(coords)
    for j in range(X.shape[0]):
        if family == "pushed" and j % 2:
            continue
        b = oracle.check_hex(X[j])["b"]
        m_star = r[j] * b.mean()
        res = oracle.min_detj_bounds(X[j], rel_tol)
        eps = 1e-12 * np.abs(b).max()
        assert res["lower"] <= m_star + eps and m_star <= res["upper"] + eps, (j, res, m_star)
        assert res["capped"] or res["upper"] - res["lower"] <= res["tol"] + eps


def test_bounds_paper_figures(golden_hexes):
    """Figs. 5 and 7 are invalid (captions): upper < 0; Fig. 6 is valid: lower > 0."""
    assert oracle.min_detj_bounds(golden_hexes["fig5_invalid"][0], 1e-6)["upper"] < 0
    assert oracle.min_detj_bounds(golden_hexes["fig7_invalid"][0], 1e-6)["upper"] < 0
    assert oracle.min_detj_bounds(golden_hexes["fig6_valid"][0], 1e-6)["lower"] > 0


def test_bounds_against_dense_sampling_and_verdicts():
    """Dense 31^3 sampling of det J (independent evaluation) never goes below lower, and
    lies above upper - tol; lower > 0 implies VALID and upper <= 0 implies INVALID."""
    P = pins.grid_points(30)
    for X in pins.random_hexes(60, 0.5, 33):
        res = oracle.min_detj_bounds(X, 1e-3)
        v = pins.detj(X, P)
        scale = max(1.0, np.abs(v).max())
        assert v.min() >= res["lower"] - 1e-12 * scale
        assert v.min() >= res["upper"] - res["tol"] - 1e-12 * scale
        flags = oracle.check_hex(X)
        if not flags["near_boundary"]:
            if res["lower"] > 0:
                assert (flags["flags"] & 3) == oracle.VALID
            if res["upper"] <= 0:
                assert (flags["flags"] & 3) == oracle.INVALID


def test_select_valid_brute_force():
    """NEXT-3 oracle against a plain loop on small inputs (all flag values, empty groups)."""
    rng = np.random.default_rng(51)
    for n in (0, 1, 17, 1000):
        flags = rng.choice(np.array([0, 1, 2, 3, 4, 5, 6], np.uint8), size=n)
        group = rng.integers(0, 7, size=n).astype(np.int32)
        ids, counts = oracle.select_valid(flags, group, 9)
        exp_ids = [i for i in range(n) if flags[i] & 3 == 1]
        exp_counts = [sum(1 for i in exp_ids if group[i] == g) for g in range(9)]
        assert ids.tolist() == exp_ids and counts.tolist() == exp_counts


# --------------------------------------------------------------------------
# NEXT-4: linear quadrangle
# --------------------------------------------------------------------------

SQ = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=np.float64)


def _quad_detj(Q, xi, eta):
    """det J of the bilinear map from the shape functions of PAPER.md:290-297 (independent)."""
    xi = np.asarray(xi, dtype=np.float64)[..., None]
    eta = np.asarray(eta, dtype=np.float64)[..., None]
    dxi = -(1 - eta) * Q[0] + (1 - eta) * Q[1] + eta * Q[2] - eta * Q[3]
    deta = -(1 - xi) * Q[0] - xi * Q[1] + xi * Q[2] + (1 - xi) * Q[3]
    return dxi[..., 0] * deta[..., 1] - dxi[..., 1] * deta[..., 0]


def test_quad_special_cases():
    """Unit square valid; bowtie (nodes 3, 4 swapped: self-intersecting) and chevron
    (non-convex: one corner reflex) invalid; a mirrored square is invalid."""
    assert oracle.check_quad(SQ)["flags"] == oracle.VALID
    assert np.array_equal(oracle.check_quad(SQ)["J"], [1, 1, 1, 1])
    assert oracle.check_quad(SQ[[0, 1, 3, 2]])["flags"] == oracle.INVALID
    chevron = np.array([[0, 0], [2, 0], [1, 0.5], [0, 2]], dtype=np.float64)
    assert oracle.check_quad(chevron)["flags"] == oracle.INVALID
    assert oracle.check_quad(SQ * [-1, 1])["flags"] == oracle.INVALID
    bad = SQ.copy(); bad[2, 0] = np.nan
    assert oracle.check_quad(bad)["flags"] == oracle.NONFINITE


def test_quad_corner_values_identity_and_areas():
    """J_k = det J at corner k = twice the signed area of the corner triangle, and
    J1 + J3 = J2 + J4; affine quads have four equal values."""
    rng = np.random.default_rng(61)
    corners = [(0, 0), (1, 0), (1, 1), (0, 1)]
    tri = [(0, 1, 3), (1, 2, 0), (2, 3, 1), (3, 0, 2)]       # corner k and its two neighbours, ccw
    for _ in range(300):
        Q = SQ + rng.uniform(-0.4, 0.4, size=(4, 2))
        r = oracle.check_quad(Q)
        for k in range(4):
            assert abs(r["J"][k] - _quad_detj(Q, *corners[k])) <= 1e-14
            a, b, c = Q[list(tri[k])]
            area2 = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0])
            assert abs(r["J"][k] - area2) <= 1e-14
        J = r["J"]
        assert abs(J[0] + J[2] - J[1] - J[3]) <= 1e-14
        A = rng.normal(size=(2, 2))
        P = SQ @ A.T + rng.normal(size=2)
        assert np.allclose(oracle.check_quad(P)["J"], np.linalg.det(A), atol=1e-14)


def test_quad_brute_force_and_exact_orientation():
    """Dense sampling never contradicts a verdict (det J is bilinear: its minimum is a
    corner value); the exact orientation sign agrees with Python rationals, including
    collinear (exactly zero) configurations, which are INVALID (reading G2)."""
    rng = np.random.default_rng(62)
    t = np.linspace(0, 1, 21)
    XI, ETA = np.meshgrid(t, t, indexing="ij")
    for _ in range(300):
        Q = SQ + rng.uniform(-0.6, 0.6, size=(4, 2))
        r = oracle.check_quad(Q)
        v = _quad_detj(Q, XI, ETA)
        if r["flags"] == oracle.VALID:
            assert v.min() > -1e-14
        else:
            assert min(r["J"]) <= 1e-14
    for _ in range(200):
        a = rng.integers(-4, 5, size=2) / 8.0
        d = rng.integers(-4, 5, size=2) / 8.0
        b = a + d
        c = a + d * rng.integers(-3, 4)                         # collinear with a, b
        for p, q, s in ((a, b, c), (a, b, rng.normal(size=2))):
            ex = (Fraction(q[0]) - Fraction(p[0])) * (Fraction(s[1]) - Fraction(p[1])) - \
                 (Fraction(q[1]) - Fraction(p[1])) * (Fraction(s[0]) - Fraction(p[0]))
            assert oracle.exact_orient2d(p, q, s) == (ex > 0) - (ex < 0)
    Q = SQ.copy(); Q[2] = [1.0, 0.0]                             # node 3 on node 2: J2 = J3 = 0 exactly
    assert oracle.check_quad(Q)["flags"] == oracle.INVALID


def test_corner_quality_indexed_driver_equals_soa_driver():
    """The indexed batch driver gathers the same 8 nodes as the SoA one (config-3 candidates,
    duplicates included): identical outputs."""
    verts, idx = hexgen.indexed_config(3, start=123, count=3000)
    a = oracle.corner_quality_indexed(verts, idx)
    b = oracle.corner_quality_soa(hexgen.indexed_to_soa(verts, idx))
    for k in ("test1", "near"):
        assert np.array_equal(a[k], b[k])
    assert np.array_equal(np.isnan(a["sj_min"]), np.isnan(b["sj_min"]))
    ok = ~np.isnan(a["sj_min"])
    assert np.array_equal(a["sj_min"][ok], b["sj_min"][ok])
