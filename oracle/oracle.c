/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the robust
 * validity check of linear hexahedra (PAPER.md, Johnen-Weill-Remacle 2017).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Compiled with -O2
 * -ffp-contract=off, no fast-math, scalar code.  Shares nothing with the CUDA
 * path: it evaluates det J analytically at all 27 nodes (the plain definition,
 * Eq. e:det3d with the section 5 derivative formulas) and applies the dense
 * Table 1 matrix T_b, while the CUDA path uses the paper's 20 tetrahedron
 * determinants and the sparse Table 3 matrix.
 *
 * Readings of the paper that this file takes (SURVEY.md
 * 8(c) G1-G14):
 *   G2  "negative" in Step 2 / recursion Step 3 means <= 0 (strict positivity,
 *       PAPER.md:263-264); "positive" means > 0.
 *   G3  sub-coefficients: per-axis quadratic de Casteljau at t = 1/2, axis
 *       order xi, eta, zeta.
 *   G4  children visited in Fig. 3 corner order; INVALID returns at once;
 *       INVALID > UNDETERMINED > VALID.
 *   G5  max depth 20: children at depth 20 are classified but not split.
 *   G8  fp sign decisions with zero tolerance 0; the 20 root samples whose
 *       |c| <= tau are re-decided in exact integer arithmetic.
 *   G13 NONFINITE (flags 3) iff a coordinate is NaN/Inf or |x| > 2^300.
 *   G14 near-boundary iff some fp decision had |min| <= tau(depth).
 */
#include "oracle.h"

#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* -------------------------------------------------------------------------
 * Node / coefficient ordering: Fig. 3.  XI2[sigma] = 2*xi.
 * b_1 = b_000, b_2 = b_200, b_9 = b_100.
 * ---------------------------------------------------------------------- */
static const int XI2[27][3] = {
    {0, 0, 0}, {2, 0, 0}, {2, 2, 0}, {0, 2, 0},   /* 1-4  corners, bottom  */
    {0, 0, 2}, {2, 0, 2}, {2, 2, 2}, {0, 2, 2},   /* 5-8  corners, top     */
    {1, 0, 0}, {2, 1, 0}, {1, 2, 0}, {0, 1, 0},   /* 9-12 edges 12 23 34 41 */
    {0, 0, 1}, {2, 0, 1}, {2, 2, 1}, {0, 2, 1},   /* 13-16 edges 15 26 37 48 */
    {1, 0, 2}, {2, 1, 2}, {1, 2, 2}, {0, 1, 2},   /* 17-20 edges 56 67 78 85 */
    {1, 1, 0}, {1, 0, 1}, {2, 1, 1},              /* 21-23 faces            */
    {1, 2, 1}, {0, 1, 1}, {1, 1, 2},              /* 24-26 faces            */
    {1, 1, 1}};                                   /* 27 centre              */

void oracle_node_xi(int sigma, double xi[3]) {
    for (int a = 0; a < 3; ++a) xi[a] = 0.5 * XI2[sigma][a];
}

/* -------------------------------------------------------------------------
 * Table 1: T_b, b = T_b c.  Written row block by row
 * block exactly as printed:
 *   rows 1-8    : I_8 on c_1..c_8
 *   rows 9-20   : -1/2 on the edge's two end corners, 2 I_12 on c_9..c_20
 *   rows 21-26  : 1/4 on the face's 4 corners, -1 on its 4 edges, 4 I_6
 *   row 27      : -1/8 on all corners, 1/2 on all edges, -2 on all faces, 8
 * ---------------------------------------------------------------------- */
static const int EDGE_ENDS[12][2] = {      /* paper node numbers */
    {1, 2}, {2, 3}, {3, 4}, {1, 4}, {1, 5}, {2, 6},
    {3, 7}, {4, 8}, {5, 6}, {6, 7}, {7, 8}, {5, 8}};
static const int FACE_CORNERS[6][4] = {
    {1, 2, 3, 4}, {1, 2, 5, 6}, {2, 3, 6, 7}, {3, 4, 7, 8}, {1, 4, 5, 8}, {5, 6, 7, 8}};
static const int FACE_EDGES[6][4] = {      /* PAPER.md:681-686, columns 9..20 */
    {9, 10, 11, 12}, {9, 13, 14, 17}, {10, 14, 15, 18},
    {11, 15, 16, 19}, {12, 13, 16, 20}, {17, 18, 19, 20}};

void oracle_tb_matrix(double T[27][27]) {
    memset(T, 0, sizeof(double) * 27 * 27);
    for (int k = 0; k < 8; ++k) T[k][k] = 1.0;
    for (int e = 0; e < 12; ++e) {
        int row = 8 + e;
        T[row][EDGE_ENDS[e][0] - 1] = -0.5;
        T[row][EDGE_ENDS[e][1] - 1] = -0.5;
        T[row][row] = 2.0;
    }
    for (int f = 0; f < 6; ++f) {
        int row = 20 + f;
        for (int q = 0; q < 4; ++q) {
            T[row][FACE_CORNERS[f][q] - 1] = 0.25;
            T[row][FACE_EDGES[f][q] - 1] = -1.0;
        }
        T[row][row] = 4.0;
    }
    for (int k = 0; k < 8; ++k) T[26][k] = -0.125;
    for (int e = 8; e < 20; ++e) T[26][e] = 0.5;
    for (int f = 20; f < 26; ++f) T[26][f] = -2.0;
    T[26][26] = 8.0;
}

void oracle_bezier_from_samples(const double c[27], double b[27]) {
    double T[27][27];
    oracle_tb_matrix(T);
    for (int s = 0; s < 27; ++s) {        /* plain matrix-vector product */
        double acc = 0.0;
        for (int t = 0; t < 27; ++t) acc += T[s][t] * c[t];
        b[s] = acc;
    }
}

/* -------------------------------------------------------------------------
 * The trilinear map and its Jacobian (PAPER.md:160-168, 416-423, 838-845,
 * App. A 1360-1378).  v_ij = n_j - n_i with the paper's 1-based node numbers.
 * ---------------------------------------------------------------------- */
typedef struct {
    double v12[3], v43[3], v56[3], v87[3];   /* d/dxi   edges */
    double v14[3], v23[3], v58[3], v67[3];   /* d/deta  edges */
    double v15[3], v26[3], v48[3], v37[3];   /* d/dzeta edges */
} edges_t;

static void edge_vectors(const double X[8][3], edges_t* E) {
    for (int a = 0; a < 3; ++a) {
        E->v12[a] = X[1][a] - X[0][a];
        E->v43[a] = X[2][a] - X[3][a];
        E->v56[a] = X[5][a] - X[4][a];
        E->v87[a] = X[6][a] - X[7][a];
        E->v14[a] = X[3][a] - X[0][a];
        E->v23[a] = X[2][a] - X[1][a];
        E->v58[a] = X[7][a] - X[4][a];
        E->v67[a] = X[6][a] - X[5][a];
        E->v15[a] = X[4][a] - X[0][a];
        E->v26[a] = X[5][a] - X[1][a];
        E->v48[a] = X[7][a] - X[3][a];
        E->v37[a] = X[6][a] - X[2][a];
    }
}

/* d/dxi x, d/deta x, d/dzeta x at (xi, eta, zeta), plus the
 * componentwise bounds sum |w||v| used by the rounding-error bound tau. */
static void derivatives(const edges_t* E, const double xi[3], double J[3][3], double Jabs[3][3]) {
    const double x = xi[0], y = xi[1], z = xi[2];
    const double w_xi[4] = {(1 - y) * (1 - z), y * (1 - z), (1 - y) * z, y * z};
    const double w_eta[4] = {(1 - x) * (1 - z), x * (1 - z), (1 - x) * z, x * z};
    const double w_zeta[4] = {(1 - x) * (1 - y), x * (1 - y), (1 - x) * y, x * y};
    for (int a = 0; a < 3; ++a) {
        const double dxi[4] = {E->v12[a], E->v43[a], E->v56[a], E->v87[a]};
        const double deta[4] = {E->v14[a], E->v23[a], E->v58[a], E->v67[a]};
        const double dzeta[4] = {E->v15[a], E->v26[a], E->v48[a], E->v37[a]};
        J[0][a] = w_xi[0] * dxi[0] + w_xi[1] * dxi[1] + w_xi[2] * dxi[2] + w_xi[3] * dxi[3];
        J[1][a] = w_eta[0] * deta[0] + w_eta[1] * deta[1] + w_eta[2] * deta[2] + w_eta[3] * deta[3];
        J[2][a] = w_zeta[0] * dzeta[0] + w_zeta[1] * dzeta[1] + w_zeta[2] * dzeta[2] + w_zeta[3] * dzeta[3];
        Jabs[0][a] = fabs(w_xi[0] * dxi[0]) + fabs(w_xi[1] * dxi[1]) + fabs(w_xi[2] * dxi[2]) + fabs(w_xi[3] * dxi[3]);
        Jabs[1][a] = fabs(w_eta[0] * deta[0]) + fabs(w_eta[1] * deta[1]) + fabs(w_eta[2] * deta[2]) + fabs(w_eta[3] * deta[3]);
        Jabs[2][a] = fabs(w_zeta[0] * dzeta[0]) + fabs(w_zeta[1] * dzeta[1]) + fabs(w_zeta[2] * dzeta[2]) + fabs(w_zeta[3] * dzeta[3]);
    }
}

/* Eq. e:det3d: det J = sum_{ijk} eps_ijk (d_xi x_i)(d_eta x_j)(d_zeta x_k). */
static const int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
static const int PERM_SIGN[6] = {+1, -1, -1, +1, +1, -1};

static double det_eps(const double J[3][3]) {
    double s = 0.0;
    for (int p = 0; p < 6; ++p)
        s += PERM_SIGN[p] * (J[0][PERM[p][0]] * J[1][PERM[p][1]] * J[2][PERM[p][2]]);
    return s;
}

static double permanent_abs(const double A[3][3]) {
    double s = 0.0;
    for (int p = 0; p < 6; ++p) s += A[0][PERM[p][0]] * A[1][PERM[p][1]] * A[2][PERM[p][2]];
    return s;
}

static double max_abs3x3(const double A[3][3]) {
    double m = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m = fmax(m, fabs(A[i][j]));
    return m;
}

double oracle_detj(const double X[8][3], const double xi[3]) {
    edges_t E;
    double J[3][3], Ja[3][3];
    edge_vectors(X, &E);
    derivatives(&E, xi, J, Ja);
    return det_eps(J);
}

void oracle_samples27(const double X[8][3], double c[27]) {
    for (int s = 0; s < 27; ++s) {
        double xi[3];
        oracle_node_xi(s, xi);
        c[s] = oracle_detj(X, xi);
    }
}

/* Eq. e:bezDefinition / e:bezExpansion: sum_ijk b_ijk B_i(xi) B_j(eta) B_k(zeta). */
static double bernstein2(int i, double t) {
    if (i == 0) return (1 - t) * (1 - t);
    if (i == 1) return 2 * t * (1 - t);
    return t * t;
}

double oracle_bezier_eval(const double b[27], const double xi[3]) {
    double s = 0.0;
    for (int sg = 0; sg < 27; ++sg)
        s += b[sg] * bernstein2(XI2[sg][0], xi[0]) * bernstein2(XI2[sg][1], xi[1]) *
             bernstein2(XI2[sg][2], xi[2]);
    return s;
}

/* -------------------------------------------------------------------------
 * Sub-coefficients ("as described in [johnen2013]";
 * reading G3): tensor-product quadratic de Casteljau at t = 1/2.  For a line
 * (p0, p1, p2): m01 = (p0+p1)/2, m12 = (p1+p2)/2, m = (m01+m12)/2; left half
 * (p0, m01, m), right half (m, m12, p2).  Child o contains corner o (Fig. 3)
 * and covers prod_a [kappa_a/2, (kappa_a+1)/2].
 * ---------------------------------------------------------------------- */
void oracle_subdivide(const double b[27], int child, double out[27]) {
    double B[3][3][3];
    for (int s = 0; s < 27; ++s) B[XI2[s][0]][XI2[s][1]][XI2[s][2]] = b[s];
    const int kap[3] = {XI2[child][0] / 2, XI2[child][1] / 2, XI2[child][2] / 2};
    for (int axis = 0; axis < 3; ++axis) {          /* xi, then eta, then zeta */
        for (int u = 0; u < 3; ++u)
            for (int w = 0; w < 3; ++w) {
                double *p0, *p1, *p2;
                if (axis == 0) { p0 = &B[0][u][w]; p1 = &B[1][u][w]; p2 = &B[2][u][w]; }
                else if (axis == 1) { p0 = &B[u][0][w]; p1 = &B[u][1][w]; p2 = &B[u][2][w]; }
                else { p0 = &B[u][w][0]; p1 = &B[u][w][1]; p2 = &B[u][w][2]; }
                const double m01 = 0.5 * (*p0 + *p1);
                const double m12 = 0.5 * (*p1 + *p2);
                const double m = 0.5 * (m01 + m12);
                if (kap[axis] == 0) { *p1 = m01; *p2 = m; }
                else { *p0 = m; *p1 = m12; }
            }
    }
    for (int s = 0; s < 27; ++s) out[s] = B[XI2[s][0]][XI2[s][1]][XI2[s][2]];
}

/* -------------------------------------------------------------------------
 * Exact sign of det J(xi_sigma): plain signed big integers.
 * Every double is m * 2^e with an integer m; multiplying all 24 coordinates
 * by 2^-emin makes them integers, and 4 * d/dxi x at xi in {0,1/2,1}^3 is an
 * integer combination of the integer edge vectors, so
 *     sign det J(xi_sigma) = sign det(4 d_xi x, 4 d_eta x, 4 d_zeta x)
 * is an integer computation (Eq. e:det3d, same Leibniz sum).
 * ---------------------------------------------------------------------- */
#define BIG_LIMBS 200
typedef struct {
    int neg;                 /* 1 if negative (never set for zero) */
    int n;                   /* limbs in use; 0 means zero */
    uint32_t d[BIG_LIMBS];   /* little-endian base 2^32 magnitude */
} big;

static void big_norm(big* a) {
    while (a->n > 0 && a->d[a->n - 1] == 0) a->n--;
    if (a->n == 0) a->neg = 0;
}

static void big_set_shifted(big* a, int64_t m, int shift) {   /* m * 2^shift, shift >= 0 */
    memset(a, 0, sizeof(*a));
    if (m == 0) return;
    uint64_t mag = m < 0 ? (uint64_t)(-m) : (uint64_t)m;
    a->neg = m < 0;
    int limb = shift / 32, bit = shift % 32;
    /* 64-bit magnitude shifted by bit lands in at most 3 limbs */
    uint64_t lo = (mag << bit) & 0xffffffffu;
    uint64_t mid = (bit == 0) ? (mag >> 32) : ((mag >> (32 - bit)) & 0xffffffffu);
    uint64_t hi = (bit == 0) ? 0 : (mag >> (64 - bit));
    if (limb + 3 > BIG_LIMBS) abort();
    a->d[limb] = (uint32_t)lo;
    a->d[limb + 1] = (uint32_t)mid;
    a->d[limb + 2] = (uint32_t)hi;
    a->n = limb + 3;
    big_norm(a);
}

static int mag_cmp(const big* a, const big* b) {
    if (a->n != b->n) return a->n > b->n ? 1 : -1;
    for (int i = a->n - 1; i >= 0; --i)
        if (a->d[i] != b->d[i]) return a->d[i] > b->d[i] ? 1 : -1;
    return 0;
}

static void mag_add(const big* a, const big* b, big* r) {      /* |r| = |a| + |b| */
    int n = a->n > b->n ? a->n : b->n;
    uint64_t carry = 0;
    big t;
    memset(&t, 0, sizeof(t));
    for (int i = 0; i < n; ++i) {
        uint64_t s = carry + (i < a->n ? a->d[i] : 0) + (i < b->n ? b->d[i] : 0);
        t.d[i] = (uint32_t)s;
        carry = s >> 32;
    }
    if (carry) {
        if (n >= BIG_LIMBS) abort();
        t.d[n++] = (uint32_t)carry;
    }
    t.n = n;
    *r = t;
}

static void mag_sub(const big* a, const big* b, big* r) {      /* |r| = |a| - |b|, |a| >= |b| */
    int64_t borrow = 0;
    big t;
    memset(&t, 0, sizeof(t));
    for (int i = 0; i < a->n; ++i) {
        int64_t s = (int64_t)a->d[i] - (i < b->n ? b->d[i] : 0) - borrow;
        borrow = s < 0;
        t.d[i] = (uint32_t)(s + (borrow ? ((int64_t)1 << 32) : 0));
    }
    t.n = a->n;
    *r = t;
}

static void big_add(const big* a, const big* b, big* r) {      /* r = a + b (signed) */
    big t;
    if (a->neg == b->neg) {
        mag_add(a, b, &t);
        t.neg = a->neg;
    } else if (mag_cmp(a, b) >= 0) {
        mag_sub(a, b, &t);
        t.neg = a->neg;
    } else {
        mag_sub(b, a, &t);
        t.neg = b->neg;
    }
    big_norm(&t);
    *r = t;
}

static void big_sub(const big* a, const big* b, big* r) {
    big nb = *b;
    if (nb.n) nb.neg = !nb.neg;
    big_add(a, &nb, r);
}

static void big_mul(const big* a, const big* b, big* r) {      /* schoolbook */
    big t;
    memset(&t, 0, sizeof(t));
    if (a->n == 0 || b->n == 0) { *r = t; return; }
    if (a->n + b->n > BIG_LIMBS) abort();
    for (int i = 0; i < a->n; ++i) {
        uint64_t carry = 0;
        for (int j = 0; j < b->n; ++j) {
            uint64_t cur = (uint64_t)a->d[i] * b->d[j] + t.d[i + j] + carry;
            t.d[i + j] = (uint32_t)cur;
            carry = cur >> 32;
        }
        t.d[i + b->n] = (uint32_t)carry;
    }
    t.n = a->n + b->n;
    t.neg = a->neg != b->neg;
    big_norm(&t);
    *r = t;
}

static void big_mul_int(const big* a, int64_t s, big* r) {
    big bs;
    big_set_shifted(&bs, s, 0);
    big_mul(a, &bs, r);
}

static int big_sign(const big* a) { return a->n == 0 ? 0 : (a->neg ? -1 : 1); }

int oracle_exact_sign(const double X[8][3], int sigma) {
    /* integer coordinates: x = m 2^e  ->  m 2^(e - emin) */
    int64_t mant[8][3];
    int expo[8][3];
    int emin = INT32_MAX;
    for (int k = 0; k < 8; ++k)
        for (int a = 0; a < 3; ++a) {
            int e = 0;
            double f = frexp(X[k][a], &e);               /* X = f 2^e, 1/2 <= |f| < 1 */
            mant[k][a] = (int64_t)ldexp(f, 53);          /* exact: at most 53 bits */
            expo[k][a] = e - 53;
            if (mant[k][a] != 0 && expo[k][a] < emin) emin = expo[k][a];
        }
    if (emin == INT32_MAX) return 0;                     /* all coordinates zero */
    big P[8][3];
    for (int k = 0; k < 8; ++k)
        for (int a = 0; a < 3; ++a) big_set_shifted(&P[k][a], mant[k][a], expo[k][a] - emin);
    /* integer weights 4*w for the node xi_sigma = XI2/2 */
    const int i2 = XI2[sigma][0], j2 = XI2[sigma][1], k2 = XI2[sigma][2];
    const int64_t w_xi[4] = {(2 - j2) * (2 - k2), j2 * (2 - k2), (2 - j2) * k2, j2 * k2};
    const int64_t w_eta[4] = {(2 - i2) * (2 - k2), i2 * (2 - k2), (2 - i2) * k2, i2 * k2};
    const int64_t w_zeta[4] = {(2 - i2) * (2 - j2), i2 * (2 - j2), (2 - i2) * j2, i2 * j2};
    /* (to, from) node pairs of the edge vectors (0-based): v12 v43 v56 v87 | v14 v23 v58 v67 | v15 v26 v48 v37 */
    static const int EV[3][4][2] = {
        {{1, 0}, {2, 3}, {5, 4}, {6, 7}},
        {{3, 0}, {2, 1}, {7, 4}, {6, 5}},
        {{4, 0}, {5, 1}, {7, 3}, {6, 2}}};
    const int64_t* W[3] = {w_xi, w_eta, w_zeta};
    big D[3][3];                                          /* D[dir][axis] = 4 d_dir x_axis */
    for (int dir = 0; dir < 3; ++dir)
        for (int a = 0; a < 3; ++a) {
            big acc;
            memset(&acc, 0, sizeof(acc));
            for (int q = 0; q < 4; ++q) {
                if (W[dir][q] == 0) continue;
                big v, wv;
                big_sub(&P[EV[dir][q][0]][a], &P[EV[dir][q][1]][a], &v);
                big_mul_int(&v, W[dir][q], &wv);
                big_add(&acc, &wv, &acc);
            }
            D[dir][a] = acc;
        }
    big det;
    memset(&det, 0, sizeof(det));
    for (int p = 0; p < 6; ++p) {
        big t1, t2;
        big_mul(&D[0][PERM[p][0]], &D[1][PERM[p][1]], &t1);
        big_mul(&t1, &D[2][PERM[p][2]], &t2);
        if (PERM_SIGN[p] > 0) big_add(&det, &t2, &det);
        else big_sub(&det, &t2, &det);
    }
    return big_sign(&det);
}

/* -------------------------------------------------------------------------
 * The algorithm, section 6 (lines 1105-1145).
 * ---------------------------------------------------------------------- */
#define U_ROUND (1.0 / 9007199254740992.0)     /* u = 2^-53 */

typedef struct {
    double E, Mb;            /* scale of the hex: edge components, max |b_root| */
    double min_ratio;        /* min |decision value| / tau(depth) */
    int64_t nodes;
    int max_depth;
    int undetermined;
    double witness[3];
    double witness_value;
} rec_ctx;

/* Combined (oracle + any implementation of the same bound) rounding-error
 * bound for a Bezier value at subdivision depth d:
 * E = max |edge-vector component| of the hex, Mb = max |b_root|.  Pinned
 * against exact rational arithmetic by tests/test_tau_bounds.py. */
double oracle_tau_depth(double E, double Mb, int depth) {
    return 16384.0 * U_ROUND * E * E * E + 16.0 * depth * U_ROUND * Mb +
           ldexp(1.0, -1040) * (1.0 + E * E);
}

static double tau_depth(const rec_ctx* ctx, int depth) {
    return oracle_tau_depth(ctx->E, ctx->Mb, depth);
}

static void note_decision(rec_ctx* ctx, double value, int depth) {
    const double r = fabs(value) / tau_depth(ctx, depth);
    if (r < ctx->min_ratio) ctx->min_ratio = r;
}

static double min_range(const double* v, int lo, int hi) {
    double m = v[lo];
    for (int i = lo + 1; i < hi; ++i) m = v[i] < m ? v[i] : m;
    return m;
}

/* recursive_subdivision(b) of PAPER.md:1129-1137.  `node` lives at depth
 * `depth` on the dyadic box origin + [0, size]^3.  Returns 0 (False/INVALID)
 * or 1 (True: positive or capped).  ctx->undetermined records caps. */
static int recursive_subdivision(const double node[27], int depth, const double origin[3],
                                 double size, rec_ctx* ctx) {
    ctx->nodes++;
    for (int o = 0; o < 8; ++o) {                         /* Step 2: for each b^i */
        double child[27];
        oracle_subdivide(node, o, child);                  /* Step 1 */
        const int cd = depth + 1;
        if (cd > ctx->max_depth) ctx->max_depth = cd;
        const double half = 0.5 * size;
        double corg[3];
        for (int a = 0; a < 3; ++a) corg[a] = origin[a] + half * (XI2[o][a] / 2);
        /* Step 3: a corner coefficient (true det J value) <= 0 -> False */
        const double mc = min_range(child, 0, 8);
        note_decision(ctx, mc, cd);
        if (mc <= 0.0) {
            for (int k = 0; k < 8; ++k)
                if (child[k] <= 0.0) {
                    for (int a = 0; a < 3; ++a) ctx->witness[a] = corg[a] + half * (XI2[k][a] / 2);
                    ctx->witness_value = child[k];
                    break;
                }
            return 0;
        }
        /* Step 4: all of b^i_9..27 > 0 -> continue */
        const double mi = min_range(child, 8, 27);
        note_decision(ctx, mi, cd);
        if (mi > 0.0) continue;
        /* depth cap (reading G5) */
        if (cd >= ORACLE_MAX_DEPTH) {
            ctx->undetermined = 1;
            continue;
        }
        /* Step 5 */
        if (!recursive_subdivision(child, cd, corg, half, ctx)) return 0;
    }
    return 1;                                             /* Step 6 */
}

static int coord_ok(double x) {
    return isfinite(x) && fabs(x) <= 0x1p300;
}

/* Rounding-error bound of the oracle's fp det J sample from the componentwise
 * magnitudes Ja of its Jacobian columns (triple product with
 * rounded inputs, 32 u perm(|J|), plus an underflow term).  Decides when Step 2
 * falls back to the exact sign (reading G8); pinned by tests/test_tau_bounds.py. */
static double sample_tau(const double Ja[3][3]) {
    const double dmax = max_abs3x3(Ja);
    return 32.0 * U_ROUND * permanent_abs(Ja) + ldexp(1.0, -1060) * (1.0 + 6.0 * dmax * dmax);
}

double oracle_sample_tau(const double X[8][3], int sigma) {
    edges_t Ev;
    double xi[3], J[3][3], Ja[3][3];
    edge_vectors(X, &Ev);
    oracle_node_xi(sigma, xi);
    derivatives(&Ev, xi, J, Ja);
    return sample_tau(Ja);
}

int oracle_check_hex(const double X[8][3], oracle_result* r) {
    memset(r, 0, sizeof(*r));
    r->margin_ratio = INFINITY;
    r->witness_value = NAN;
    for (int k = 0; k < 8; ++k)
        for (int a = 0; a < 3; ++a)
            if (!coord_ok(X[k][a])) {
                r->verdict = ORACLE_NONFINITE;
                r->flags = ORACLE_NONFINITE;
                for (int s = 0; s < 27; ++s) r->c[s] = r->b[s] = NAN;
                return r->flags;
            }

    edges_t Ev;
    edge_vectors(X, &Ev);
    double E = 0.0;
    {
        const double* vs[12] = {Ev.v12, Ev.v43, Ev.v56, Ev.v87, Ev.v14, Ev.v23,
                                Ev.v58, Ev.v67, Ev.v15, Ev.v26, Ev.v48, Ev.v37};
        for (int q = 0; q < 12; ++q)
            for (int a = 0; a < 3; ++a) E = fmax(E, fabs(vs[q][a]));
    }
    r->E = E;

    /* Step 1: the Jacobian determinant at the 27 nodes (the first 20 are the
     * paper's 20 "volumes" times 6; the oracle evaluates the
     * definition directly). */
    double tau_c[27];
    for (int s = 0; s < 27; ++s) {
        double xi[3], J[3][3], Ja[3][3];
        oracle_node_xi(s, xi);
        derivatives(&Ev, xi, J, Ja);
        r->c[s] = det_eps(J);
        tau_c[s] = sample_tau(Ja);
    }

    /* Step 2: if at least one of the 20 values is <= 0, return False.  Values
     * within their rounding bound of 0 are decided exactly (reading G8). */
    int invalid = 0;
    for (int s = 0; s < 20 && !invalid; ++s) {
        int sign;
        if (fabs(r->c[s]) <= tau_c[s]) {
            sign = oracle_exact_sign(X, s);
            r->exact_used++;
        } else {
            sign = r->c[s] > 0.0 ? 1 : -1;
        }
        if (sign <= 0) {
            invalid = 1;
            oracle_node_xi(s, r->witness);
            r->witness_value = r->c[s];
        }
    }

    /* Step 3: b = T_b c (Table 1; equal to Table 3 applied to c_1..20 by Cor. 1) */
    oracle_bezier_from_samples(r->c, r->b);
    if (invalid) {
        r->verdict = ORACLE_INVALID;
        r->flags = ORACLE_INVALID;
        return r->flags;
    }

    rec_ctx ctx;
    memset(&ctx, 0, sizeof(ctx));
    ctx.E = E;
    for (int s = 0; s < 27; ++s) ctx.Mb = fmax(ctx.Mb, fabs(r->b[s]));
    ctx.min_ratio = INFINITY;

    /* Step 4: all b_9..27 > 0 -> True */
    const double m4 = min_range(r->b, 8, 27);
    note_decision(&ctx, m4, 0);
    if (m4 > 0.0) {
        r->verdict = ORACLE_VALID;
    } else {
        /* Step 5: recursive_subdivision(b) */
        r->subdivided = 1;
        const double origin[3] = {0.0, 0.0, 0.0};
        const int ok = recursive_subdivision(r->b, 0, origin, 1.0, &ctx);
        if (!ok) {
            r->verdict = ORACLE_INVALID;
            memcpy(r->witness, ctx.witness, sizeof(ctx.witness));
            r->witness_value = ctx.witness_value;
        } else {
            r->verdict = ctx.undetermined ? ORACLE_UNDETERMINED : ORACLE_VALID;
        }
    }
    r->nodes = ctx.nodes;
    r->max_depth = ctx.max_depth;
    r->margin_ratio = ctx.min_ratio;
    r->near_boundary = ctx.min_ratio <= 1.0;
    r->flags = r->verdict | (r->subdivided ? ORACLE_FLAG_SUBDIVIDED : 0);
    return r->flags;
}

/* Steps 4-5 alone on a given coefficient vector (used by the tests to pin the
 * subdivision logic, e.g. the depth cap, on polynomials that are not det J). */
int oracle_classify_coeffs(const double b[27], double E, oracle_result* r) {
    memset(r, 0, sizeof(*r));
    memcpy(r->b, b, sizeof(double) * 27);
    r->E = E;
    r->witness_value = NAN;
    rec_ctx ctx;
    memset(&ctx, 0, sizeof(ctx));
    ctx.E = E;
    for (int s = 0; s < 27; ++s) ctx.Mb = fmax(ctx.Mb, fabs(b[s]));
    ctx.min_ratio = INFINITY;
    const double m4 = min_range(b, 8, 27);
    note_decision(&ctx, m4, 0);
    if (m4 > 0.0) {
        r->verdict = ORACLE_VALID;
    } else {
        r->subdivided = 1;
        const double origin[3] = {0.0, 0.0, 0.0};
        if (!recursive_subdivision(b, 0, origin, 1.0, &ctx)) {
            r->verdict = ORACLE_INVALID;
            memcpy(r->witness, ctx.witness, sizeof(ctx.witness));
            r->witness_value = ctx.witness_value;
        } else {
            r->verdict = ctx.undetermined ? ORACLE_UNDETERMINED : ORACLE_VALID;
        }
    }
    r->nodes = ctx.nodes;
    r->max_depth = ctx.max_depth;
    r->margin_ratio = ctx.min_ratio;
    r->near_boundary = ctx.min_ratio <= 1.0;
    r->flags = r->verdict | (r->subdivided ? ORACLE_FLAG_SUBDIVIDED : 0);
    return r->flags;
}

/* -------------------------------------------------------------------------
 * Batch drivers
 * ---------------------------------------------------------------------- */
int oracle_num_threads(int nthreads) {
#ifdef _OPENMP
    return nthreads > 0 ? nthreads : omp_get_max_threads();
#else
    (void)nthreads;
    return 1;
#endif
}

static void store_one(const oracle_result* r, int64_t i, int64_t n, uint8_t* flags_out,
                      double* coeffs_out, uint8_t* near_out, int64_t* nodes_out, uint8_t* exact_out) {
    if (flags_out) flags_out[i] = (uint8_t)r->flags;
    if (coeffs_out)
        for (int s = 0; s < 27; ++s) coeffs_out[(int64_t)s * n + i] = r->b[s];
    if (near_out) near_out[i] = (uint8_t)r->near_boundary;
    if (nodes_out) nodes_out[i] = r->nodes;
    if (exact_out) exact_out[i] = (uint8_t)(r->exact_used > 255 ? 255 : r->exact_used);
}

void oracle_check_soa(const double* coords, int64_t n, uint8_t* flags_out, double* coeffs_out,
                      uint8_t* near_out, int64_t* nodes_out, uint8_t* exact_out, int nthreads) {
    const int nt = oracle_num_threads(nthreads);
    (void)nt;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nt)
    for (int64_t i = 0; i < n; ++i) {
        double X[8][3];
        for (int k = 0; k < 8; ++k)
            for (int a = 0; a < 3; ++a) X[k][a] = coords[(int64_t)(3 * k + a) * n + i];
        oracle_result r;
        oracle_check_hex(X, &r);
        store_one(&r, i, n, flags_out, coeffs_out, near_out, nodes_out, exact_out);
    }
}

void oracle_check_indexed(const double* vertices, const int32_t* hex_idx, int64_t n,
                          uint8_t* flags_out, double* coeffs_out, uint8_t* near_out,
                          int64_t* nodes_out, uint8_t* exact_out, int nthreads) {
    const int nt = oracle_num_threads(nthreads);
    (void)nt;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nt)
    for (int64_t i = 0; i < n; ++i) {
        double X[8][3];
        for (int k = 0; k < 8; ++k)
            for (int a = 0; a < 3; ++a) X[k][a] = vertices[(int64_t)hex_idx[i * 8 + k] * 3 + a];
        oracle_result r;
        oracle_check_hex(X, &r);
        store_one(&r, i, n, flags_out, coeffs_out, near_out, nodes_out, exact_out);
    }
}

/* -------------------------------------------------------------------------
 * NEXT-2: corner screening quantities.
 * At corner sigma (0..7) the Jacobian columns are the three edge vectors
 * leaving the corner; the scaled Jacobian divides det J by
 * the product of their lengths.
 * ---------------------------------------------------------------------- */
void oracle_corner_quality(const double X[8][3], double* sj_min, int* test1, int* near) {
    for (int k = 0; k < 8; ++k)
        for (int a = 0; a < 3; ++a)
            if (!coord_ok(X[k][a])) {             /* NONFINITE input (reading G13) */
                *sj_min = NAN;
                *test1 = 0;
                *near = 0;
                return;
            }
    edges_t E;
    edge_vectors(X, &E);
    double m = INFINITY;
    int all_pos = 1, nr = 0, undefined = 0;
    for (int k = 0; k < 8; ++k) {
        double xi[3], J[3][3], Ja[3][3];
        oracle_node_xi(k, xi);
        derivatives(&E, xi, J, Ja);
        const double d = det_eps(J);
        /* reading G8, as in Step 2: a corner value within its rounding bound of 0
         * (sample_tau, pinned by tests/test_tau_bounds.py) takes its exact sign;
         * outside it the fp sign is the exact sign */
        const double tau = sample_tau(Ja);
        if (fabs(d) <= tau) {
            nr = 1;
            if (oracle_exact_sign(X, k) <= 0) all_pos = 0;
        } else if (d < 0.0) {
            all_pos = 0;
        }
        double len[3];
        for (int r = 0; r < 3; ++r) len[r] = sqrt(J[r][0] * J[r][0] + J[r][1] * J[r][1] + J[r][2] * J[r][2]);
        if (len[0] == 0.0 || len[1] == 0.0 || len[2] == 0.0) undefined = 1;
        const double sj = d / (len[0] * len[1] * len[2]);
        if (sj < m) m = sj;
    }
    *sj_min = undefined ? NAN : m;
    *test1 = all_pos;
    *near = nr;
}

void oracle_corner_quality_soa(const double* coords, int64_t n, double* sj_out, uint8_t* test1_out,
                               uint8_t* near_out, int nthreads) {
    const int nt = oracle_num_threads(nthreads);
    (void)nt;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nt)
    for (int64_t i = 0; i < n; ++i) {
        double X[8][3];
        for (int k = 0; k < 8; ++k)
            for (int a = 0; a < 3; ++a) X[k][a] = coords[(int64_t)(3 * k + a) * n + i];
        double sj;
        int t1, nr;
        oracle_corner_quality(X, &sj, &t1, &nr);
        if (sj_out) sj_out[i] = sj;
        if (test1_out) test1_out[i] = (uint8_t)t1;
        if (near_out) near_out[i] = (uint8_t)nr;
    }
}

void oracle_corner_quality_indexed(const double* vertices, const int32_t* hex_idx, int64_t n, double* sj_out,
                                   uint8_t* test1_out, uint8_t* near_out, int nthreads) {
    const int nt = oracle_num_threads(nthreads);
    (void)nt;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nt)
    for (int64_t i = 0; i < n; ++i) {
        double X[8][3];
        for (int k = 0; k < 8; ++k)
            for (int a = 0; a < 3; ++a) X[k][a] = vertices[(int64_t)hex_idx[i * 8 + k] * 3 + a];
        double sj;
        int t1, nr;
        oracle_corner_quality(X, &sj, &t1, &nr);
        if (sj_out) sj_out[i] = sj;
        if (test1_out) test1_out[i] = (uint8_t)t1;
        if (near_out) near_out[i] = (uint8_t)nr;
    }
}

/* -------------------------------------------------------------------------
 * NEXT-1: bounds on min det J (min b <= min det J <= min
 * of the corner coefficients; "sharpened as much as desired by subdividing").
 * ---------------------------------------------------------------------- */
static void bounds_rec(const double node[27], int depth, double tol, double* upper, double* lower,
                       int* capped, int64_t* nodes) {
    double child[8][27];
    (*nodes)++;
    for (int o = 0; o < 8; ++o) {                 /* children, and their corner values */
        oracle_subdivide(node, o, child[o]);
        const double mc = min_range(child[o], 0, 8);
        if (mc < *upper) *upper = mc;
    }
    for (int o = 0; o < 8; ++o) {
        const double m = min_range(child[o], 0, 27);
        if (m >= *upper - tol) {                  /* cannot hide a value below upper - tol */
            if (m < *lower) *lower = m;
        } else if (depth + 1 >= ORACLE_MAX_DEPTH) {
            if (m < *lower) *lower = m;
            *capped = 1;
        } else {
            bounds_rec(child[o], depth + 1, tol, upper, lower, capped, nodes);
        }
    }
}

void oracle_min_detj_bounds(const double X[8][3], double rel_tol, oracle_bounds* r) {
    memset(r, 0, sizeof(*r));
    for (int k = 0; k < 8; ++k)
        for (int a = 0; a < 3; ++a)
            if (!coord_ok(X[k][a])) {
                r->lower = r->upper = r->tol = NAN;
                return;
            }
    double c[27], b[27];
    oracle_samples27(X, c);
    oracle_bezier_from_samples(c, b);
    double scale = 0.0;
    for (int s = 0; s < 27; ++s) scale = fmax(scale, fabs(b[s]));
    r->tol = rel_tol * scale;
    r->upper = min_range(b, 0, 8);
    r->lower = INFINITY;
    const double m = min_range(b, 0, 27);
    if (m >= r->upper - r->tol) r->lower = m;
    else bounds_rec(b, 0, r->tol, &r->upper, &r->lower, &r->capped, &r->nodes);
}

void oracle_min_detj_bounds_soa(const double* coords, int64_t n, double rel_tol, double* lower_out,
                                double* upper_out, uint8_t* capped_out, int nthreads) {
    const int nt = oracle_num_threads(nthreads);
    (void)nt;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nt)
    for (int64_t i = 0; i < n; ++i) {
        double X[8][3];
        for (int k = 0; k < 8; ++k)
            for (int a = 0; a < 3; ++a) X[k][a] = coords[(int64_t)(3 * k + a) * n + i];
        oracle_bounds r;
        oracle_min_detj_bounds(X, rel_tol, &r);
        if (lower_out) lower_out[i] = r.lower;
        if (upper_out) upper_out[i] = r.upper;
        if (capped_out) capped_out[i] = (uint8_t)r.capped;
    }
}

/* -------------------------------------------------------------------------
 * NEXT-4: linear quadrangle, section 2.1 (lines 282-349): det J is
 * bilinear, its minimum is at a corner, so the element is valid iff the four
 * corner values are positive.
 * ---------------------------------------------------------------------- */
int oracle_exact_orient2d(const double a[2], const double b[2], const double c[2]) {
    /* (b-a) x (c-a) = a x b + b x c + c x a with u x v = u_x v_y - u_y v_x: 6 products of
     * input doubles, evaluated on integers after a common power-of-two scaling */
    const double* P[3] = {a, b, c};
    int64_t mant[3][2];
    int expo[3][2], emin = INT32_MAX;
    for (int k = 0; k < 3; ++k)
        for (int t = 0; t < 2; ++t) {
            int e = 0;
            const double f = frexp(P[k][t], &e);
            mant[k][t] = (int64_t)ldexp(f, 53);
            expo[k][t] = e - 53;
            if (mant[k][t] != 0 && expo[k][t] < emin) emin = expo[k][t];
        }
    if (emin == INT32_MAX) return 0;
    big B[3][2];
    for (int k = 0; k < 3; ++k)
        for (int t = 0; t < 2; ++t) big_set_shifted(&B[k][t], mant[k][t], expo[k][t] - emin);
    big acc;
    memset(&acc, 0, sizeof(acc));
    for (int k = 0; k < 3; ++k) {                 /* P_k x P_{k+1} */
        const int l = (k + 1) % 3;
        big t1, t2;
        big_mul(&B[k][0], &B[l][1], &t1);
        big_mul(&B[k][1], &B[l][0], &t2);
        big_add(&acc, &t1, &acc);
        big_sub(&acc, &t2, &acc);
    }
    return big_sign(&acc);
}

int oracle_check_quad(const double Q[4][2], double J[4], int* near) {
    *near = 0;
    for (int k = 0; k < 4; ++k)
        for (int a = 0; a < 2; ++a)
            if (!coord_ok(Q[k][a])) {
                for (int q = 0; q < 4; ++q) J[q] = NAN;
                return ORACLE_NONFINITE;
            }
    double v12[2], v43[2], v14[2], v23[2];
    for (int a = 0; a < 2; ++a) {
        v12[a] = Q[1][a] - Q[0][a];
        v43[a] = Q[2][a] - Q[3][a];
        v14[a] = Q[3][a] - Q[0][a];
        v23[a] = Q[2][a] - Q[1][a];
    }
    const double* U[4] = {v12, v12, v43, v43};
    const double* W[4] = {v14, v23, v23, v14};
    /* corner k as an orientation (origin, xi-neighbour, eta-neighbour) of input points */
    static const int ORI[4][3] = {{0, 1, 3}, {0, 1, 2}, {2, 3, 1}, {3, 0, 2}};
    int valid = 1;
    for (int k = 0; k < 4; ++k) {
        J[k] = U[k][0] * W[k][1] - U[k][1] * W[k][0];
        const double tau = 8.0 * U_ROUND * (fabs(U[k][0] * W[k][1]) + fabs(U[k][1] * W[k][0])) + ldexp(1.0, -1060);
        if (fabs(J[k]) <= tau) *near = 1;
        if (oracle_exact_orient2d(Q[ORI[k][0]], Q[ORI[k][1]], Q[ORI[k][2]]) <= 0) valid = 0;
    }
    return valid ? ORACLE_VALID : ORACLE_INVALID;
}

void oracle_check_quad_soa(const double* coords, int64_t n, uint8_t* flags_out, double* J_out,
                           uint8_t* near_out, int nthreads) {
    const int nt = oracle_num_threads(nthreads);
    (void)nt;
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t i = 0; i < n; ++i) {
        double Q[4][2], J[4];
        int nr;
        for (int k = 0; k < 4; ++k)
            for (int a = 0; a < 2; ++a) Q[k][a] = coords[(int64_t)(2 * k + a) * n + i];
        const int f = oracle_check_quad(Q, J, &nr);
        if (flags_out) flags_out[i] = (uint8_t)f;
        if (J_out)
            for (int k = 0; k < 4; ++k) J_out[(int64_t)k * n + i] = J[k];
        if (near_out) near_out[i] = (uint8_t)nr;
    }
}
