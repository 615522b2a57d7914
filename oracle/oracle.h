/*
 * oracle.h -- plain CPU oracle for the validity of linear hexahedra
 *             (Johnen, Weill, Remacle, "Robust and efficient validation of the
 *             linear hexahedral element", IMR26 2017; /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1706_01613_b200/csrc) and the CUDA path never calls it.
 *
 * Conventions (Fig. 3; Appendix A):
 *   X[k][a]   node k = 0..7 (paper's nodes 1..8), axis a = x,y,z.
 *   sigma     Bezier / sample index 0..26 (paper's 1..27); XI2[sigma] = 2*xi.
 *   flags     bits 0-1 verdict (0 INVALID, 1 VALID, 2 UNDETERMINED,
 *             3 NONFINITE), bit 2 SUBDIVIDED (root undecided after Step 4).
 */
#ifndef HEXVAL_ORACLE_H
#define HEXVAL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_INVALID 0
#define ORACLE_VALID 1
#define ORACLE_UNDETERMINED 2
#define ORACLE_NONFINITE 3
#define ORACLE_FLAG_SUBDIVIDED 4
#define ORACLE_MAX_DEPTH 20

typedef struct oracle_result {
    int verdict;            /* ORACLE_INVALID .. ORACLE_NONFINITE */
    int subdivided;         /* 1 iff Step 5 (recursive_subdivision) was entered */
    int flags;              /* verdict | (subdivided << 2) */
    int exact_used;         /* samples whose sign was taken in exact arithmetic */
    int near_boundary;      /* some fp sign decision had |value| <= tau */
    int max_depth;          /* deepest child depth classified (0 if none) */
    int64_t nodes;          /* number of recursive_subdivision calls */
    double margin_ratio;    /* min over fp decisions of |min(tested set)| / tau */
    double E;               /* max |component| over the 12 edge vectors */
    double c[27];           /* det J at the 27 uniform nodes (Eq. e:det3d) */
    double b[27];           /* Bezier coefficients b = T_b c (Table 1) */
    double witness[3];      /* reference point whose det J value decided INVALID */
    double witness_value;   /* that value (fp; exact sign when decided exactly) */
} oracle_result;

/* Whole algorithm of PAPER.md section 6 (lines 1105-1145) on one hexahedron. */
int oracle_check_hex(const double X[8][3], oracle_result* r);

/* Batch drivers (OpenMP over hexes; nthreads <= 0 means all cores).
 * coords: SoA, coords[(3*k+a)*n + i].  coeffs_out (optional): coeffs[s*n+i].
 * near_out / nodes_out / exact_out optional per-hex outputs. */
void oracle_check_soa(const double* coords, int64_t n, uint8_t* flags_out,
                      double* coeffs_out, uint8_t* near_out, int64_t* nodes_out,
                      uint8_t* exact_out, int nthreads);
void oracle_check_indexed(const double* vertices, const int32_t* hex_idx, int64_t n,
                          uint8_t* flags_out, double* coeffs_out, uint8_t* near_out,
                          int64_t* nodes_out, uint8_t* exact_out, int nthreads);

/* Pieces, exported so the tests can pin each one separately. */
double oracle_detj(const double X[8][3], const double xi[3]);          /* Eq. e:det3d */
void   oracle_samples27(const double X[8][3], double c[27]);           /* c_sigma = det J(xi_sigma) */
void   oracle_bezier_from_samples(const double c[27], double b[27]);   /* Table 1 */
void   oracle_tb_matrix(double T[27][27]);                             /* Table 1 as a dense matrix */
double oracle_bezier_eval(const double b[27], const double xi[3]);     /* Eq. e:bezExpansion */
void   oracle_subdivide(const double b[27], int child, double out[27]);/* de Casteljau, t = 1/2 */
int    oracle_exact_sign(const double X[8][3], int sigma);             /* sign of det J(xi_sigma), exact */
void   oracle_node_xi(int sigma, double xi[3]);                        /* xi_sigma */
int    oracle_num_threads(int nthreads);
/* Rounding-error bounds used by the readings G8 / G14:
 *   oracle_sample_tau   bound on |fl(det J(xi_sigma)) - det J(xi_sigma)| of oracle_samples27's
 *                       value; Step 2 re-decides a sample exactly when |c| <= it;
 *   oracle_tau_depth    combined bound (this oracle and the CUDA path) on a Bezier value at
 *                       subdivision depth `depth` of a hex with edge scale E and max |b_root| Mb;
 *                       a decision with |value| <= it marks the hex near-boundary. */
double oracle_sample_tau(const double X[8][3], int sigma);
double oracle_tau_depth(double E, double Mb, int depth);
/* Steps 4-5 on a given coefficient vector; E sets tau. */
int    oracle_classify_coeffs(const double b[27], double E, oracle_result* r);

/* NEXT-2, screening by-products of the 8 corner samples:
 *   sj_min  min over the 8 corners of the scaled Jacobian det J / (|d_xi x| |d_eta x| |d_zeta x|)
 *           at the corner (Fig. 7 caption "0.64"); NaN if a corner edge
 *           has zero length (the metric is undefined there, SPEC.md baselines);
 *   test1   1 iff det J > 0 at all 8 corners (Ushakova Test 1, the 8 corner tetrahedra,
 *           PAPER.md:107-109, 1260-1263), each sign decided exactly;
 *   near    1 iff some corner det J is within its fp64 rounding bound of 0.
 * A NONFINITE hex (reading G13) gives sj_min = NaN, test1 = 0. */
void   oracle_corner_quality(const double X[8][3], double* sj_min, int* test1, int* near);

/* NEXT-1, bounds on min det J (reading G15 in DESIGN.md):
 *   lower = min of the Bezier coefficients of the leaves of a subdivision tree (convex
 *           hull property), upper = min of all corner coefficients met (actual values);
 *   depth-first recursion in Fig. 3 child order; a node is split iff the min of its
 *   coefficients is < upper - tol, tol = rel_tol * max|b_root|; depth cap 20 (a leaf
 *   at the cap sets `capped`).  Without the cap, upper - lower <= tol on return.
 *   NONFINITE input gives NaN bounds. */
typedef struct oracle_bounds {
    double lower, upper, tol;
    int capped;
    int64_t nodes;          /* nodes split */
} oracle_bounds;
void   oracle_min_detj_bounds(const double X[8][3], double rel_tol, oracle_bounds* r);
void   oracle_min_detj_bounds_soa(const double* coords, int64_t n, double rel_tol, double* lower_out,
                                  double* upper_out, uint8_t* capped_out, int nthreads);
void   oracle_corner_quality_soa(const double* coords, int64_t n, double* sj_out, uint8_t* test1_out,
                                 uint8_t* near_out, int nthreads);
void   oracle_corner_quality_indexed(const double* vertices, const int32_t* hex_idx, int64_t n, double* sj_out,
                                     uint8_t* test1_out, uint8_t* near_out, int nthreads);

/* NEXT-4, linear quadrangle: Q[k][a], nodes 1..4 counter-clockwise
 * (L1 = (1-xi)(1-eta), L2 = xi(1-eta), L3 = xi eta, L4 = (1-xi) eta).  J[k] = det J at
 * corner k: J1 = v12 x v14, J2 = v12 x v23, J3 = v43 x v23, J4 = v43 x v14 (reading Q1).
 * Returns the flags byte: VALID iff all four corner values are > 0, signs decided
 * exactly; INVALID otherwise; NONFINITE for a non-finite or |x| > 2^300 coordinate.
 * near = 1 iff some |J_k| is within its fp64 rounding bound of 0. */
int    oracle_check_quad(const double Q[4][2], double J[4], int* near);
int    oracle_exact_orient2d(const double a[2], const double b[2], const double c[2]); /* sign((b-a) x (c-a)) */
void   oracle_check_quad_soa(const double* coords, int64_t n, uint8_t* flags_out, double* J_out,
                             uint8_t* near_out, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
