// hexval_device.cuh -- device arithmetic of the hot path (sm_100a, fp64 CUDA cores).
//
// Every operation is written with explicit round-to-nearest intrinsics and the
// library is compiled with -fmad=false, so each kernel that calls these
// functions produces bit-identical values (pass 1, the exact-sign kernel and
// the subdivision kernel all recompute the same root coefficients).
//
// Paper references are to /root/reference/PAPER.md (Johnen, Weill, Remacle 2017).
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace hexval {

constexpr int MAX_DEPTH = 20;
constexpr double U_ROUND = 1.1102230246251565404e-16;   // 2^-53

// ---------------------------------------------------------------------------
// small vector helpers
// ---------------------------------------------------------------------------
struct V3 {
    double x, y, z;
};

__device__ __forceinline__ V3 vsub(const V3& a, const V3& b) {
    return {__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)};
}
__device__ __forceinline__ V3 vadd(const V3& a, const V3& b) {
    return {__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y), __dadd_rn(a.z, b.z)};
}

// det(a, b, c) = a . (b x c)   (6 x signed tet volume)
__device__ __forceinline__ double det3(const V3& a, const V3& b, const V3& c) {
    const double wx = __fma_rn(b.y, c.z, -__dmul_rn(b.z, c.y));
    const double wy = __fma_rn(b.z, c.x, -__dmul_rn(b.x, c.z));
    const double wz = __fma_rn(b.x, c.y, -__dmul_rn(b.y, c.x));
    return __fma_rn(a.z, wz, __fma_rn(a.y, wy, __dmul_rn(a.x, wx)));
}

// high 32 bits of a double read as a signed int: for |x| >= 2^-1042 (and for
// +-0) the sign of the key equals the sign of x, and keys of positive
// doubles are ordered like the doubles.  Used for integer-pipe min / sign
// tests.
__device__ __forceinline__ int key(double x) { return __double2hiint(x); }
__device__ __forceinline__ int abskey(double x) { return __double2hiint(x) & 0x7fffffff; }

// max of abskey over N values: masked keys, a serial chain of maxima (the
// compiler forms 3-input VIMNMX3); measured equal to a balanced tree and 2-10%
// faster than signed/unsigned maxima of the raw keys, which need no masks but
// two reductions (profiles/r02/PASS1_EXPERIMENTS.md).
template <int N>
__device__ __forceinline__ int max3_tree(const int* k) {
    if constexpr (N == 1) return k[0];
    else if constexpr (N == 2) return max(k[0], k[1]);
    else {
        constexpr int M = (N + 2) / 3;
        int r[M];
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const int a = k[3 * j];
            const int b = 3 * j + 1 < N ? k[3 * j + 1] : a;
            const int c = 3 * j + 2 < N ? k[3 * j + 2] : a;
            r[j] = max(a, max(b, c));
        }
        return max3_tree<M>(r);
    }
}
template <int N>
__device__ __forceinline__ int max_abskey(const double* x) {
#ifndef HEXVAL_ABSKEY_TREE
    int m = 0;
#pragma unroll
    for (int j = 0; j < N; ++j) m = max(m, abskey(x[j]));
    return m;
#else
    int a[N];
#pragma unroll
    for (int j = 0; j < N; ++j) a[j] = abskey(x[j]);
    return max3_tree<N>(a);
#endif
}

// ---------------------------------------------------------------------------
// S1 + S2: the 20 Jacobian samples as tetrahedron determinants (section 5,
// PAPER.md:819-878, Fig. 4).  X[3k + a] = axis a of node k (Fig. 3 order).
//   c[0..7]  = det J at the 8 corners
//   d[0..11] = 4 det J at the 12 edge midpoints  (generalising J_9,
//              d_9 = det(v12, v14+v23, v15+v26))
// Edge k of d[] is Fig. 3 node 9+k.  Also returns the per-hex scale
// E = max |component| of the 12 edge vectors (as an upper bound key).
// ---------------------------------------------------------------------------
struct Samples {
    double c[8];
    double d[12];
    int ekey;        // abskey of max |edge component|
    int range_key = 0;     // in: max abskey of node 1's coordinates (0 if the caller tests the range itself)
    bool suspect = false;  // out: max(ekey, range_key) >= 2^297 -- the hex may be NONFINITE (hexval.cu, out_of_range)
};

struct NoCornerHook {
    __device__ __forceinline__ void operator()(const V3*, const double*, int) const {}
};

// corner(E, c, ekey): optional consumer of the 12 edge vectors E = {v12, v43,
// v56, v87, v14, v23, v58, v67, v15, v26, v48, v37}, the 8 corner samples c
// and the edge-scale key, called once they exist (the fused NEXT-2 screening
// outputs).
template <class CornerHook = NoCornerHook>
__device__ __forceinline__ void samples20(const double* X, Samples& s, CornerHook&& corner = CornerHook()) {
    const V3 n1{X[0], X[1], X[2]}, n2{X[3], X[4], X[5]}, n3{X[6], X[7], X[8]}, n4{X[9], X[10], X[11]};
    const V3 n5{X[12], X[13], X[14]}, n6{X[15], X[16], X[17]}, n7{X[18], X[19], X[20]}, n8{X[21], X[22], X[23]};
    // edge vectors v_ij = n_j - n_i
    const V3 v12 = vsub(n2, n1), v43 = vsub(n3, n4), v56 = vsub(n6, n5), v87 = vsub(n7, n8);
    const V3 v14 = vsub(n4, n1), v23 = vsub(n3, n2), v58 = vsub(n8, n5), v67 = vsub(n7, n6);
    const V3 v15 = vsub(n5, n1), v26 = vsub(n6, n2), v48 = vsub(n8, n4), v37 = vsub(n7, n3);
    const double comps[36] = {v12.x, v12.y, v12.z, v43.x, v43.y, v43.z, v56.x, v56.y, v56.z, v87.x, v87.y, v87.z,
                              v14.x, v14.y, v14.z, v23.x, v23.y, v23.z, v58.x, v58.y, v58.z, v67.x, v67.y, v67.z,
                              v15.x, v15.y, v15.z, v26.x, v26.y, v26.z, v48.x, v48.y, v48.z, v37.x, v37.y, v37.z};
    const int e = max_abskey<36>(comps);
    s.ekey = e;
    s.suspect = max(e, s.range_key) >= 0x52800000;        // 2^297 (decided here, before the determinants)

    // corners: det(d_xi x, d_eta x, d_zeta x) with the 3 edges at the corner
    s.c[0] = det3(v12, v14, v15);
    s.c[1] = det3(v12, v23, v26);
    s.c[2] = det3(v43, v23, v37);
    s.c[3] = det3(v43, v14, v48);
    s.c[4] = det3(v56, v58, v15);
    s.c[5] = det3(v56, v67, v26);
    s.c[6] = det3(v87, v67, v37);
    s.c[7] = det3(v87, v58, v48);
    {
        const V3 E[12] = {v12, v43, v56, v87, v14, v23, v58, v67, v15, v26, v48, v37};
        corner(E, s.c, e);
    }
    // twice the mid-edge derivatives (each shared by two edges)
    const V3 Se0 = vadd(v14, v23), Se1 = vadd(v58, v67);   // d_eta  at xi=1/2, zeta=0/1
    const V3 Sz0 = vadd(v15, v26), Sz1 = vadd(v48, v37);   // d_zeta at xi=1/2, eta=0/1
    const V3 Tx0 = vadd(v12, v43), Tx1 = vadd(v56, v87);   // d_xi   at eta=1/2, zeta=0/1
    const V3 Tz0 = vadd(v15, v48), Tz1 = vadd(v26, v37);   // d_zeta at eta=1/2, xi=0/1
    const V3 Ux0 = vadd(v12, v56), Ux1 = vadd(v43, v87);   // d_xi   at zeta=1/2, eta=0/1
    const V3 Ue0 = vadd(v14, v58), Ue1 = vadd(v23, v67);   // d_eta  at zeta=1/2, xi=0/1
    s.d[0] = det3(v12, Se0, Sz0);    //  9: edge 1-2
    s.d[1] = det3(Tx0, v23, Tz1);    // 10: edge 2-3
    s.d[2] = det3(v43, Se0, Sz1);    // 11: edge 3-4
    s.d[3] = det3(Tx0, v14, Tz0);    // 12: edge 4-1
    s.d[4] = det3(Ux0, Ue0, v15);    // 13: edge 1-5
    s.d[5] = det3(Ux0, Ue1, v26);    // 14: edge 2-6
    s.d[6] = det3(Ux1, Ue1, v37);    // 15: edge 3-7
    s.d[7] = det3(Ux1, Ue0, v48);    // 16: edge 4-8
    s.d[8] = det3(v56, Se1, Sz0);    // 17: edge 5-6
    s.d[9] = det3(Tx1, v67, Tz1);    // 18: edge 6-7
    s.d[10] = det3(v87, Se1, Sz1);   // 19: edge 7-8
    s.d[11] = det3(Tx1, v58, Tz0);   // 20: edge 8-5
}

// Step-2 rounding bound for the computed c[] and d[] (DESIGN.md "Error
// bounds"): |fl(x) - x| <= 264 u E^3 (+ underflow), tau2 = 512 u E^3 + ...
__device__ __forceinline__ double step2_tau(int ekey) {
    const double E = __hiloint2double(ekey, 0xffffffff);           // >= max |edge component|
    const double E2 = __dmul_rn(E, E);
    const double t = __dmul_rn(__dmul_rn(512.0 * U_ROUND, E2), E);
    return __fma_rn(8.7e-317 /* ~2^-1050 */, __dadd_rn(1.0, E2), t);
}

// ---------------------------------------------------------------------------
// S4: b = T~ c20 (Table 3), in scaled form
//   c  (corners)            = b_1..8
//   e2 = d_e - c_a - c_b    = 2 b_e      (edge rows: 2 I_12, -1/2 at the ends)
//   f4 = sum d_e - 3 sum c  = 4 b_f      (face rows: 1 on 4 edges, -3/4 on 4 corners)
//   z8 = sum d_e - 5 sum c  = 8 b_27     (last row: 1/2 on edges, -5/8 on corners)
// with d = 4 c_e.  The scalings are exact powers of two, so signs are those
// of the Bezier coefficients.
// ---------------------------------------------------------------------------
struct Coeffs {
    double e2[12];
    double f4[6];
    double z8;
};

__device__ __forceinline__ double sum4(double a, double b, double c, double d) {
    return __dadd_rn(__dadd_rn(a, b), __dadd_rn(c, d));
}

__device__ __forceinline__ void transform(const Samples& s, Coeffs& t) {
    const double* c = s.c;
    const double* d = s.d;
    // edges (Fig. 3 nodes 9..20): (1,2) (2,3) (3,4) (1,4) (1,5) (2,6) (3,7) (4,8) (5,6) (6,7) (7,8) (5,8)
    t.e2[0] = __dsub_rn(__dsub_rn(d[0], c[0]), c[1]);
    t.e2[1] = __dsub_rn(__dsub_rn(d[1], c[1]), c[2]);
    t.e2[2] = __dsub_rn(__dsub_rn(d[2], c[2]), c[3]);
    t.e2[3] = __dsub_rn(__dsub_rn(d[3], c[0]), c[3]);
    t.e2[4] = __dsub_rn(__dsub_rn(d[4], c[0]), c[4]);
    t.e2[5] = __dsub_rn(__dsub_rn(d[5], c[1]), c[5]);
    t.e2[6] = __dsub_rn(__dsub_rn(d[6], c[2]), c[6]);
    t.e2[7] = __dsub_rn(__dsub_rn(d[7], c[3]), c[7]);
    t.e2[8] = __dsub_rn(__dsub_rn(d[8], c[4]), c[5]);
    t.e2[9] = __dsub_rn(__dsub_rn(d[9], c[5]), c[6]);
    t.e2[10] = __dsub_rn(__dsub_rn(d[10], c[6]), c[7]);
    t.e2[11] = __dsub_rn(__dsub_rn(d[11], c[4]), c[7]);
    // faces 21..26: corners {1234} {1256} {2367} {3478} {1458} {5678}
    //               edges   {9,10,11,12} {9,13,14,17} {10,14,15,18} {11,15,16,19} {12,13,16,20} {17,18,19,20}
    // Corner sums through shared pairs (14 adds instead of 18); the 4 vertical
    // edge pairs of faces 22 and 24 are reused by the centre row.
    const double p01 = __dadd_rn(c[0], c[1]), p23 = __dadd_rn(c[2], c[3]);
    const double p45 = __dadd_rn(c[4], c[5]), p67 = __dadd_rn(c[6], c[7]);
    const double C21 = __dadd_rn(p01, p23), C26 = __dadd_rn(p45, p67);
    const double C22 = __dadd_rn(p01, p45), C24 = __dadd_rn(p23, p67);
    const double C23 = __dadd_rn(__dadd_rn(c[1], c[2]), __dadd_rn(c[5], c[6]));
    const double C25 = __dadd_rn(__dadd_rn(c[0], c[3]), __dadd_rn(c[4], c[7]));
    const double s45 = __dadd_rn(d[4], d[5]), s67 = __dadd_rn(d[6], d[7]);   // edges 13+14, 15+16
    const double D21 = sum4(d[0], d[1], d[2], d[3]);
    const double D26 = sum4(d[8], d[9], d[10], d[11]);
    const double D22 = __dadd_rn(__dadd_rn(d[0], d[8]), s45);
    const double D24 = __dadd_rn(__dadd_rn(d[2], d[10]), s67);
    const double D23 = __dadd_rn(__dadd_rn(d[1], d[9]), __dadd_rn(d[5], d[6]));
    const double D25 = __dadd_rn(__dadd_rn(d[3], d[11]), __dadd_rn(d[4], d[7]));
    t.f4[0] = __fma_rn(-3.0, C21, D21);
    t.f4[1] = __fma_rn(-3.0, C22, D22);
    t.f4[2] = __fma_rn(-3.0, C23, D23);
    t.f4[3] = __fma_rn(-3.0, C24, D24);
    t.f4[4] = __fma_rn(-3.0, C25, D25);
    t.f4[5] = __fma_rn(-3.0, C26, D26);
    // centre: all 12 edges = bottom ring + top ring + 4 verticals; all 8 corners
    const double Dall = __dadd_rn(__dadd_rn(D21, D26), __dadd_rn(s45, s67));
    const double Call = __dadd_rn(C21, C26);
    t.z8 = __fma_rn(-5.0, Call, Dall);
}

// Step 4: all of b_9..27 > 0  (integer-pipe sign test on keys)
__device__ __forceinline__ bool step4_positive(const Coeffs& t) {
    int m = key(t.z8);
#pragma unroll
    for (int e = 0; e < 12; ++e) m = min(m, key(t.e2[e]));
#pragma unroll
    for (int f = 0; f < 6; ++f) m = min(m, key(t.f4[f]));
    return m > 0;
}

// Bezier coefficients in true scale, node layout P[i + 3j + 9k] with
// (i, j, k) = 2 xi (b_1 = b_000, b_2 = b_200, b_9 = b_100).
// Fig. 3 index -> layout slot:
__device__ __constant__ static const unsigned char kSigmaToSlot[27] = {
    0, 2, 8, 6, 18, 20, 26, 24,           // corners 1..8
    1, 5, 7, 3, 9, 11, 17, 15,            // edges 9..16
    19, 23, 25, 21,                       // edges 17..20
    4, 10, 14, 16, 12, 22,                // faces 21..26
    13};                                  // centre 27

__device__ __forceinline__ void root_coeffs(const Samples& s, const Coeffs& t, double* P) {
    P[0] = s.c[0];  P[2] = s.c[1];  P[8] = s.c[2];  P[6] = s.c[3];
    P[18] = s.c[4]; P[20] = s.c[5]; P[26] = s.c[6]; P[24] = s.c[7];
    P[1] = __dmul_rn(0.5, t.e2[0]);  P[5] = __dmul_rn(0.5, t.e2[1]);
    P[7] = __dmul_rn(0.5, t.e2[2]);  P[3] = __dmul_rn(0.5, t.e2[3]);
    P[9] = __dmul_rn(0.5, t.e2[4]);  P[11] = __dmul_rn(0.5, t.e2[5]);
    P[17] = __dmul_rn(0.5, t.e2[6]); P[15] = __dmul_rn(0.5, t.e2[7]);
    P[19] = __dmul_rn(0.5, t.e2[8]); P[23] = __dmul_rn(0.5, t.e2[9]);
    P[25] = __dmul_rn(0.5, t.e2[10]); P[21] = __dmul_rn(0.5, t.e2[11]);
    P[4] = __dmul_rn(0.25, t.f4[0]);  P[10] = __dmul_rn(0.25, t.f4[1]);
    P[14] = __dmul_rn(0.25, t.f4[2]); P[16] = __dmul_rn(0.25, t.f4[3]);
    P[12] = __dmul_rn(0.25, t.f4[4]); P[22] = __dmul_rn(0.25, t.f4[5]);
    P[13] = __dmul_rn(0.125, t.z8);
}

// ---------------------------------------------------------------------------
// K5: exact sign of one root sample, Kulisch-style long accumulator.
// A sample is det(a, b, c) where every component of a, b, c is a signed sum of
// 2 or 4 input coordinates, so det = sum of +-x*y*z over input doubles.  Each
// x*y*z is an exact 159-bit integer times 2^(ex+ey+ez); all of them are added
// into a 70-word two's-complement fixed-point accumulator whose LSB is 2^-3222
// (3 x the smallest subnormal exponent) and whose range covers |x| <= 2^300.
// ---------------------------------------------------------------------------
constexpr int KW = 70;
constexpr int KBASE = -3222;

struct Mant {
    uint64_t m;
    int e;
    int neg;
};

__device__ __forceinline__ Mant split_double(double x) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
    const int E = (int)((bits >> 52) & 0x7ff);
    const uint64_t F = bits & ((1ull << 52) - 1);
    Mant r;
    r.neg = (int)(bits >> 63);
    if (E == 0) { r.m = F; r.e = -1074; }
    else { r.m = F | (1ull << 52); r.e = E - 1075; }
    return r;
}

__device__ void kulisch_add(uint64_t* acc, double x, double y, double z, int sign) {
    const Mant a = split_double(x), b = split_double(y), c = split_double(z);
    if (a.m == 0 || b.m == 0 || c.m == 0) return;
    const int neg = (sign < 0) ^ a.neg ^ b.neg ^ c.neg;
    // 53 x 53 -> 106 bits
    const uint64_t lo1 = a.m * b.m, hi1 = __umul64hi(a.m, b.m);
    // (hi1:lo1) x c.m -> 3 words
    const uint64_t w0 = lo1 * c.m;
    const uint64_t t = __umul64hi(lo1, c.m);
    const uint64_t ulo = hi1 * c.m, uhi = __umul64hi(hi1, c.m);
    const uint64_t w1 = t + ulo;
    const uint64_t w2 = uhi + (w1 < t ? 1ull : 0ull);
    const int sh = a.e + b.e + c.e - KBASE;
    const int wd = sh >> 6, bt = sh & 63;
    uint64_t v[4];
    v[0] = w0 << bt;
    v[1] = bt ? ((w1 << bt) | (w0 >> (64 - bt))) : w1;
    v[2] = bt ? ((w2 << bt) | (w1 >> (64 - bt))) : w2;
    v[3] = bt ? (w2 >> (64 - bt)) : 0ull;
    if (!neg) {
        uint64_t carry = 0;
        for (int q = 0; q < 4; ++q) {
            const uint64_t s1 = acc[wd + q] + v[q];
            const uint64_t c1 = s1 < v[q];
            const uint64_t s2 = s1 + carry;
            const uint64_t c2 = s2 < carry;
            acc[wd + q] = s2;
            carry = c1 | c2;
        }
        for (int q = wd + 4; carry && q < KW; ++q) { acc[q] += 1; carry = acc[q] == 0; }
    } else {
        uint64_t borrow = 0;
        for (int q = 0; q < 4; ++q) {
            const uint64_t o = acc[wd + q];
            const uint64_t d1 = o - v[q];
            const uint64_t b1 = o < v[q];
            const uint64_t d2 = d1 - borrow;
            const uint64_t b2 = d1 < borrow;
            acc[wd + q] = d2;
            borrow = b1 | b2;
        }
        for (int q = wd + 4; borrow && q < KW; ++q) { borrow = acc[q] == 0; acc[q] -= 1; }
    }
}

__device__ int kulisch_sign(const uint64_t* acc) {
    if ((long long)acc[KW - 1] < 0) return -1;
    for (int q = KW - 1; q >= 0; --q)
        if (acc[q]) return 1;
    return 0;
}

// Sample vectors as (node, sign) lists.  Vector slot: up to 4 terms; node < 0
// ends the list.  Table derived from samples20() above.
struct VecTerms {
    signed char node[4];
    signed char sgn[4];
};
// direct edge vector v_ij = n_j - n_i (0-based i, j)
#define HV_E(i, j) {{(j), (i), -1, -1}, {1, -1, 0, 0}}
// summed vector v_ij + v_kl
#define HV_S(i, j, k, l) {{(j), (i), (l), (k)}, {1, -1, 1, -1}}
__device__ __constant__ static const VecTerms kSampleVecs[20][3] = {
    {HV_E(0, 1), HV_E(0, 3), HV_E(0, 4)},                 // c1 = det(v12, v14, v15)
    {HV_E(0, 1), HV_E(1, 2), HV_E(1, 5)},                 // c2 = det(v12, v23, v26)
    {HV_E(3, 2), HV_E(1, 2), HV_E(2, 6)},                 // c3 = det(v43, v23, v37)
    {HV_E(3, 2), HV_E(0, 3), HV_E(3, 7)},                 // c4 = det(v43, v14, v48)
    {HV_E(4, 5), HV_E(4, 7), HV_E(0, 4)},                 // c5 = det(v56, v58, v15)
    {HV_E(4, 5), HV_E(5, 6), HV_E(1, 5)},                 // c6 = det(v56, v67, v26)
    {HV_E(7, 6), HV_E(5, 6), HV_E(2, 6)},                 // c7 = det(v87, v67, v37)
    {HV_E(7, 6), HV_E(4, 7), HV_E(3, 7)},                 // c8 = det(v87, v58, v48)
    {HV_E(0, 1), HV_S(0, 3, 1, 2), HV_S(0, 4, 1, 5)},     //  9: det(v12, Se0, Sz0)
    {HV_S(0, 1, 3, 2), HV_E(1, 2), HV_S(1, 5, 2, 6)},     // 10: det(Tx0, v23, Tz1)
    {HV_E(3, 2), HV_S(0, 3, 1, 2), HV_S(3, 7, 2, 6)},     // 11: det(v43, Se0, Sz1)
    {HV_S(0, 1, 3, 2), HV_E(0, 3), HV_S(0, 4, 3, 7)},     // 12: det(Tx0, v14, Tz0)
    {HV_S(0, 1, 4, 5), HV_S(0, 3, 4, 7), HV_E(0, 4)},     // 13: det(Ux0, Ue0, v15)
    {HV_S(0, 1, 4, 5), HV_S(1, 2, 5, 6), HV_E(1, 5)},     // 14: det(Ux0, Ue1, v26)
    {HV_S(3, 2, 7, 6), HV_S(1, 2, 5, 6), HV_E(2, 6)},     // 15: det(Ux1, Ue1, v37)
    {HV_S(3, 2, 7, 6), HV_S(0, 3, 4, 7), HV_E(3, 7)},     // 16: det(Ux1, Ue0, v48)
    {HV_E(4, 5), HV_S(4, 7, 5, 6), HV_S(0, 4, 1, 5)},     // 17: det(v56, Se1, Sz0)
    {HV_S(4, 5, 7, 6), HV_E(5, 6), HV_S(1, 5, 2, 6)},     // 18: det(Tx1, v67, Tz1)
    {HV_E(7, 6), HV_S(4, 7, 5, 6), HV_S(3, 7, 2, 6)},     // 19: det(v87, Se1, Sz1)
    {HV_S(4, 5, 7, 6), HV_E(4, 7), HV_S(0, 4, 3, 7)},     // 20: det(Tx1, v58, Tz0)
};
#undef HV_E
#undef HV_S

// true iff some vector of sample j is a direct edge vector that is exactly 0
// (coincident end nodes): then the sample is exactly 0 (its fp value is +-0).
__device__ __forceinline__ bool sample_has_zero_edge(const double* X, int j) {
#pragma unroll 1
    for (int v = 0; v < 3; ++v) {
        const VecTerms& T = kSampleVecs[j][v];
        if (T.node[2] >= 0) continue;                       // summed vector
        const int a = T.node[0], b = T.node[1];
        if (X[3 * a] == X[3 * b] && X[3 * a + 1] == X[3 * b + 1] && X[3 * a + 2] == X[3 * b + 2]) return true;
    }
    return false;
}

// exact sign of sample j (0..19) of the hex with coordinates X
__device__ __noinline__ int exact_sample_sign(const double* X, int j) {
    if (sample_has_zero_edge(X, j)) return 0;
    uint64_t acc[KW];
#pragma unroll 1
    for (int q = 0; q < KW; ++q) acc[q] = 0;
    const VecTerms& A = kSampleVecs[j][0];
    const VecTerms& B = kSampleVecs[j][1];
    const VecTerms& C = kSampleVecs[j][2];
    // det(a, b, c) = sum over permutations (i, k, l) of sgn * a_i b_k c_l
    const signed char perm[6][3] = {{0, 1, 2}, {1, 2, 0}, {2, 0, 1}, {0, 2, 1}, {1, 0, 2}, {2, 1, 0}};
#pragma unroll 1
    for (int p = 0; p < 6; ++p) {
        const int ps = p < 3 ? 1 : -1;
        const int i = perm[p][0], k = perm[p][1], l = perm[p][2];
#pragma unroll 1
        for (int ta = 0; ta < 4 && A.node[ta] >= 0; ++ta)
#pragma unroll 1
            for (int tb = 0; tb < 4 && B.node[tb] >= 0; ++tb)
#pragma unroll 1
                for (int tc = 0; tc < 4 && C.node[tc] >= 0; ++tc) {
                    const int sg = ps * A.sgn[ta] * B.sgn[tb] * C.sgn[tc];
                    kulisch_add(acc, X[3 * A.node[ta] + i], X[3 * B.node[tb] + k], X[3 * C.node[tc] + l], sg);
                }
    }
    return kulisch_sign(acc);
}

}  // namespace hexval
