// hexval.cu -- kernels and C ABI of the B200 hot path for the robust validity
// check of linear hexahedra (section 6).
//
//   K1/K2 pass 1         one hex per thread (Pass1Body): 20 tet determinants,
//                        Step 2, 27 Bezier coefficients, Step 4, flags,
//                        optional coefficients / fused NEXT-2 screening
//                        outputs, and (K3) warp-aggregated compaction of
//                        undecided / ambiguous hexes.  Pipelines:
//                        soa_cp_kernel (SoA planes, per-thread cp.async double
//                        buffering), idx_cp_kernel (int32 connectivity, rows
//                        and vertex gathers by cp.async, three deep),
//                        plain_kernel (unaligned inputs; HEXVAL_PASS1=ldg) and
//                        pass1_soa_wtma_kernel (per-warp TMA; A/B variant).
//   K5    exact path     exact signs of root samples within their rounding
//                        bound of 0 (Kulisch accumulator), then Steps 3-4;
//                        drained by K4 while it fills its batches.
//   K4    subdiv_kernel  persistent grid; each warp takes batches of 32 queued
//                        hexes and splits up to 32 same-depth nodes per step
//                        (one per lane), children pushed on a per-warp
//                        depth-sorted stack in global memory.
//   NEXT rows            bounds_kernel (NEXT-1, K4's machinery with a bounds
//                        policy), quality_kernel (NEXT-2), select_* (NEXT-3),
//                        quad_kernel (NEXT-4).
//
// All launches go on the caller's stream; queue lengths are read on the
// device, so there is no host synchronisation inside a call.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "hexval.h"
#include "hexval_device.cuh"
#include "scratch.cuh"

using namespace hexval;

// Debug builds (-DHEXVAL_DEBUG, e.g. `build.py --out libhexval_debug.so -D HEXVAL_DEBUG`)
// trap on any violated capacity / index invariant; compute-sanitizer is not
// available on the GPU pool, so the GPU tests are also run against that build.
#ifdef HEXVAL_DEBUG
#define HV_CHECK(cond) \
    do {               \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define HV_CHECK(cond) \
    do {               \
    } while (0)
#endif

namespace {

constexpr int P1_THREADS = 256;
// K4 / bounds kernel geometry (compile-time; A/B builds override with -D):
// threads per block and the minimum number of resident blocks per SM that
// bounds the register budget (128 x 2: <= 255 registers, 8 warps/SM).
#ifndef HEXVAL_K4_THREADS
#define HEXVAL_K4_THREADS 128
#endif
#ifndef HEXVAL_K4_MINB
#define HEXVAL_K4_MINB 2
#endif
constexpr int K4_THREADS = HEXVAL_K4_THREADS;
constexpr int K4_MINB = HEXVAL_K4_MINB;
// optional explicit register cap (e.g. 1-warp blocks with -DHEXVAL_K4_MAXNREG=224: 9 warps/SM)
#ifdef HEXVAL_K4_MAXNREG
#define HV_K4_BOUNDS __maxnreg__(HEXVAL_K4_MAXNREG)
#else
#define HV_K4_BOUNDS __launch_bounds__(K4_THREADS, K4_MINB)
#endif


// flags placeholders written by pass 1 for hexes that later kernels finish
constexpr uint8_t PENDING_EXACT = 0xFF;

struct Ctl {                 // per-call control block (device scratch)
    unsigned int n_sub;      // subdivision queue length
    unsigned int n_exact;    // exact-sign queue length
    unsigned int k4_next;    // dynamic fetch cursor of the subdivision kernel
    unsigned int ex_next;    // fetch cursor of the exact queue (drained by the subdivision kernel)
    unsigned int pad[4];
};

// ---------------------------------------------------------------------------
// loaders: SoA planes or indexed gather
// ---------------------------------------------------------------------------
struct SoaLoader {
#ifdef HEXVAL_SOA_INT_STEP2
    static constexpr bool kIntStep2 = true;      // A/B build: integer-pipe slow path for SoA too
#else
    static constexpr bool kIntStep2 = false;     // see step2_class
#endif
    const double* __restrict__ coords;
    int64_t n;
    // pass 1: streamed once, evict-first
    __device__ __forceinline__ void load_stream(int64_t i, double* X) const {
#pragma unroll
        for (int p = 0; p < 24; ++p) X[p] = __ldcs(coords + (int64_t)p * n + i);
    }
    __device__ __forceinline__ void load(int64_t i, double* X) const {
#pragma unroll
        for (int p = 0; p < 24; ++p) X[p] = __ldg(coords + (int64_t)p * n + i);
    }
    // SoA has no connectivity: coincident nodes are found by the exact kernel
    __device__ __forceinline__ bool dup_face_pair(int64_t) const { return false; }
};

struct IdxLoader {
    static constexpr bool kIntStep2 = true;      // see step2_class
    const double* __restrict__ verts;
    const int32_t* __restrict__ idx;
    uint32_t dupf = 0;                           // shared-memory address of this thread's precomputed duplicate-id
                                                 // flag (the cp.async pipeline), else 0: re-read the ids
    __device__ __forceinline__ void load(int64_t i, double* X) const {
        int v[8];
        if ((((uintptr_t)idx) & 15) == 0) {
            const int4 a = __ldcs(reinterpret_cast<const int4*>(idx) + 2 * i);
            const int4 b = __ldcs(reinterpret_cast<const int4*>(idx) + 2 * i + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __ldcs(idx + 8 * i + k);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double* p = verts + 3 * (int64_t)v[k];
            X[3 * k] = __ldg(p);
            X[3 * k + 1] = __ldg(p + 1);
            X[3 * k + 2] = __ldg(p + 2);
        }
    }
    __device__ __forceinline__ void load_stream(int64_t i, double* X) const { load(i, X); }
    // two nodes sharing a face have the same vertex id (see face_pair_coincident)
    __device__ __forceinline__ bool dup_face_pair(int64_t i) const;
};

// NONFINITE (reading G13): a coordinate is NaN/Inf or |x| > 2^300
__device__ __forceinline__ bool out_of_range(const double* X) {
    if (max_abskey<24>(X) < 0x52B00000) return false;   // every |x| < 2^300
    bool bad = false;
#pragma unroll
    for (int p = 0; p < 24; ++p) bad |= !(fabs(X[p]) <= 0x1p300);
    return bad;
}
// The same test for a hex whose edge-scale key is known (pass 1): every node is joined to
// node 1 by at most 3 hex edges, so edge components and node-1 coordinates all below 2^297
// put every |x| below 2^297 (1 + 3 (1 + 2u)) < 2^300 (the computed components are within a
// factor 1 + u of the true differences), and a NaN or Inf coordinate makes the components of
// its 3 edges NaN or Inf (key >= 0x7ff00000).  3 masked keys instead of 24 on the fast path
// (k1 = max abskey of node 1, taken before the samples so that X need not stay live); the
// slow path re-reads the hex and runs the exact test, out of line.
template <class L>
__device__ __noinline__ bool out_of_range_slow(const L ld, int64_t i) {
    double X[24];
    ld.load(i, X);
    bool bad = false;
#pragma unroll
    for (int p = 0; p < 24; ++p) bad |= !(fabs(X[p]) <= 0x1p300);
    return bad;
}
__device__ __forceinline__ int node1_key(const double* X) { return max(abskey(X[0]), max(abskey(X[1]), abskey(X[2]))); }
constexpr int RANGE_FAST_KEY = 0x52800000;               // 2^297

// Two nodes that share a face coincide (exact double equality of all three
// coordinates) => some Step-2 sample is exactly 0 => INVALID (reading G2):
//  * an edge pair makes a direct edge vector 0, and the corner samples at both
//    ends contain it;
//  * a face-diagonal pair (a, c) of face (a, b, c, d) makes the two in-face
//    edge vectors at b (and at d) equal up to sign, so det J at corner b is 0.
// Exact for every input; the exact kernel (K5) tests it before any long-accumulator work.
__device__ __constant__ static const unsigned char kFacePairs[24][2] = {
    {0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6}, {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7},   // edges
    {0, 2}, {1, 3}, {4, 6}, {5, 7}, {0, 5}, {1, 4}, {1, 6}, {2, 5}, {2, 7}, {3, 6}, {0, 7}, {3, 4}};  // face diagonals

__device__ __forceinline__ bool face_pair_coincident(const double* X) {
    bool hit = false;
#pragma unroll
    for (int q = 0; q < 24; ++q) {
        const int a = kFacePairs[q][0], b = kFacePairs[q][1];
        hit |= (X[3 * a] == X[3 * b]) & (X[3 * a + 1] == X[3 * b + 1]) & (X[3 * a + 2] == X[3 * b + 2]);
    }
    return hit;
}

__device__ __forceinline__ bool ids_dup_face_pair(const int* v) {
    bool hit = false;
#pragma unroll
    for (int q = 0; q < 24; ++q) hit |= v[kFacePairs[q][0]] == v[kFacePairs[q][1]];
    return hit;
}

__device__ __forceinline__ bool IdxLoader::dup_face_pair(int64_t i) const {
    if (dupf) {
        unsigned short f;
        asm volatile("ld.shared.u8 %0, [%1];" : "=h"(f) : "r"(dupf));
        return f != 0;
    }
    int v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(idx + 8 * i + k);
    bool hit = false;
#pragma unroll
    for (int q = 0; q < 24; ++q) hit |= v[kFacePairs[q][0]] == v[kFacePairs[q][1]];
    return hit;
}

// Test 1 in exact arithmetic for a hex whose corner samples are not all
// robustly signed (corner_quality gave T1_PENDING): two nodes sharing a face
// coincide => a corner sample is exactly 0 (face_pair_coincident) => fails;
// else every corner within tau2 of 0 takes its exact sign (K5 long
// accumulator).  Out of line; re-reads the hex's coordinates.
template <class L>
__device__ __noinline__ uint8_t exact_test1(const L ld, int64_t i) {
    if (ld.dup_face_pair(i)) return 0;
    double X[24];
    ld.load(i, X);
    if (face_pair_coincident(X)) return 0;
    Samples s;
    samples20(X, s);
    const int T = key(step2_tau(s.ekey));
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
        if (abskey(s.c[k]) <= T) {
            if (exact_sample_sign(X, k) <= 0) return 0;
        } else if (s.c[k] < 0.0) {
            return 0;
        }
    }
    return 1;
}

// Step 2 classification shared by pass 1 and the exact kernel.
enum : int { ST_INVALID = 0, ST_VALID = 1, ST_NONFINITE = 3, ST_SUB = 4, ST_EXACT = 5 };

// INT_SLOW selects the slow path (some sample <= tau2 in its hi word): FP64
// compares, or the integer pipe.  Measured on B200 with 3 interleaved A/B runs
// (profiles/r01): FP64 compares are faster on SoA config 1 (337 vs 349 us; the
// slow path is taken by ~80% of the warps there and the FP64 pipe has room),
// the integer pipe on indexed config 3 (1606 vs 1795 us; 36% invalid hexes,
// the FP64 pipe is the bottleneck).
template <bool INT_SLOW>
__device__ __forceinline__ int step2_class(const Samples& s, double tau2) {
    const int T = key(tau2);                          // tau2 > 0: key == abskey
    int km = key(s.c[0]);
#pragma unroll
    for (int k = 1; k < 8; ++k) km = min(km, key(s.c[k]));
#pragma unroll
    for (int e = 0; e < 12; ++e) km = min(km, key(s.d[e]));
    if (km > T) return ST_VALID;                       // every sample > tau2 > 0: robustly positive
    if (!INT_SLOW) {
#ifndef HEXVAL_STEP2_NO_NEGKEY
        // robustly negative sample first (one unsigned max over the keys: the sign bit
        // makes negatives exceed positives, then larger magnitude = larger key):
        // |x| > tau2 whenever its hi word exceeds tau2's, so the verdict is the one
        // the compares below would reach; most INVALID hexes stop here
        unsigned um = (unsigned)key(s.c[0]);
#pragma unroll
        for (int k = 1; k < 8; ++k) um = max(um, (unsigned)key(s.c[k]));
#pragma unroll
        for (int e = 0; e < 12; ++e) um = max(um, (unsigned)key(s.d[e]));
        if (um > (0x80000000u | (unsigned)T)) return ST_INVALID;
#endif
        bool neg = false, amb = false;
#pragma unroll
        for (int k = 0; k < 8; ++k) { neg |= s.c[k] < -tau2; amb |= fabs(s.c[k]) <= tau2; }
#pragma unroll
        for (int e = 0; e < 12; ++e) { neg |= s.d[e] < -tau2; amb |= fabs(s.d[e]) <= tau2; }
        if (neg) return ST_INVALID;
        return amb ? ST_EXACT : ST_VALID;
    }
    // Integer pipe, conservative in the hi words: a sample is robustly negative
    // if its sign is set and its hi word exceeds that of tau2 (then |x| > tau2);
    // it is ambiguous if |x|'s hi word <= that of tau2.  Here km <= T, so once no
    // sample is robustly negative some sample is ambiguous: either a key is negative
    // -- then um is the largest such key and um <= (sign | T) puts every negative
    // sample's |x| hi word at or below T -- or all keys are >= 0 and km is the
    // smallest |x| hi word.  No minimum over the masked keys is needed (session 4:
    // 20 LOP3 + 10 VIMNMX3 fewer per hex on the indexed path).
    unsigned um = (unsigned)key(s.c[0]);
#pragma unroll
    for (int k = 1; k < 8; ++k) um = max(um, (unsigned)key(s.c[k]));
#pragma unroll
    for (int e = 0; e < 12; ++e) um = max(um, (unsigned)key(s.d[e]));
    return um > (0x80000000u | (unsigned)T) ? ST_INVALID : ST_EXACT;
}

__device__ __forceinline__ void write_coeffs(double* __restrict__ coeffs, int64_t n, int64_t i,
                                             const Samples& s, const Coeffs& t) {
    double P[27];
    root_coeffs(s, t, P);
#pragma unroll
    for (int sg = 0; sg < 27; ++sg) __stcs(coeffs + (int64_t)sg * n + i, P[kSigmaToSlot[sg]]);
}

// K3, warp-aggregated: one atomic per warp that has something to append.
__device__ __forceinline__ void warp_append(bool pred, uint32_t val, uint32_t* __restrict__ q, unsigned int* counter) {
    const unsigned bal = __ballot_sync(0xffffffffu, pred);
    if (bal == 0) return;                                   // warp-uniform
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(bal) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(counter, (unsigned)__popc(bal));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (pred) q[base + __popc(bal & ((1u << lane) - 1u))] = val;
}

// Per-thread verdict counters of a persistent kernel, flushed once per warp.
struct P1Counts {
    unsigned v = 0, i = 0, n = 0;
    __device__ __forceinline__ void add(int st) { v += st == ST_VALID; i += st == ST_INVALID; n += st == ST_NONFINITE; }
    __device__ __forceinline__ void flush(hexval_stats* stats) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            v += __shfl_xor_sync(0xffffffffu, v, o);
            i += __shfl_xor_sync(0xffffffffu, i, o);
            n += __shfl_xor_sync(0xffffffffu, n, o);
        }
        if ((threadIdx.x & 31) == 0) {
            if (v) atomicAdd(&stats->n_valid, (unsigned long long)v);
            if (i) atomicAdd(&stats->n_invalid, (unsigned long long)i);
            if (n) atomicAdd(&stats->n_nonfinite, (unsigned long long)n);
        }
    }
};

template <bool STATS>
__device__ __forceinline__ void warp_epilogue(int st, int64_t i, Ctl* ctl, uint32_t* __restrict__ qsub,
                                              uint32_t* __restrict__ qexact, hexval_stats* stats) {
    warp_append(st == ST_SUB, (uint32_t)i, qsub, &ctl->n_sub);
    warp_append(st == ST_EXACT, (uint32_t)i, qexact, &ctl->n_exact);
    if (STATS) {
        const unsigned nv = __popc(__ballot_sync(0xffffffffu, st == ST_VALID));
        const unsigned ni = __popc(__ballot_sync(0xffffffffu, st == ST_INVALID));
        const unsigned nn = __popc(__ballot_sync(0xffffffffu, st == ST_NONFINITE));
        if ((threadIdx.x & 31) == 0) {
            if (nv) atomicAdd(&stats->n_valid, (unsigned long long)nv);
            if (ni) atomicAdd(&stats->n_invalid, (unsigned long long)ni);
            if (nn) atomicAdd(&stats->n_nonfinite, (unsigned long long)nn);
        }
    }
}

// ---------------------------------------------------------------------------
// K1 / K2: pass 1
// ---------------------------------------------------------------------------
__device__ __forceinline__ double len2(const V3& v) {
    return __fma_rn(v.z, v.z, __fma_rn(v.y, v.y, __dmul_rn(v.x, v.x)));
}

// NEXT-2 per hex from the 12 edge vectors E (samples20 order), the 8 corner
// samples c and the edge-scale key: Test 1 (all 8 corner det J > 0, PAPER.md:
// 107-109, 1260-1263) and the minimum corner scaled Jacobian
// c / (|d_xi x||d_eta x||d_zeta x|), the argmin taken by
// cross-multiplication so only the winner pays a division and a sqrt.  Shared
// by quality_kernel and the fused pass 1 (bit-identical outputs).
// t1 = 1: every corner sample robustly positive; 0: some corner robustly
// negative; T1_PENDING: some |c| <= tau2 (Step 2's rounding bound) and none
// robustly negative -- the caller decides it in exact arithmetic (exact_test1).
constexpr uint8_t T1_PENDING = 2;
// or'ed into t1 when the hex's edge scale is outside [2^-64, 2^64): the products below
// (squared-length products ~E^6, cross-multiplied ~E^12) could overflow or underflow,
// so the caller recomputes sj in a power-of-two rescaled frame (corner_sj_rescaled)
constexpr uint8_t SJ_RESCALE = 4;

__device__ __forceinline__ void corner_quality(const V3* E, const double* c, int ekey, double& sj, uint8_t& t1);

// min corner scaled Jacobian from the 12 edge vectors and the 8 corner samples
__device__ __forceinline__ double corner_sj(const V3* E, const double* c) {
    const double l12 = len2(E[0]), l43 = len2(E[1]), l56 = len2(E[2]), l87 = len2(E[3]);
    const double l14 = len2(E[4]), l23 = len2(E[5]), l58 = len2(E[6]), l67 = len2(E[7]);
    const double l15 = len2(E[8]), l26 = len2(E[9]), l48 = len2(E[10]), l37 = len2(E[11]);
    const double P[8] = {__dmul_rn(__dmul_rn(l12, l14), l15), __dmul_rn(__dmul_rn(l12, l23), l26),
                         __dmul_rn(__dmul_rn(l43, l23), l37), __dmul_rn(__dmul_rn(l43, l14), l48),
                         __dmul_rn(__dmul_rn(l56, l58), l15), __dmul_rn(__dmul_rn(l56, l67), l26),
                         __dmul_rn(__dmul_rn(l87, l67), l37), __dmul_rn(__dmul_rn(l87, l58), l48)};
#ifndef HEXVAL_SJ_SEQUENTIAL
    // argmin of c_k |c_k| / P_k as a three-round tournament (the lower index wins a tie, as in
    // a sequential scan; seven cross-multiplied compares either way, but a dependency chain of
    // three instead of seven: fused screening 401.3 -> 397.4 us, quality 293.0 -> 291.3 us on
    // config 1, profiles/r02/s4/s4d)
    double N[8], Q[8], C[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { N[k] = __dmul_rn(c[k], fabs(c[k])); Q[k] = P[k]; C[k] = c[k]; }
#pragma unroll
    for (int h = 1; h < 8; h *= 2)
#pragma unroll
        for (int k = 0; k < 8; k += 2 * h)
            if (__dmul_rn(N[k + h], Q[k]) < __dmul_rn(N[k], Q[k + h])) { N[k] = N[k + h]; Q[k] = Q[k + h]; C[k] = C[k + h]; }
    const double bp = Q[0], bc = C[0];
#else
    double bn = __dmul_rn(c[0], fabs(c[0])), bp = P[0], bc = c[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) {
        const double nk = __dmul_rn(c[k], fabs(c[k]));
        if (__dmul_rn(nk, bp) < __dmul_rn(bn, P[k])) { bn = nk; bp = P[k]; bc = c[k]; }   // nk/P[k] < bn/bp
    }
#endif
    // a zero-length corner edge (P == 0): P >= 0 always, and a positive high word proves
    // P > 0, so the FP64 compares run only when some P is 0 or below 2^-1042 (rare)
    int pk = key(P[0]);
#pragma unroll
    for (int k = 1; k < 8; ++k) pk = min(pk, key(P[k]));
    bool zero_edge = false;
    if (pk <= 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) zero_edge |= !(P[k] > 0.0);
    }
    // the winner's c / sqrt(P) as c * rsqrt(P) (a few ulps; the parity tolerance is 1e-13)
    return zero_edge ? __longlong_as_double(0x7ff8000000000000ll) : __dmul_rn(bc, rsqrt(bp));
}

__device__ __forceinline__ void corner_quality(const V3* E, const double* c, int ekey, double& sj, uint8_t& t1) {
    const bool in_range = ekey >= 0x3BF00000 && ekey < 0x43F00000;   // 2^-64 <= E < 2^64
    sj = corner_sj(E, c);                              // replaced by the rescaled value when !in_range
    int km = key(c[0]);
#pragma unroll
    for (int k = 1; k < 8; ++k) km = min(km, key(c[k]));
    const int T = key(step2_tau(ekey));                // tau2 > 0: key == abskey
    if (km > T) {
        t1 = 1;
    } else {
        unsigned um = (unsigned)key(c[0]);
#pragma unroll
        for (int k = 1; k < 8; ++k) um = max(um, (unsigned)key(c[k]));
        t1 = um > (0x80000000u | (unsigned)T) ? 0 : T1_PENDING;   // a robustly negative corner, else exact
    }
    if (!in_range) t1 |= SJ_RESCALE;
}

// corner_sj for a hex whose edge scale is extreme: re-read the coordinates, scale the edge
// vectors by 2^-e (E in [2^e, 2^(e+1)); exact) and recompute the 8 corner samples there --
// the scaled Jacobian is invariant under the scaling.  Out of line (rare).
template <class L>
__device__ __forceinline__ double corner_sj_rescaled(const L& ld, int64_t i) {
    double X[24];
    ld.load(i, X);
    V3 E[12];
    {
        const V3 n1{X[0], X[1], X[2]}, n2{X[3], X[4], X[5]}, n3{X[6], X[7], X[8]}, n4{X[9], X[10], X[11]};
        const V3 n5{X[12], X[13], X[14]}, n6{X[15], X[16], X[17]}, n7{X[18], X[19], X[20]}, n8{X[21], X[22], X[23]};
        E[0] = vsub(n2, n1); E[1] = vsub(n3, n4); E[2] = vsub(n6, n5); E[3] = vsub(n7, n8);
        E[4] = vsub(n4, n1); E[5] = vsub(n3, n2); E[6] = vsub(n8, n5); E[7] = vsub(n7, n6);
        E[8] = vsub(n5, n1); E[9] = vsub(n6, n2); E[10] = vsub(n8, n4); E[11] = vsub(n7, n3);
    }
    int ek = 0;
    for (int q = 0; q < 12; ++q) ek = max(ek, max(abskey(E[q].x), max(abskey(E[q].y), abskey(E[q].z))));
    const int e = max((ek >> 20) - 1023, -1022);
    const double f = __hiloint2double((1023 - e) << 20, 0);          // 2^-e
    for (int q = 0; q < 12; ++q) E[q] = {__dmul_rn(E[q].x, f), __dmul_rn(E[q].y, f), __dmul_rn(E[q].z, f)};
    const double c[8] = {det3(E[0], E[4], E[8]), det3(E[0], E[5], E[9]), det3(E[1], E[5], E[11]),
                         det3(E[1], E[4], E[10]), det3(E[2], E[6], E[8]), det3(E[2], E[7], E[9]),
                         det3(E[3], E[7], E[11]), det3(E[3], E[6], E[10])};
    return corner_sj(E, c);
}

// The rare paths of the NEXT-2 outputs in one out-of-line call (one call site per kernel
// keeps the streaming kernels' register allocation unchanged): sj in a rescaled frame
// (SJ_RESCALE) and Test 1 in exact arithmetic (T1_PENDING).
struct QualOut {
    double sj;
    unsigned t1;
};
template <class L>
__device__ __noinline__ QualOut quality_slow(const L ld, int64_t i, double sj, unsigned t1) {
    if (t1 & SJ_RESCALE) sj = corner_sj_rescaled(ld, i);
    t1 &= 3u;
    if (t1 == T1_PENDING) t1 = exact_test1(ld, i);
    return QualOut{sj, t1};
}

// S1-S5 + S8 for one hex whose 24 coordinates are in registers; returns the
// pass-1 state (ST_*).
// QUAL: also the fused NEXT-2 screening outputs (corner_quality) of the hex.
template <bool COEFFS, class L, bool QUAL = false, bool FAST_RANGE = true>
__device__ __forceinline__ int pass1_hex(const L& ld, const double* X, int64_t i, int64_t n,
                                         uint8_t* __restrict__ flags, double* __restrict__ coeffs,
                                         double* __restrict__ sj_out = nullptr, uint8_t* __restrict__ t1_out = nullptr) {
    int st;
    double sj = __longlong_as_double(0x7ff8000000000000ll);
    uint8_t t1 = 0;
    if constexpr (QUAL && FAST_RANGE) {
        // the fused screening kernels (166 registers, not at a register cliff) take the
        // NONFINITE test from the edge-scale key: 3 masked keys instead of 24 per hex
        // (399.2 -> 391.7 us on config 1).  In the validity kernels, which sit at 128
        // registers, the same reordering spilled loop state (328 -> 358 us): they keep
        // the test on the 24 coordinates up front.
        Samples s;
        s.range_key = node1_key(X);                           // samples20 folds the edge-scale key into it
        samples20(X, s, [&](const V3* E, const double* c, int ek) { corner_quality(E, c, ek, sj, t1); });   // S1 + S2
        // NONFINITE (reading G13) is decided last, when little is live across the out-of-line
        // exact test; until then a suspect hex (possibly NaN / out-of-range samples) only goes
        // through the register arithmetic below, never through the exact-sign machinery
        const bool suspect = s.suspect;
        st = step2_class<L::kIntStep2>(s, step2_tau(s.ekey));   // S3 (Step 2)
        if (st == ST_EXACT && ld.dup_face_pair(i)) st = ST_INVALID;   // a sample is exactly 0
        {
            Coeffs t;
            transform(s, t);                                  // S4 (Step 3)
            if (st == ST_VALID && !step4_positive(t)) st = ST_SUB;   // S5 (Step 4)
            if (COEFFS) write_coeffs(coeffs, n, i, s, t);
        }
        if (suspect && out_of_range_slow(ld, i)) {
            st = ST_NONFINITE;
            sj = __longlong_as_double(0x7ff8000000000000ll);
            t1 = 0;
        } else if (t1 & (SJ_RESCALE | T1_PENDING)) {
            const QualOut q = quality_slow(ld, i, sj, t1);
            sj = q.sj;
            t1 = (uint8_t)q.t1;
        }
    } else {
        // validity kernels (128 registers: the reordering above spills there, 328 -> 358 us):
        // the structure of the up-front test is kept, but its fast path looks at node 1 only
        // (3 masked keys instead of 24); a hex whose node 1 is in range while some edge
        // component is not below 2^297 -- possibly NONFINITE -- goes to the exact queue, where
        // exact_hex runs the exact range test first (config 1 332.2 -> 327.5 us, config 2
        // 270.2 -> 266.7 us, config 3 unchanged; profiles/r02/s4/s4r)
        bool nonfinite = false;
        if (!QUAL && FAST_RANGE) {
            if (node1_key(X) >= RANGE_FAST_KEY) {             // rare: the exact test on the 24 coordinates
#pragma unroll
                for (int p = 0; p < 24; ++p) nonfinite |= !(fabs(X[p]) <= 0x1p300);
            }
        } else {
            nonfinite = out_of_range(X);
        }
        if (nonfinite) {
            st = ST_NONFINITE;
        } else {
            Samples s;
            if (QUAL) samples20(X, s, [&](const V3* E, const double* c, int ek) { corner_quality(E, c, ek, sj, t1); });
            else samples20(X, s);                             // S1 + S2
            st = step2_class<L::kIntStep2>(s, step2_tau(s.ekey));   // S3 (Step 2)
            if (st == ST_EXACT && ld.dup_face_pair(i)) st = ST_INVALID;   // a sample is exactly 0
            Coeffs t;
            transform(s, t);                                  // S4 (Step 3)
            if (st == ST_VALID && !step4_positive(t)) st = ST_SUB;   // S5 (Step 4)
            // node 1 is in range but some edge component is huge: the exact queue decides
            // (exact_hex runs the exact range test first)
            if (!QUAL && FAST_RANGE && s.suspect) st = ST_EXACT;
            if (COEFFS) write_coeffs(coeffs, n, i, s, t);
            if (QUAL && (t1 & (SJ_RESCALE | T1_PENDING))) {
                const QualOut q = quality_slow(ld, i, sj, t1);
                sj = q.sj;
                t1 = (uint8_t)q.t1;
            }
        }
    }
    uint8_t f;
    switch (st) {
        case ST_INVALID: f = HEXVAL_INVALID; break;
        case ST_VALID: f = HEXVAL_VALID; break;
        case ST_NONFINITE: f = HEXVAL_NONFINITE; break;
        case ST_SUB: f = HEXVAL_FLAG_SUBDIVIDED; break;
        default: f = PENDING_EXACT; break;
    }
    __stcs(flags + i, f);
    if (QUAL) {
        __stcs(sj_out + i, sj);
        __stcs(t1_out + i, t1);
    }
    return st;
}

// One hex per thread, plain loads: the fallback pass 1 (unaligned inputs,
// HEXVAL_PASS1=ldg) and the NEXT-1 root phase.  Body: see Pass1Body.
template <class L, class Body>
__global__ void __launch_bounds__(P1_THREADS, 2) plain_kernel(L ld, int64_t n, Body body) {
    const int64_t i = (int64_t)blockIdx.x * P1_THREADS + threadIdx.x;
    int st = -1;
    if (i < n) {
        double X[24];
        ld.load_stream(i, X);
        st = body.template hex<L, false>(ld, X, i);
    }
    body.epilogue(st, i);
    body.finish();
}

// ---------------------------------------------------------------------------
// K1 (warp-TMA variant): persistent SoA pass 1.  Every warp owns two shared
// memory buffers; lane 0 stages the 24 coordinate planes of the warp's next
// 32-hex chunk with bulk async copies (cp.async.bulk + mbarrier complete_tx)
// while the warp computes the current chunk, so each warp always has one
// chunk (6 KB) in flight without spending registers on it, and no block-wide
// barrier is needed (compaction is warp-aggregated).
// ---------------------------------------------------------------------------
constexpr int WT_THREADS = 256;
constexpr int WT_WARPS = WT_THREADS / 32;
constexpr int WT_ROW = 34;                        // doubles per staged plane row: 32 + room for an 8-B shift
constexpr int WT_BUF = 24 * WT_ROW;               // doubles per buffer
constexpr size_t WT_SMEM = (size_t)WT_WARPS * 2 * WT_BUF * sizeof(double);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)                       // suspend-time hint (ns): sleep, do not spin
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

// Stage chunk c (hexes 32c .. 32c+31, all < n) into buf.  Plane p starts at
// element e = p*n + 32c; coords is 16-B aligned on this path, so e is odd
// exactly when n and p are odd: then the copy starts one element early (an
// element of plane p-1) and covers 34 doubles (272 B), and the reader shifts
// by one.  With n odd a full chunk ends before n, so e + 32 <= 24n - 1.
__device__ __forceinline__ void wt_issue(const double* __restrict__ coords, int64_t n, int64_t c, double* buf,
                                         uint64_t* bar) {
    const uint64_t policy = policy_evict_first();
    const bool odd = n & 1;
    mbar_expect_tx(bar, odd ? 12u * 256u + 12u * 272u : 24u * 256u);
#pragma unroll 4
    for (int p = 0; p < 24; ++p) {
        const int64_t e = (int64_t)p * n + c * 32;
        if (e & 1) bulk_g2s(buf + p * WT_ROW, coords + e - 1, 272u, bar, policy);
        else bulk_g2s(buf + p * WT_ROW, coords + e, 256u, bar, policy);
    }
}

template <bool COEFFS, bool STATS>
__global__ void __launch_bounds__(WT_THREADS, 2)
    pass1_soa_wtma_kernel(const double* __restrict__ coords, int64_t n, uint8_t* __restrict__ flags,
                          double* __restrict__ coeffs, Ctl* ctl, uint32_t* __restrict__ qsub,
                          uint32_t* __restrict__ qexact, hexval_stats* stats) {
    extern __shared__ __align__(128) double wt_buf[];        // [warp][2][24][WT_ROW]
    __shared__ __align__(8) uint64_t bars[WT_WARPS][2];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* const mybuf = wt_buf + (size_t)wib * 2 * WT_BUF;
    uint64_t* const mybar = bars[wib];
    const int64_t n_full = n / 32;                           // full 32-hex chunks
    const int64_t nw = (int64_t)gridDim.x * WT_WARPS;
    const int64_t gw = (int64_t)blockIdx.x * WT_WARPS + wib;
    const int shift = (int)(n & 1);
    if (lane == 0) {
        mbar_init(&mybar[0], 1);
        mbar_init(&mybar[1], 1);
        mbar_fence_init();
        if (gw < n_full) wt_issue(coords, n, gw, mybuf, &mybar[0]);
        if (gw + nw < n_full) wt_issue(coords, n, gw + nw, mybuf + WT_BUF, &mybar[1]);
    }
    __syncwarp();
    int k = 0;
    for (int64_t c = gw; c < n_full; c += nw, ++k) {
        const int b = k & 1;
        mbar_wait(&mybar[b], (unsigned)((k >> 1) & 1));
        const double* src = mybuf + b * WT_BUF + lane;
        double X[24];
#pragma unroll
        for (int p = 0; p < 24; ++p) X[p] = src[p * WT_ROW + (shift & p)];
        const int64_t i = c * 32 + lane;
        const int st = pass1_hex<COEFFS>(SoaLoader{coords, n}, X, i, n, flags, coeffs);
        __syncwarp();                                        // every lane has consumed buffer b
        if (lane == 0 && c + 2 * nw < n_full) wt_issue(coords, n, c + 2 * nw, mybuf + b * WT_BUF, &mybar[b]);
        warp_epilogue<STATS>(st, i, ctl, qsub, qexact, stats);
    }
    // ragged tail (n mod 32 hexes): one warp, plain loads
    if (n_full * 32 < n && gw == n_full % nw) {
        const int64_t i = n_full * 32 + lane;
        int st = -1;
        if (i < n) {
            double X[24];
#pragma unroll
            for (int p = 0; p < 24; ++p) X[p] = __ldcs(coords + (int64_t)p * n + i);
            st = pass1_hex<COEFFS>(SoaLoader{coords, n}, X, i, n, flags, coeffs);
        }
        warp_epilogue<STATS>(st, i, ctl, qsub, qexact, stats);
    }
}

// ---------------------------------------------------------------------------
// K1 (cp.async variant): persistent SoA pass 1.  Each thread prefetches the
// 24 coordinates of its hex in the block's next 256-hex tile into its own
// shared-memory slots with 8-byte async copies (LDGSTS) while it computes the
// current tile; cp.async.wait_group blocks in hardware (no spinning) and no
// block barrier is needed because every thread reads only what it copied.
// ---------------------------------------------------------------------------
#ifndef HEXVAL_CP_THREADS
#define HEXVAL_CP_THREADS 256
#endif
constexpr int CP_THREADS = HEXVAL_CP_THREADS;        // A/B builds: 128 x 4 or 256 x 2 CTAs/SM (16 warps/SM)
// The fused validity + screening pass (QUAL bodies) carries more live state per hex: it runs
// with its own block size (A/B knob; 384 x 1 = 12 warps/SM at <= 168 registers).
#ifndef HEXVAL_SCREEN_THREADS
#define HEXVAL_SCREEN_THREADS 384
#endif
#ifndef HEXVAL_CP_STAGES
#define HEXVAL_CP_STAGES 2
#endif
template <int T, int S = 2> constexpr size_t cp_smem() { return (size_t)S * 24 * T * sizeof(double); }
template <int T> constexpr int cp_minb() { return T >= 512 ? 1 : 512 / T; }

__device__ __forceinline__ void cp_async8(uint32_t dst, const double* src, uint64_t policy) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "l"(policy)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int T>
__device__ __forceinline__ void cp_issue_hex(const double* __restrict__ coords, int64_t n, int64_t i, uint32_t dst) {
    if (i < n) {
        const uint64_t policy = policy_evict_first();
#pragma unroll
        for (int p = 0; p < 24; ++p) cp_async8(dst + p * T * 8, coords + (int64_t)p * n + i, policy);
    }
    cp_async_commit();                                        // (possibly empty) group per tile
}

// Per-hex bodies run by the pipelines below.  hex() runs on the lanes that
// own a hex (X in registers) and returns a state; epilogue() is warp-collective
// (every lane, st = -1 without a hex); finish() once per thread at the end.
template <bool COEFFS, bool STATS, bool QUAL = false>
struct Pass1Body {                                           // K1/K2: S1-S8 + K3 (+ NEXT-2 outputs)
    static constexpr int THREADS = QUAL ? HEXVAL_SCREEN_THREADS : CP_THREADS;
    static constexpr int MINB = cp_minb<THREADS>();
    static constexpr int STAGES = QUAL ? 2 : HEXVAL_CP_STAGES;   // SoA pipeline depth (soa_cp_kernel)
    int64_t n;
    uint8_t* flags;
    double* coeffs;
    Ctl* ctl;
    uint32_t* qsub;
    uint32_t* qexact;
    hexval_stats* stats;
    double* sj;
    uint8_t* t1;
    P1Counts cnt;
    // FAST_RANGE: see pass1_hex; plain_kernel (128 registers) keeps the up-front range test
    template <class L, bool FAST_RANGE = true>
    __device__ __forceinline__ int hex(const L& ld, const double* X, int64_t i) {
        return pass1_hex<COEFFS, L, QUAL, FAST_RANGE>(ld, X, i, n, flags, coeffs, sj, t1);
    }
    __device__ __forceinline__ void epilogue(int st, int64_t i) {
        warp_epilogue<false>(st, i, ctl, qsub, qexact, stats);
        if (STATS) cnt.add(st);
    }
    __device__ __forceinline__ void finish() {
        if (STATS) cnt.flush(stats);
    }
};

template <class Body>
__global__ void __launch_bounds__(Body::THREADS, Body::MINB)
    soa_cp_kernel(const double* __restrict__ coords, int64_t n, Body body) {
    constexpr int CP_THREADS = Body::THREADS;
    extern __shared__ __align__(128) double cp_buf[];        // [2][24][CP_THREADS]
    const int tid = threadIdx.x;
    // 32-bit tile counters (n <= INT32_MAX): loop state that fits one register each, so the
    // register allocator does not spill it next to the hex's values
#ifdef HEXVAL_LOOP64
    using tile_t = int64_t;                                  // A/B build: round 1's 64-bit loop state
#else
    using tile_t = int;
#endif
    const tile_t tiles = (tile_t)((n + CP_THREADS - 1) / CP_THREADS);
    const tile_t G = (tile_t)gridDim.x;
    const uint32_t s0 = smem_u32(cp_buf + tid);
    constexpr int S = Body::STAGES;                          // tiles in flight + 1
    constexpr uint32_t SB = 24 * CP_THREADS * 8;             // bytes per stage
    tile_t t = blockIdx.x;
#pragma unroll
    for (int j = 0; j < S; ++j) cp_issue_hex<CP_THREADS>(coords, n, (int64_t)(t + j * G) * CP_THREADS + tid, s0 + j * SB);
    // buffer index: k & 1 for the default double buffer (the generic counter below costs
    // 1.3% on config 1: 333.4 vs 328.9 us, 4 interleaved reps, profiles/r02/PASS1_EXPERIMENTS.md)
    int b = 0;
    for (int k = 0; t < tiles; t += G, ++k) {
        if (S == 2) b = k & 1;
        cp_async_wait<S - 1>();                              // tile k has landed (tiles k+1.. may be in flight)
        const int64_t i = (int64_t)t * CP_THREADS + tid;
        int st = -1;
        if (i < n) {
            const double* src = cp_buf + b * 24 * CP_THREADS + tid;
            double X[24];
#pragma unroll
            for (int p = 0; p < 24; ++p) X[p] = src[p * CP_THREADS];
            st = body.hex(SoaLoader{coords, n}, X, i);
        }
        // refill this buffer with tile k+S (X was consumed above: program order)
        cp_issue_hex<CP_THREADS>(coords, n, (int64_t)(t + S * G) * CP_THREADS + tid, S == 2 ? (b ? s0 + SB : s0) : s0 + b * SB);
        body.epilogue(st, i);
        if (S != 2) b = b + 1 == S ? 0 : b + 1;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    body.finish();
}

// K1 (bulk variant, HEXVAL_PASS1=bulk): the CTA's 256-hex tile is staged by 24
// bulk copies of 2 KB (one per coordinate plane, issued by lanes 0-23 of warp 0)
// completing on a per-stage "full" mbarrier; each warp reads its hexes, arrives on
// the stage's "empty" mbarrier, and warp 0 refills a stage once all 8 warps have
// read it.  Per hex this replaces 24 8-byte cp.async copies and their 64-bit
// address arithmetic (~72 instructions per warp tile) by ~10; small (256-B, one per
// warp) bulk copies are bound by the copy engine's request rate (wtma variant).
// Full tiles only; the ragged tail (n mod 256 hexes) is done with plain loads.
// Measured on config 1 (profiles/r02/PASS1_EXPERIMENTS.md): 344 us vs 329 us for the
// per-thread cp.async pipeline -- the fewer instructions do not pay for coupling the
// CTA's 8 warps to one refill; kept as a tuning alternative.
constexpr int BK_THREADS = 256;
constexpr int BK_ROW = BK_THREADS + 2;            // doubles per staged plane: 256 + one element of shift, rounded to 16 B
constexpr int BK_STAGE = 24 * BK_ROW;             // doubles per stage
constexpr size_t BK_SMEM = (size_t)2 * BK_STAGE * sizeof(double);

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// warp 0: stage tile t (hexes 256t .. 256t+255, all < n) into buf; plane p starts at element
// e = p n + 256 t, copied from e - (e & 1) (16-B aligned: coords is 16-B aligned on this path)
__device__ __forceinline__ void bk_issue(const double* __restrict__ coords, int64_t n, int t, double* buf,
                                         uint64_t* full, int lane) {
    const bool odd = n & 1;
    if (lane == 0) mbar_expect_tx(full, odd ? 12u * 2064u + 12u * 2048u : 24u * 2048u);
    __syncwarp();
    if (lane < 24) {
        const int64_t e = (int64_t)lane * n + (int64_t)t * BK_THREADS;
        const uint64_t policy = policy_evict_first();
        if (e & 1) bulk_g2s(buf + lane * BK_ROW, coords + e - 1, 2064u, full, policy);
        else bulk_g2s(buf + lane * BK_ROW, coords + e, 2048u, full, policy);
    }
}

template <class Body>
__global__ void __launch_bounds__(BK_THREADS, 2)
    soa_bulk_kernel(const double* __restrict__ coords, int64_t n, Body body) {
    extern __shared__ __align__(128) double bk_buf[];        // [2][24][BK_ROW]
    __shared__ __align__(8) uint64_t full[2], empty[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tiles = (int)(n / BK_THREADS);                 // full tiles
    const int G = (int)gridDim.x;
    const int shift = (int)(n & 1);                          // odd planes start one element into their row
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_init(&empty[0], BK_THREADS / 32);
        mbar_init(&empty[1], BK_THREADS / 32);
        mbar_fence_init();
    }
    __syncthreads();
    int t = blockIdx.x;
    if (warp == 0) {
        if (t < tiles) bk_issue(coords, n, t, bk_buf, &full[0], lane);
        if (t + G < tiles) bk_issue(coords, n, t + G, bk_buf + BK_STAGE, &full[1], lane);
    }
    for (int k = 0; t < tiles; t += G, ++k) {
        const int b = k & 1;
        const unsigned ph = (unsigned)((k >> 1) & 1);
        mbar_wait(&full[b], ph);
        const double* src = bk_buf + b * BK_STAGE + tid;
        double X[24];
#pragma unroll
        for (int p = 0; p < 24; ++p) X[p] = src[p * BK_ROW + (shift & p)];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[b]);                // this warp has read stage b
        // refill before computing: the warps read a stage together once it lands (refilling
        // after the compute measured 344.5 vs 343.9 us and spilled 20 B)
        if (warp == 0 && t + 2 * G < tiles) {
            mbar_wait(&empty[b], ph);                        // every warp has read stage b
            bk_issue(coords, n, t + 2 * G, bk_buf + b * BK_STAGE, &full[b], lane);
        }
        const int64_t i = (int64_t)t * BK_THREADS + tid;
        const int st = body.template hex<SoaLoader, false>(SoaLoader{coords, n}, X, i);
        body.epilogue(st, i);
    }
    // ragged tail: the block that would own tile `tiles` does the last n mod 256 hexes with plain loads
    if ((int64_t)tiles * BK_THREADS < n && blockIdx.x == tiles % G) {
        const int64_t i = (int64_t)tiles * BK_THREADS + tid;
        int st = -1;
        if (i < n) {
            double X[24];
#pragma unroll
            for (int p = 0; p < 24; ++p) X[p] = __ldcs(coords + (int64_t)p * n + i);
            st = body.template hex<SoaLoader, false>(SoaLoader{coords, n}, X, i);
        }
        body.epilogue(st, i);
    }
    body.finish();
}

// K2 (cp.async variant): the same pipeline for int32 connectivity, three deep:
// while a thread computes its hex of tile k, the coordinates of its hex in
// tile k+1 are in flight (gathered with async copies from the vertex array,
// L1-allocating: neighbouring hexes share vertices) and so is the 32-byte
// connectivity row of tile k+2 (two 16-byte async copies into shared memory);
// after computing, the thread reads that row from shared memory and issues the
// gathers of tile k+2.  No register holds prefetched data across the compute.
template <int T> constexpr size_t cpi_smem() { return cp_smem<T>() + (size_t)2 * T * 32; }   // + two idx tiles

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_idx_row(const int32_t* __restrict__ idx, int64_t n, int64_t i, uint32_t dst) {
    if (i < n) {
        cp_async16(dst, idx + 8 * i);
        cp_async16(dst + 16, idx + 8 * i + 4);
    }
}

template <int CP_THREADS>
__device__ __forceinline__ void cp_gather_row(const double* __restrict__ verts, int64_t n, int64_t i,
                                              const int32_t* row, uint32_t dst, uint8_t* dupf) {
    if (i < n) {
        const int4 a = *reinterpret_cast<const int4*>(row);
        const int4 b = *reinterpret_cast<const int4*>(row + 4);
        const int v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        // the coincident-node rule on the ids while they are at hand: read back only by
        // hexes whose Step 2 is not decided in fp64 (IdxLoader::dup_face_pair)
#ifndef HEXVAL_NO_DUPFLAG
        *dupf = ids_dup_face_pair(v);
#endif
        uint64_t policy;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(policy));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double* src = verts + 3 * (int64_t)v[k];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) cp_async8(dst + (3 * k + ax) * CP_THREADS * 8, src + ax, policy);
        }
    }
}

template <class Body>
__global__ void __launch_bounds__(Body::THREADS, Body::MINB)
    idx_cp_kernel(const double* __restrict__ verts, const int32_t* __restrict__ idx, int64_t n, Body body) {
    constexpr int CP_THREADS = Body::THREADS;
    extern __shared__ __align__(128) double cp_buf[];        // [2][24][CP_THREADS] coords, then [2][CP_THREADS][8] ids
    const int tid = threadIdx.x;
    const int tiles = (int)((n + CP_THREADS - 1) / CP_THREADS);   // 32-bit loop state (see soa_cp_kernel)
    const int G = (int)gridDim.x;
    const uint32_t s0 = smem_u32(cp_buf + tid);
    const uint32_t s1 = s0 + 24 * CP_THREADS * 8;
    int32_t* const rows = reinterpret_cast<int32_t*>(cp_buf + 2 * 24 * CP_THREADS);
    int32_t* const row0 = rows + 8 * tid;                     // id row of tiles with even k
    int32_t* const row1 = rows + 8 * (CP_THREADS + tid);      // ... odd k
    // duplicate-id flags of tiles with even / odd k in a static array: their shared address
    // is a link-time constant plus tid, which the compiler rematerializes on the slow path
    // (a dynamic-smem base kept across the compute went to the stack frame and its reload
    // was the kernel's hottest stall, 6.6% of the samples on config 3)
    __shared__ uint8_t s_dup[2][CP_THREADS];
    uint8_t* const dup0 = &s_dup[0][tid];
    uint8_t* const dup1 = &s_dup[1][tid];
    const uint32_t r0 = smem_u32(row0), r1 = smem_u32(row1);
    int t = blockIdx.x;
    auto hex_of = [&](int tile) { return (int64_t)tile * CP_THREADS + tid; };
    // prologue: rows of tiles 0 and 1 synchronously, then groups G0 = {gathers 0, row 2}, G1 = {gathers 1, row 3}
    cp_idx_row(idx, n, hex_of(t), r0);
    cp_idx_row(idx, n, hex_of(t + G), r1);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    cp_gather_row<CP_THREADS>(verts, n, hex_of(t), row0, s0, dup0);
    cp_idx_row(idx, n, hex_of(t + 2 * G), r0);
    cp_async_commit();
    cp_gather_row<CP_THREADS>(verts, n, hex_of(t + G), row1, s1, dup1);
    cp_idx_row(idx, n, hex_of(t + 3 * G), r1);
    cp_async_commit();
    for (int k = 0; t < tiles; t += G, ++k) {
        const int bb = k & 1;
        cp_async_wait1();                                    // group k: coords of tile k, row of tile k+2
        const int64_t i = hex_of(t);
        int st = -1;
        if (i < n) {
            const double* src = cp_buf + bb * 24 * CP_THREADS + tid;
            double X[24];
#pragma unroll
            for (int p = 0; p < 24; ++p) X[p] = src[p * CP_THREADS];
#ifndef HEXVAL_NO_DUPFLAG
            // the flag's 32-bit shared address, read on the slow path only (a generic pointer
            // kept across the compute was spilled and its reload stalled: profiles/r02)
            st = body.hex(IdxLoader{verts, idx, smem_u32(bb ? dup1 : dup0)}, X, i);
#else
            st = body.hex(IdxLoader{verts, idx}, X, i);
#endif
        }
        // group k+2: gathers of tile k+2 (row read from shared memory), row of tile k+4
        cp_gather_row<CP_THREADS>(verts, n, hex_of(t + 2 * G), bb ? row1 : row0, bb ? s1 : s0, bb ? dup1 : dup0);
        cp_idx_row(idx, n, hex_of(t + 4 * G), bb ? r1 : r0);
        cp_async_commit();
        body.epilogue(st, i);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    body.finish();
}

// ---------------------------------------------------------------------------
// NEXT-2: screening by-products of the 8 corner samples:
// the minimum corner scaled Jacobian det J / (|d_xi x||d_eta x||d_zeta x|)
// and Ushakova's Test 1 -- det J > 0 at all 8 corners
// (PAPER.md:107-109, 1260-1263).  One hex per thread, streaming; the argmin
// over the corners compares c|c|/P by cross-multiplication (P = product of the
// squared edge lengths), so only the winner takes a division and a sqrt.
// ---------------------------------------------------------------------------

#ifndef HEXVAL_QUALITY_MINB
#define HEXVAL_QUALITY_MINB 3
#endif
constexpr int QUALITY_MINB = HEXVAL_QUALITY_MINB;   // 3: 80 registers (24 warps/SM): 304 us on config 1 vs 328 us at 2 (128 registers, no spills)

template <class L>
__global__ void __launch_bounds__(256, QUALITY_MINB) quality_kernel(L ld, int64_t n, double* __restrict__ sj_out,
                                                       uint8_t* __restrict__ t1_out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double X[24];
    ld.load_stream(i, X);
    double sj = __longlong_as_double(0x7ff8000000000000ll);   // NaN: undefined / NONFINITE
    uint8_t t1 = 0;
    if (!out_of_range(X)) {
        const V3 n1{X[0], X[1], X[2]}, n2{X[3], X[4], X[5]}, n3{X[6], X[7], X[8]}, n4{X[9], X[10], X[11]};
        const V3 n5{X[12], X[13], X[14]}, n6{X[15], X[16], X[17]}, n7{X[18], X[19], X[20]}, n8{X[21], X[22], X[23]};
        const V3 v12 = vsub(n2, n1), v43 = vsub(n3, n4), v56 = vsub(n6, n5), v87 = vsub(n7, n8);
        const V3 v14 = vsub(n4, n1), v23 = vsub(n3, n2), v58 = vsub(n8, n5), v67 = vsub(n7, n6);
        const V3 v15 = vsub(n5, n1), v26 = vsub(n6, n2), v48 = vsub(n8, n4), v37 = vsub(n7, n3);
        // corner k: (d_xi, d_eta, d_zeta) = the three edges leaving it
        const double c[8] = {det3(v12, v14, v15), det3(v12, v23, v26), det3(v43, v23, v37), det3(v43, v14, v48),
                             det3(v56, v58, v15), det3(v56, v67, v26), det3(v87, v67, v37), det3(v87, v58, v48)};
        const V3 E[12] = {v12, v43, v56, v87, v14, v23, v58, v67, v15, v26, v48, v37};
        int ek = 0;
#pragma unroll
        for (int q = 0; q < 12; ++q) ek = max(ek, max(abskey(E[q].x), max(abskey(E[q].y), abskey(E[q].z))));
        corner_quality(E, c, ek, sj, t1);
        if (t1 & (SJ_RESCALE | T1_PENDING)) {
            const QualOut q = quality_slow(ld, i, sj, t1);
            sj = q.sj;
            t1 = (uint8_t)q.t1;
        }
    }
    if (sj_out) __stcs(sj_out + i, sj);
    if (t1_out) __stcs(t1_out + i, t1);
}

// ---------------------------------------------------------------------------
// K5: exact signs for ambiguous root samples, then Steps 3-4
// ---------------------------------------------------------------------------
// Steps 2-4 of one hex with exact signs for the samples within tau2 of 0
// (PAPER.md:1114-1117); returns INVALID, VALID or FLAG_SUBDIVIDED (undecided
// after Step 4).  Kept out of line: the long accumulator lives in local memory.
__device__ __noinline__ uint8_t exact_resolve(const double* X) {
    Samples s;
    samples20(X, s);
    const int T = key(step2_tau(s.ekey));
    double v[20];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = s.c[j];
#pragma unroll
    for (int e = 0; e < 12; ++e) v[8 + e] = s.d[e];
#pragma unroll 1
    for (int j = 0; j < 20; ++j) {
        if ((unsigned)key(v[j]) > (0x80000000u | (unsigned)T)) return HEXVAL_INVALID;   // robustly negative
        if (abskey(v[j]) <= T && exact_sample_sign(X, j) <= 0) return HEXVAL_INVALID;   // exact sign
    }
    Coeffs t;
    transform(s, t);
    return step4_positive(t) ? HEXVAL_VALID : HEXVAL_FLAG_SUBDIVIDED;
}

// ---------------------------------------------------------------------------
// K4: recursive_subdivision, depth-first per thread
// ---------------------------------------------------------------------------
// Warp-cooperative design: each warp owns a batch of up to 32 queued hexes
// and a node stack in global memory.  Every step the 32 lanes split up to 32
// nodes of the same depth (the top level of the stack) into their 8 children
// (de Casteljau at t = 1/2 per axis, reading G3), classify each child
// and push the undecided ones with a warp prefix sum.
// Only nodes of one depth are popped per step (the top level of the stack) and
// their children are pushed on top, so the stack is sorted by depth.  Children
// at depth 20 are classified but never pushed (reading G5).  Per-hex state
// (INVALID / depth cap reached) lives in shared memory; nodes of a hex already
// found INVALID are dropped (the paper's early return).
//
// Stack capacity.  A step that pops k nodes pushes at most 8k, so the height h
// grows by at most 7k.  The pop size is capacity-adaptive (pop_size): with
// K4_TM = K4_CAP - K4_RESERVE, a normal step takes k = min(32, top-level count,
// (K4_TM - h) / 7) nodes and ends with h <= K4_TM; when not even one node fits
// under K4_TM the step pops exactly one node.  A run of such one-node steps is
// plain depth-first search from a state with h0 <= K4_TM (the state after a
// normal step, or a fresh batch of <= 32 roots): the nodes of that state only get
// consumed, and the run adds at most 7 unexpanded siblings per deeper level, so
// h <= h0 + 7 * (MAX_DEPTH - 1) < K4_TM + K4_RESERVE = K4_CAP throughout, and the
// run ends as soon as a node fits under K4_TM again.  Every step pops at least one
// node, so the traversal always progresses; the capacity only bounds how wide it
// runs.  Measured on config 4 (profiles/r02/s4): K4_CAP = 1024 (229 KB per warp, 271 MB per
// arena) runs at the speed and lane use (0.837) of the unconditional worst case reserved
// before (19 levels x 256 nodes = 4864 slots, 1.3 GB per arena); 512 slots throttle the
// pops (lane use 0.42, 422 ms vs 252 ms), 416 more so (0.26, 626 ms) -- still correct: the
// whole GPU suite passes with HEXVAL_K4_CAP=416 and the invariant traps on.
constexpr int K4_WARPS = K4_THREADS / 32;
#ifndef HEXVAL_K4_CAP
#define HEXVAL_K4_CAP 1024
#endif
constexpr int K4_CAP = HEXVAL_K4_CAP;
constexpr int K4_RESERVE = 7 * MAX_DEPTH;
constexpr int K4_TM = K4_CAP - K4_RESERVE;
static_assert(K4_TM >= 8 * 32, "a batch of 32 roots and their 256 children fit under the threshold");
static_assert(K4_CAP % 4 == 0, "128-byte lines hold 4 slots of one vector");
constexpr int K4_STRIDE = K4_CAP;   // slots between the 7 vector planes of a warp's stack (padding measured: no effect)

// nodes to pop from a stack of height h whose top level holds tcnt nodes
__device__ __forceinline__ int pop_size(int tcnt, int h) {
    return min(min(32, tcnt), max(1, (K4_TM - h) / 7));
}

struct WarpStacks {
    double* coef;           // [warp][7][K4_STRIDE][4]: 32-byte vectors of a node's 28 values (27 coefficients
                            // in layout i + 3j + 9k, then the node's meta word)
};

// 256-bit global accesses (sm_100: LDG/STG.E.ENL2.256): a node is 7 of them.
#if defined(HEXVAL_K4_LD_DEFAULT)
#define HV_LD_V4 "ld.global.v4.f64"
#elif defined(HEXVAL_K4_LD_L1LAST)
#define HV_LD_V4 "ld.global.L1::evict_last.v4.f64"
#else
#define HV_LD_V4 "ld.global.L1::evict_first.v4.f64"
#endif
__device__ __forceinline__ void ld_v4(const double* p, double& a, double& b, double& c, double& d) {
    asm volatile(HV_LD_V4 " {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p) : "memory");
}
// L1 policy of the stack traffic (measured on config 4, profiles/r02/K4_EXPERIMENTS.md): pushes
// keep their lines in L1 (a pop on the same SM follows soon), popped lines are dead -- evict
// them first: 267 ms vs 270 ms with default policies, 279 ms with no-allocate stores
#if defined(HEXVAL_K4_ST_L1NOALLOC)
#define HV_ST_V4 "st.global.L1::no_allocate.v4.f64"
#elif defined(HEXVAL_K4_ST_DEFAULT)
#define HV_ST_V4 "st.global.v4.f64"
#else
#define HV_ST_V4 "st.global.L1::evict_last.v4.f64"
#endif
__device__ __forceinline__ void st_v4(double* p, double a, double b, double c, double d) {
    asm volatile(HV_ST_V4 " [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// Popped stack lines are dead; HEXVAL_K4_DISCARD invalidates them in L2 instead of
// letting them be written back: lines wholly inside the popped slots [lo, lo + k)
// (4 slots per 128-byte line; the line of slot lo + k - 1 extends only into free
// slots above the top).  Measured on config 4 (K4_EXPERIMENTS.md): HBM writes
// 195 -> 27.7 GB per call, but the kernel 249 -> 265 ms (the CCTL per line costs more
// than the write-backs, which HBM absorbs at ~0.8 TB/s): off by default.
__device__ __forceinline__ void discard_popped(const double* sc, int lo, int k, int lane) {
#ifdef HEXVAL_K4_DISCARD
    const int f = (lo + 3) >> 2, nl = ((lo + k - 1) >> 2) - f + 1;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int idx = lane + 32 * r, q = idx >> 3, j = idx & 7;
        if (q < 7 && j < nl)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(sc + ((size_t)q * K4_STRIDE + 4 * (f + j)) * 4) : "memory");
    }
#endif
}

// A node on the stack: 7 x 32-byte vectors per slot, coalesced over the warp's
// consecutive slots; value 27 is the meta word (low half: owner = batch slot of
// the node's hex; high half: the node's scale pattern, see SplitScale).
__device__ __forceinline__ unsigned long long stack_load(const double* sc, int slot, double* P) {
    double m;
#pragma unroll
    for (int q = 0; q < 7; ++q) {
        const double* src = sc + ((size_t)q * K4_STRIDE + slot) * 4;
        if (q < 6) ld_v4(src, P[4 * q], P[4 * q + 1], P[4 * q + 2], P[4 * q + 3]);
        else ld_v4(src, P[24], P[25], P[26], m);
    }
    return (unsigned long long)__double_as_longlong(m);
}
__device__ __forceinline__ void stack_store_if(bool on, double* sc, int slot, const double* C, unsigned long long meta) {
    // one predicate for the node's 7 vector stores (offsets: K4_STRIDE * 32 bytes per vector)
    double* dst = sc + (size_t)slot * 4;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %29, 0;\n\t"
                 "@q " HV_ST_V4 " [%0], {%1,%2,%3,%4};\n\t"
                 "@q " HV_ST_V4 " [%0+%30], {%5,%6,%7,%8};\n\t"
                 "@q " HV_ST_V4 " [%0+%31], {%9,%10,%11,%12};\n\t"
                 "@q " HV_ST_V4 " [%0+%32], {%13,%14,%15,%16};\n\t"
                 "@q " HV_ST_V4 " [%0+%33], {%17,%18,%19,%20};\n\t"
                 "@q " HV_ST_V4 " [%0+%34], {%21,%22,%23,%24};\n\t"
                 "@q " HV_ST_V4 " [%0+%35], {%25,%26,%27,%28};\n\t}"
                 ::"l"(dst), "d"(C[0]), "d"(C[1]), "d"(C[2]), "d"(C[3]), "d"(C[4]), "d"(C[5]), "d"(C[6]), "d"(C[7]),
                 "d"(C[8]), "d"(C[9]), "d"(C[10]), "d"(C[11]), "d"(C[12]), "d"(C[13]), "d"(C[14]), "d"(C[15]),
                 "d"(C[16]), "d"(C[17]), "d"(C[18]), "d"(C[19]), "d"(C[20]), "d"(C[21]), "d"(C[22]), "d"(C[23]),
                 "d"(C[24]), "d"(C[25]), "d"(C[26]), "d"(__longlong_as_double((long long)meta)), "r"((unsigned)on),
                 "n"(1 * K4_STRIDE * 32), "n"(2 * K4_STRIDE * 32), "n"(3 * K4_STRIDE * 32), "n"(4 * K4_STRIDE * 32),
                 "n"(5 * K4_STRIDE * 32), "n"(6 * K4_STRIDE * 32)
                 : "memory");
}
__device__ __forceinline__ void stack_store(double* sc, int slot, const double* C, unsigned long long meta) {
#pragma unroll
    for (int q = 0; q < 7; ++q) {
        double* dst = sc + ((size_t)q * K4_STRIDE + slot) * 4;
        if (q < 6) st_v4(dst, C[4 * q], C[4 * q + 1], C[4 * q + 2], C[4 * q + 3]);
        else st_v4(dst, C[24], C[25], C[26], __longlong_as_double((long long)meta));
    }
}

// One line (p0, p1, p2) split at t = 1/2: m01 = (p0+p1)/2, m = (p0+2p1+p2)/4,
// m12 = (p1+p2)/2 (A.4 of SURVEY.md; 1 DMUL + 4 DFMA).  True values: used by
// the NEXT-1 bounds kernel, whose decisions compare coefficients with a bound.
__device__ __forceinline__ void line_split(double p0, double p1, double p2, double& m01, double& m, double& m12) {
    const double h1 = __dmul_rn(0.5, p1);
    m01 = __fma_rn(0.5, p0, h1);
    m12 = __fma_rn(0.5, p2, h1);
    m = __fma_rn(0.25, p0, __fma_rn(0.25, p2, h1));
}

// xi split of a node P (layout i + 3j + 9k) into G1[a + 5j + 15k], a = 0..4
// (both halves: the left child takes a = 0..2, the right one a = 2..4).
__device__ __forceinline__ void split_xi(const double* P, double* G1) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double p0 = P[3 * j + 9 * k], p1 = P[1 + 3 * j + 9 * k], p2 = P[2 + 3 * j + 9 * k];
            double m01, m, m12;
            line_split(p0, p1, p2, m01, m, m12);
            double* g = G1 + 5 * j + 15 * k;
            g[0] = p0; g[1] = m01; g[2] = m; g[3] = m12; g[4] = p2;
        }
}

// Quarter (hx, hy) of the children: eta half hy of xi half hx of G1, then
// both zeta halves: Z[a + 3u + 9v], xi index a (0..2), eta index u (0..2),
// zeta index v (0..4); child hz takes v = 2hz .. 2hz+2.
__device__ __forceinline__ void split_quarter(const double* G1, int hx, int hy, double* Z) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double B[9];                                     // B[u + 3k]: eta half hy of column a
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double* g = G1 + 2 * hx + a + 15 * k;
            double m01, m, m12;
            line_split(g[0], g[5], g[10], m01, m, m12);
            if (hy == 0) { B[3 * k] = g[0]; B[1 + 3 * k] = m01; B[2 + 3 * k] = m; }
            else { B[3 * k] = m; B[1 + 3 * k] = m12; B[2 + 3 * k] = g[10]; }
        }
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            double m01, m, m12;
            line_split(B[u], B[u + 3], B[u + 6], m01, m, m12);
            double* z = Z + a + 3 * u;
            z[0] = B[u]; z[9] = m01; z[18] = m; z[27] = m12; z[36] = B[u + 6];
        }
    }
}

// ---- K4's de Casteljau on power-of-two scaled values -----------------------
// The validity decisions only use signs, so K4 keeps each node's coefficients
// scaled by positive powers of two and splits a line with 3 FP64 instructions
// instead of 5.  Scales are separable: the value at (i, j, k) is the true value
// times s_x(i) s_y(j) s_z(k), and per axis only the ratios r01 = s(1)/s(0) and
// r21 = s(1)/s(2) (powers of two) are needed:
//   s01 = fma(r01, p0, p1) = s(1) (P0 + P1)      [= 2 s(1) * oracle's m01 exactly]
//   s12 = fma(r21, p2, p1) = s(1) (P1 + P2)
//   s   = s01 + s12        = 2 s(1) (m01 + m12)  [= 4 s(1) * oracle's m exactly]
// (P = true values).  Because r*p is exact and a power-of-two scaling commutes
// with rounding, every value is bit for bit the oracle's de Casteljau value
// (oracle.c oracle_subdivide: m01 = (p0+p1)/2, m = (m01+m12)/2) times its scale
// -- K4 makes the same decisions as the oracle's recursion on the same root.
// The five split positions carry scales (s0, 2s1, 4s1, 2s1, s2): the left child
// keeps (s0, 2s1, 4s1), i.e. r01' = 2 r01, r21' = 1/2; the right child
// (4s1, 2s1, s2): r01' = 1/2, r21' = 2 r21.  A ratio exponent e >= -1 grows by
// at most one per level, and a scale by at most 4x per axis and level (2^120
// over 20 levels; roots are normalised, see CoordRoot).  Pattern word: six
// 5-bit fields f = e + 1 (r01, r21 for x, y, z); the root's is all ones.
constexpr unsigned ROOT_PATTERN = 0x02108421u;

__device__ __forceinline__ double pow2_field(unsigned f) {      // 2^(f-1), f in [0, 31]
    return __hiloint2double((int)((1022u + f) << 20), 0);
}

struct SplitScale {
    double r01[3], r21[3];   // per axis x, y, z
    unsigned lo[3], hi[3];   // child pattern fields per axis: left child (f01+1, 0), right child (0, f21+1), packed
    __device__ __forceinline__ void unpack(unsigned pat) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const unsigned f01 = (pat >> (10 * a)) & 31u, f21 = (pat >> (10 * a + 5)) & 31u;
            r01[a] = pow2_field(f01);
            r21[a] = pow2_field(f21);
            lo[a] = (f01 + 1u) << (10 * a);
            hi[a] = (f21 + 1u) << (10 * a + 5);
        }
    }
    __device__ __forceinline__ unsigned child(int hx, int hy, int hz) const {
        return (hx ? hi[0] : lo[0]) | (hy ? hi[1] : lo[1]) | (hz ? hi[2] : lo[2]);
    }
};

__device__ __forceinline__ void line_split_s(double p0, double p1, double p2, double r01, double r21, double& s01,
                                             double& sm, double& s12) {
    s01 = __fma_rn(r01, p0, p1);
    s12 = __fma_rn(r21, p2, p1);
    sm = __dadd_rn(s01, s12);
}

__device__ __forceinline__ void split_xi_s(const double* P, const SplitScale& sc, double* G1) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double p0 = P[3 * j + 9 * k], p1 = P[1 + 3 * j + 9 * k], p2 = P[2 + 3 * j + 9 * k];
            double s01, sm, s12;
            line_split_s(p0, p1, p2, sc.r01[0], sc.r21[0], s01, sm, s12);
            double* g = G1 + 5 * j + 15 * k;
            g[0] = p0; g[1] = s01; g[2] = sm; g[3] = s12; g[4] = p2;
        }
}

__device__ __forceinline__ void split_quarter_s(const double* G1, int hx, int hy, const SplitScale& sc, double* Z) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double B[9];                                     // B[u + 3k]: eta half hy of column a
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double* g = G1 + 2 * hx + a + 15 * k;
            double s01, sm, s12;
            line_split_s(g[0], g[5], g[10], sc.r01[1], sc.r21[1], s01, sm, s12);
            if (hy == 0) { B[3 * k] = g[0]; B[1 + 3 * k] = s01; B[2 + 3 * k] = sm; }
            else { B[3 * k] = sm; B[1 + 3 * k] = s12; B[2 + 3 * k] = g[10]; }
        }
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            double s01, sm, s12;
            line_split_s(B[u], B[u + 3], B[u + 6], sc.r01[2], sc.r21[2], s01, sm, s12);
            double* z = Z + a + 3 * u;
            z[0] = B[u]; z[9] = s01; z[18] = sm; z[27] = s12; z[36] = B[u + 6];
        }
    }
}


struct K4Warp {
    unsigned status[32];    // per batch slot: bit 0 INVALID found, bit 1 depth cap reached
    uint32_t hex[32];       // hex id of each batch slot
};

// Per-level node counts of a warp's depth-sorted stack, kept in registers: the
// top level's count warp-uniform (tcnt), the count of each level L below it in
// lane L (lcnt; 0 for empty levels and for the top level and above).  A step's
// pop size is then known without a shared-memory round trip, and the next
// nonempty level is one ballot away (profiles/r02/K4_EXPERIMENTS.md: the
// shared-memory counters' load-use chains were 8% of the kernel's stall samples).
static_assert(MAX_DEPTH < 32, "one lane per stack level");
struct LevelCounts {
    int tcnt = 0, lcnt = 0;
    // after a step at level d (the top level) that pushed `pushed` nodes at level d+1
    __device__ __forceinline__ void after_step(int lane, int d, int pushed, int& D) {
        if (pushed) {
            if (lane == d) lcnt = tcnt;                   // level d keeps what was not popped
            tcnt = pushed;
            D = d + 1;
        } else if (tcnt == 0) {
            const unsigned ne = __ballot_sync(0xffffffffu, lcnt > 0);   // nonempty levels below d
            D = ne ? 31 - __clz(ne) : 0;
            tcnt = __shfl_sync(0xffffffffu, lcnt, D);
            if (lane == D) lcnt = 0;
        }
    }
};

// 32-bit shared-memory load that the compiler keeps where it is written: the
// status of a popped node's hex is read after the xi split, off the pop's
// load-use chain
__device__ __forceinline__ unsigned ld_shared_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}

// Root coefficients of queued item h: recomputed from the coordinates with
// the pass-1 arithmetic, or read from caller-supplied Bezier coefficients
// (hexval_classify_bezier).  Both are normalised by a power of two when their
// magnitude is extreme (coordinates beyond 2^+-200, coefficients beyond
// 2^+-896), so that the subdivision's scaled values neither overflow nor
// lose bits to subnormals; otherwise they are bit-identical to pass 1's.
template <class L>
__device__ __noinline__ uint8_t exact_hex(const L ld, uint32_t h) {
    double X[24];
    ld.load(h, X);
    // pass 1 also queues its range suspects here (pass1_hex): the exact NONFINITE test first
    bool bad = false;
#pragma unroll
    for (int p = 0; p < 24; ++p) bad |= !(fabs(X[p]) <= 0x1p300);
    if (bad) return HEXVAL_NONFINITE;
    return face_pair_coincident(X) ? (uint8_t)HEXVAL_INVALID : exact_resolve(X);
}

// 2^-e where 2^e <= max < 2^(e+1), for a max given as its (positive) hi word
__device__ __forceinline__ double inv_pow2_of_key(int k) {
    const int e = (k >> 20) - 1023;                       // unbiased exponent (k normal)
    return __hiloint2double((1023 - e) << 20, 0);
}

template <class L>
struct CoordRoot {
    L ld;
    __device__ __forceinline__ void operator()(uint32_t h, double* P) const {
        double X[24];
        ld.load(h, X);
        int mk = 0;
#pragma unroll
        for (int p = 0; p < 24; ++p) mk = max(mk, abskey(X[p]));
        if (mk < 0x33700000 || mk >= 0x4C700000) {                 // max|x| < 2^-200 or >= 2^200
            const double f = mk >= 0x00100000 ? inv_pow2_of_key(mk) : 0x1p1000;
#pragma unroll
            for (int p = 0; p < 24; ++p) X[p] = __dmul_rn(X[p], f);
        }
        Samples s;
        samples20(X, s);
        Coeffs t;
        transform(s, t);
        root_coeffs(s, t, P);
    }
    // K5 fused into K4: Steps 2-4 of an ambiguous hex with exact signs (out of line)
    __device__ __forceinline__ uint8_t exact(uint32_t h) const { return exact_hex(ld, h); }
};

struct CoeffRoot {
    const double* __restrict__ b;   // coefficient-major, b[sigma*n + h]
    int64_t n;
    __device__ __forceinline__ void operator()(uint32_t h, double* P) const {
        int mk = 0;
#pragma unroll
        for (int sg = 0; sg < 27; ++sg) {
            P[kSigmaToSlot[sg]] = __ldg(b + (int64_t)sg * n + h);
            mk = max(mk, abskey(P[kSigmaToSlot[sg]]));
        }
        if (mk < 0x07F00000 || mk >= 0x77F00000) {                 // max|b| < 2^-896 or >= 2^896
            const double f = mk >= 0x00100000 ? inv_pow2_of_key(mk) : 0x1p1000;
#pragma unroll
            for (int c = 0; c < 27; ++c) P[c] = __dmul_rn(P[c], f);
        }
    }
    __device__ __forceinline__ uint8_t exact(uint32_t) const { return HEXVAL_FLAG_SUBDIVIDED; }   // no exact queue
};

template <class R, bool STATS>
__global__ void HV_K4_BOUNDS subdiv_kernel(R root, uint8_t* __restrict__ flags, Ctl* ctl,
                                                            const uint32_t* __restrict__ qsub,
                                                            const uint32_t* __restrict__ qexact, WarpStacks ws,
                                                            hexval_stats* stats) {
    __shared__ K4Warp wst[K4_WARPS];
    const int lane = threadIdx.x & 31;
    K4Warp& W = wst[threadIdx.x >> 5];
    const size_t gw = (size_t)blockIdx.x * K4_WARPS + (threadIdx.x >> 5);
    double* const sc = ws.coef + gw * 28 * K4_STRIDE;
    const unsigned total = *((volatile unsigned*)&ctl->n_sub);
    const unsigned n_exact = *((volatile unsigned*)&ctl->n_exact);
    bool ex_left = n_exact > 0;                          // warp-uniform: the exact queue may hold items
    const unsigned lt_mask = (1u << lane) - 1u;
    LevelCounts lc;
    int top = 0, D = 0, nb = 0;                         // warp-uniform: stack size, top level, batch size
    unsigned long long nodes = 0, n_inv = 0, n_val = 0, n_und = 0, n_ex = 0, n_exi = 0, n_exv = 0, n_exn = 0, steps = 0;
    int maxd = 0;
    for (;;) {
        double P[27];
        bool act;
        int owner = lane, d, popped;
        unsigned pat = ROOT_PATTERN;                     // scale pattern of the node (see SplitScale)
        if (top == 0) {
            // batch done: write its verdicts (precedence INVALID > UNDETERMINED > VALID, reading G4)
            if (lane < nb) {
                const unsigned st = W.status[lane];
                const uint8_t v = (st & 1u) ? HEXVAL_INVALID : ((st & 2u) ? HEXVAL_UNDETERMINED : HEXVAL_VALID);
                flags[W.hex[lane]] = v | HEXVAL_FLAG_SUBDIVIDED;
                if (STATS) { n_inv += v == HEXVAL_INVALID; n_val += v == HEXVAL_VALID; n_und += v == HEXVAL_UNDETERMINED; }
            }
            // fill the next batch: first ambiguous hexes from the exact queue (K5 fused
            // here: each lane resolves one; the undecided ones join this warp's batch,
            // and at most as many are claimed as there are free slots), then hexes
            // pass 1 left undecided
            nb = 0;
            while (ex_left && nb < 32) {
                const unsigned want = 32u - (unsigned)nb;
                unsigned eb = 0;
                if (lane == 0) eb = atomicAdd(&ctl->ex_next, want);
                eb = __shfl_sync(0xffffffffu, eb, 0);
                const unsigned got = eb < n_exact ? min(want, n_exact - eb) : 0u;
                ex_left = got == want;
                if (got == 0) break;
                bool sub = false;
                uint32_t h = 0;
                if ((unsigned)lane < got) {
                    h = qexact[eb + lane];
                    const uint8_t f = root.exact(h);
                    if (f == HEXVAL_FLAG_SUBDIVIDED) sub = true;
                    else flags[h] = f;
                    if (STATS) { n_ex += f != HEXVAL_NONFINITE; n_exi += f == HEXVAL_INVALID; n_exv += f == HEXVAL_VALID; n_exn += f == HEXVAL_NONFINITE; }
                }
                const unsigned bal = __ballot_sync(0xffffffffu, sub);
                if (sub) W.hex[nb + __popc(bal & lt_mask)] = h;
                nb += __popc(bal);
                if (got < want) break;
            }
            if (nb < 32) {
                unsigned base = 0;
                const unsigned want = 32u - (unsigned)nb;
                if (lane == 0) base = atomicAdd(&ctl->k4_next, want);
                base = __shfl_sync(0xffffffffu, base, 0);
                const unsigned got = base < total ? min(want, total - base) : 0u;
                if ((unsigned)lane >= (unsigned)nb && (unsigned)lane < nb + got) W.hex[lane] = qsub[base + lane - nb];
                nb += (int)got;
            }
            __syncwarp();
            if (nb == 0) break;
            // the batch's roots (pass 1's arithmetic, normalised if extreme) go onto the
            // stack as level 0, so that every step takes its nodes from one place
            if (lane < nb) {
                W.status[lane] = 0;
                double rc[27];
                root(W.hex[lane], rc);
                stack_store(sc, lane, rc, (unsigned long long)(unsigned)lane | ((unsigned long long)ROOT_PATTERN << 32));
            }
            top = nb;
            lc.tcnt = nb;
            D = 0;
            __syncwarp();
        }
        {
            const int k = pop_size(lc.tcnt, top);
            HV_CHECK(D >= 0 && D < MAX_DEPTH && k > 0 && k <= top);
            act = lane < k;
            d = D;
            {
                // lanes >= k load the last popped node again (same lines, no extra traffic)
                // and drop it: an unconditional load keeps P out of a divergent merge
                const int slot = top - k + min(lane, k - 1);
                const unsigned long long meta = stack_load(sc, slot, P);
                owner = (int)(unsigned)meta;
                pat = (unsigned)(meta >> 32);
            }
            top -= k;
            lc.tcnt -= k;
            popped = k;
        }
        // ---- split every active node into its 8 children --------------------
        SplitScale ss;
        ss.unpack(pat);
        double G1[45];
        split_xi_s(P, ss, G1);
        discard_popped(sc, top, popped, lane);   // P is consumed: the popped lines are dead
        if (d > 0 && act) act = (ld_shared_u32(&W.status[owner]) & 1u) == 0;   // hex already INVALID: drop the node
        if (STATS) {
            const unsigned actmask = __ballot_sync(0xffffffffu, act);
            if (actmask) { nodes += __popc(actmask); maxd = max(maxd, d + 1); }
            ++steps;
        }
        bool inval = false, capped = false;
        int pushed = 0;                                  // warp-uniform
        const bool can_push = d + 1 < MAX_DEPTH;
        // classify and push the two children (zeta halves) of quarter (hx, hy)
        auto quarter = [&](const int hx, const int hy, const double* Z) {
                // classify the two children (zeta halves hz = 0, 1) from per-plane key
                // minima: planes v = 0, 2, 4 split into their 4 corners and 5 others,
                // planes 1 and 3 lie inside both children
                int pc[3], pr[3], pa[2];
#pragma unroll
                for (int w = 0; w < 3; ++w) {
                    const double* z = Z + 18 * w;
                    pc[w] = min(min(key(z[0]), key(z[2])), min(key(z[6]), key(z[8])));
                    pr[w] = min(min(min(key(z[1]), key(z[3])), key(z[4])), min(key(z[5]), key(z[7])));
                }
#pragma unroll
                for (int w = 0; w < 2; ++w) {
                    const double* z = Z + 9 + 18 * w;
                    pa[w] = min(min(min(key(z[0]), key(z[1])), min(key(z[2]), key(z[3]))),
                                min(min(key(z[4]), key(z[5])), min(min(key(z[6]), key(z[7])), key(z[8]))));
                }
                bool push[2];
#pragma unroll
                for (int hz = 0; hz < 2; ++hz) {
                    const int mc = min(pc[hz], pc[hz + 1]);
                    const int mi = min(min(pr[hz], pr[hz + 1]), pa[hz]);
                    const bool bad = act && mc <= 0;               // a corner value <= 0: INVALID
                    const bool und = act && mc > 0 && mi <= 0;     // undecided child
                    inval |= bad;
                    capped |= und && !can_push;
                    push[hz] = und && can_push;
                }
                const unsigned b0 = __ballot_sync(0xffffffffu, push[0] && !inval);
                const unsigned b1 = __ballot_sync(0xffffffffu, push[1] && !inval);
                if (b0 | b1) {
                    const int c0 = __popc(b0);
#pragma unroll
                    for (int hz = 0; hz < 2; ++hz) {
                        const unsigned bm = hz ? b1 : b0;
#ifndef HEXVAL_K4_BRANCHED_PUSH
                        if (bm) {                                  // warp-uniform; the lanes' stores are predicated
                            const bool mine = (bm >> lane) & 1u;
                            const int slot = top + pushed + (hz ? c0 : 0) + __popc(bm & lt_mask);
                            HV_CHECK(!mine || (slot >= 0 && slot < K4_CAP && owner >= 0 && owner < 32));
#else
                        if (bm & (1u << lane)) {
                            const bool mine = true;
                            const int slot = top + pushed + (hz ? c0 : 0) + __popc(bm & lt_mask);
                            HV_CHECK(slot >= 0 && slot < K4_CAP && owner >= 0 && owner < 32);
#endif
                            double C[27];
#pragma unroll
                            for (int v = 0; v < 3; ++v)
#pragma unroll
                                for (int u = 0; u < 3; ++u)
#pragma unroll
                                    for (int a = 0; a < 3; ++a) C[a + 3 * u + 9 * v] = Z[a + 3 * u + 9 * (2 * hz + v)];
                            stack_store_if(mine, sc, slot, C,
                                           (unsigned long long)(unsigned)owner |
                                               ((unsigned long long)ss.child(hx, hy, hz) << 32));
                        }
                    }
                    pushed += c0 + __popc(b1);
                }
        };
#pragma unroll
        for (int hx = 0; hx < 2; ++hx)
#pragma unroll
            for (int hy = 0; hy < 2; ++hy) {
                double Z[45];
                split_quarter_s(G1, hx, hy, ss, Z);
                quarter(hx, hy, Z);
            }
        if (inval) atomicOr(&W.status[owner], 1u);
        if (capped) atomicOr(&W.status[owner], 2u);
        top += pushed;
        lc.after_step(lane, d, pushed, D);
        __syncwarp();
    }
    if (STATS) {
        // warp-aggregated counters
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            n_inv += __shfl_xor_sync(0xffffffffu, n_inv, o);
            n_val += __shfl_xor_sync(0xffffffffu, n_val, o);
            n_und += __shfl_xor_sync(0xffffffffu, n_und, o);
            n_ex += __shfl_xor_sync(0xffffffffu, n_ex, o);
            n_exi += __shfl_xor_sync(0xffffffffu, n_exi, o);
            n_exv += __shfl_xor_sync(0xffffffffu, n_exv, o);
            n_exn += __shfl_xor_sync(0xffffffffu, n_exn, o);
        }
        if (lane == 0 && (n_ex | n_exn)) {
            if (n_ex) atomicAdd(&stats->n_exact, n_ex);
            if (n_exi) atomicAdd(&stats->n_invalid, n_exi);
            if (n_exv) atomicAdd(&stats->n_valid, n_exv);
            if (n_exn) atomicAdd(&stats->n_nonfinite, n_exn);
        }
        if (lane == 0) {
            const unsigned long long nsub = n_inv + n_val + n_und;
            if (nsub) {
                atomicAdd(&stats->n_subdivided, nsub);
                atomicAdd(&stats->n_nodes, nodes);
                atomicAdd(&stats->n_lane_steps, 32ull * steps);
                atomicMax(&stats->max_depth, (unsigned long long)maxd);
                if (n_inv) atomicAdd(&stats->n_invalid, n_inv);
                if (n_val) atomicAdd(&stats->n_valid, n_val);
                if (n_und) atomicAdd(&stats->n_undetermined, n_und);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// NEXT-1: certified bounds on min det J: lower =
// min of the Bezier coefficients over the leaves of a subdivision tree (convex
// hull property), upper = min of every corner coefficient met (actual values
// of det J).  A node is split iff min(b) < upper - tol, tol = rel_tol *
// max|b_root| (reading G15), so on return upper - lower <= tol unless the
// depth cap was reached.  Same warp-cooperative machinery as K4: every hex of
// [0, n) is a batch entry; the per-hex upper/lower live in shared memory as
// order-preserving 64-bit keys updated with atomicMin.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long okey(double x) {     // unsigned order == double order
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }

struct BWarp {
    unsigned long long upper[32], lower[32];
    double tol[32];
    unsigned capped[32];
    uint32_t hex[32];
};

// Root phase of NEXT-1: one hex per thread; a hex whose root coefficients
// already satisfy min(b) >= upper - tol is finished here, the others are
// appended (warp-aggregated) to the queue the warp-cooperative kernel drains.
__device__ __forceinline__ double root_bounds(const double* P, double rel_tol, double& up, double& mn) {
    mn = P[0];
    double sc_ = fabs(P[0]);
#pragma unroll
    for (int c = 1; c < 27; ++c) { mn = dmin(mn, P[c]); sc_ = fmax(sc_, fabs(P[c])); }
    up = dmin(dmin(dmin(P[0], P[2]), dmin(P[6], P[8])), dmin(dmin(P[18], P[20]), dmin(P[24], P[26])));
    return __dmul_rn(rel_tol, sc_);
}

struct BoundsRootBody {
    double rel_tol;
    double* lower;
    double* upper;
    uint8_t* status;
    unsigned* qcount;
    uint32_t* q;
    template <class L, bool = true>
    __device__ __forceinline__ int hex(const L&, const double* X, int64_t i) {
        double lo, up;
        uint8_t st = 0;
        bool queue = false;
        if (out_of_range(X)) {
            lo = up = __longlong_as_double(0x7ff8000000000000ll);
            st = 2;                                          // NONFINITE
        } else {
            Samples smp;
            samples20(X, smp);
            Coeffs t;
            transform(smp, t);
            double P[27];
            root_coeffs(smp, t, P);
            double mn;
            const double tol = root_bounds(P, rel_tol, up, mn);
            lo = mn;
            queue = !(mn >= up - tol);
        }
        if (!queue) {
            __stcs(lower + i, lo);
            __stcs(upper + i, up);
            if (status) __stcs(status + i, st);
        }
        return queue ? 1 : 0;
    }
    __device__ __forceinline__ void epilogue(int st, int64_t i) { warp_append(st == 1, (uint32_t)i, q, qcount); }
    __device__ __forceinline__ void finish() {}
};

template <class L>
__global__ void HV_K4_BOUNDS bounds_kernel(L ld, double rel_tol, double* __restrict__ lower_out,
                                                            double* __restrict__ upper_out, uint8_t* __restrict__ status_out,
                                                            unsigned* ctlq, const uint32_t* __restrict__ q, WarpStacks ws,
                                                            unsigned long long* nodes_out) {
    __shared__ BWarp wst[K4_WARPS];
    const int lane = threadIdx.x & 31;
    BWarp& W = wst[threadIdx.x >> 5];
    const size_t gw = (size_t)blockIdx.x * K4_WARPS + (threadIdx.x >> 5);
    double* const sc = ws.coef + gw * 28 * K4_STRIDE;
    const unsigned lt_mask = (1u << lane) - 1u;
    LevelCounts lc;
    int top = 0, D = 0, nb = 0;
    unsigned long long nodes = 0;
    const unsigned total = *((volatile unsigned*)&ctlq[0]);
    for (;;) {
        double P[27];
        bool act = false;
        int owner = lane, d;
        if (top == 0) {
            if (lane < nb) {                              // batch done
                const uint32_t h = W.hex[lane];
                const bool nf = W.capped[lane] & 2u;
                lower_out[h] = nf ? __longlong_as_double(0x7ff8000000000000ll) : okey_inv(W.lower[lane]);
                upper_out[h] = nf ? __longlong_as_double(0x7ff8000000000000ll) : okey_inv(W.upper[lane]);
                if (status_out) status_out[h] = (uint8_t)W.capped[lane];
            }
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(&ctlq[1], 32u);
            base = __shfl_sync(0xffffffffu, base, 0);
            nb = base < total ? (int)min(32u, total - base) : 0;
            if (nb == 0) break;
            d = 0;
            if (lane < nb) {
                const uint32_t h = q[base + lane];
                W.hex[lane] = h;
                W.capped[lane] = 0;
                double X[24];
                ld.load(h, X);
                Samples smp;
                samples20(X, smp);
                Coeffs t;
                transform(smp, t);
                root_coeffs(smp, t, P);                      // bit-identical to the root phase
                double up, mn;
                const double tol = root_bounds(P, rel_tol, up, mn);
                W.tol[lane] = tol;
                W.upper[lane] = okey(up);
                W.lower[lane] = okey(__longlong_as_double(0x7ff0000000000000ll));
                act = true;                                  // queued: the root is split
            }
        } else {
            const int k = pop_size(lc.tcnt, top);
            HV_CHECK(D > 0 && D < MAX_DEPTH && k > 0 && k <= top);
            d = D;
            if (lane < k) {
                const int slot = top - k + lane;
                owner = (int)(unsigned)stack_load(sc, slot, P);
                // upper may have dropped since the push: the node may now be a leaf
                double mn = P[0];
#pragma unroll
                for (int c = 1; c < 27; ++c) mn = dmin(mn, P[c]);
                const double U = okey_inv(W.upper[owner]);
                if (mn >= U - W.tol[owner]) atomicMin(&W.lower[owner], okey(mn));
                else act = true;
            }
            top -= k;
            lc.tcnt -= k;
        }
        __syncwarp();
        nodes += __popc(__ballot_sync(0xffffffffu, act));
        double G1[45];
        split_xi(P, G1);
        int pushed = 0;
        const bool can_push = d + 1 < MAX_DEPTH;
        const double tol = W.tol[owner];
#pragma unroll
        for (int hx = 0; hx < 2; ++hx)
#pragma unroll
            for (int hy = 0; hy < 2; ++hy) {
                double Z[45];
                split_quarter(G1, hx, hy, Z);
                // mins per zeta plane (the two children share plane 2): 5 plane
                // mins and 3 plane-corner mins instead of two 27- and 8-value scans
                double pm[5], pc[3];
#pragma unroll
                for (int v = 0; v < 5; ++v) {
                    const double* z = Z + 9 * v;
                    const double c4 = dmin(dmin(z[0], z[2]), dmin(z[6], z[8]));
                    if (!(v & 1)) pc[v >> 1] = c4;
                    pm[v] = dmin(dmin(dmin(c4, z[4]), dmin(z[1], z[3])), dmin(z[5], z[7]));
                }
                const double cmin[2] = {dmin(pc[0], pc[1]), dmin(pc[1], pc[2])};
                const double amin[2] = {dmin(dmin(pm[0], pm[1]), pm[2]), dmin(dmin(pm[2], pm[3]), pm[4])};
                if (act) atomicMin(&W.upper[owner], okey(dmin(cmin[0], cmin[1])));
                __syncwarp();
                const double U = okey_inv(W.upper[owner]);
                bool push[2];
#pragma unroll
                for (int hz = 0; hz < 2; ++hz) {
                    const bool leaf = act && (amin[hz] >= U - tol || !can_push);
                    if (leaf) {
                        atomicMin(&W.lower[owner], okey(amin[hz]));
                        if (!(amin[hz] >= U - tol)) atomicOr(&W.capped[owner], 1u);   // depth cap
                    }
                    push[hz] = act && !leaf;
                }
                const unsigned b0 = __ballot_sync(0xffffffffu, push[0]);
                const unsigned b1 = __ballot_sync(0xffffffffu, push[1]);
                if (b0 | b1) {
                    const int c0 = __popc(b0);
#pragma unroll
                    for (int hz = 0; hz < 2; ++hz) {
                        const unsigned bm = hz ? b1 : b0;
                        if (bm & (1u << lane)) {
                            const int slot = top + pushed + (hz ? c0 : 0) + __popc(bm & lt_mask);
                            HV_CHECK(slot >= 0 && slot < K4_CAP && owner >= 0 && owner < 32);
                            double C[27];
#pragma unroll
                            for (int v = 0; v < 3; ++v)
#pragma unroll
                                for (int u = 0; u < 3; ++u)
#pragma unroll
                                    for (int a = 0; a < 3; ++a) C[a + 3 * u + 9 * v] = Z[a + 3 * u + 9 * (2 * hz + v)];
                            stack_store(sc, slot, C, owner);

                        }
                    }
                    pushed += c0 + __popc(b1);
                }
            }
        top += pushed;
        lc.after_step(lane, d, pushed, D);
        __syncwarp();
    }
    if (nodes_out && lane == 0 && nodes) atomicAdd(nodes_out, nodes);
}

// ---------------------------------------------------------------------------
// NEXT-3: candidate-set filtering for indirect hex meshing (PAPER.md:80-85,
// 1247-1250): the ids of the VALID candidates in increasing order, and
// optionally the number of VALID candidates per group (e.g. per grid cell).
// Three kernels: per-tile counts (16 flags per thread, one 16-B load), a
// one-CTA exclusive scan of the tile counts, and the ordered write.
// ---------------------------------------------------------------------------
constexpr int SEL_THREADS = 256;
constexpr int SEL_TILE = SEL_THREADS * 16;

__device__ __forceinline__ unsigned valid_mask16(const uint8_t* __restrict__ flags, int64_t n, int64_t i0) {
    unsigned m = 0;
    if (i0 + 16 <= n && ((((uintptr_t)(flags + i0)) & 15) == 0)) {
        const uint4 w = __ldcs(reinterpret_cast<const uint4*>(flags + i0));
        const unsigned ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int b = 0; b < 4; ++b) m |= ((((ws[q] >> (8 * b)) & 3u) == HEXVAL_VALID) ? 1u : 0u) << (4 * q + b);
    } else {
#pragma unroll
        for (int b = 0; b < 16; ++b)
            if (i0 + b < n && (flags[i0 + b] & 3) == HEXVAL_VALID) m |= 1u << b;
    }
    return m;
}

__global__ void __launch_bounds__(SEL_THREADS) select_count_kernel(const uint8_t* __restrict__ flags, int64_t n,
                                                                     const int32_t* __restrict__ group,
                                                                     int32_t* __restrict__ group_counts,
                                                                     unsigned* __restrict__ tile_counts) {
    __shared__ unsigned s_w[SEL_THREADS / 32];
    const int64_t i0 = (int64_t)blockIdx.x * SEL_TILE + (int64_t)threadIdx.x * 16;
    const unsigned m = valid_mask16(flags, n, i0);
    if (group_counts && m) {
        if (i0 + 16 <= n && ((((uintptr_t)(group + i0)) & 15) == 0)) {
            // the 16 group ids in four 16-B loads, then one reduction per VALID candidate
            int g[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int4 v = __ldcs(reinterpret_cast<const int4*>(group + i0) + q);
                g[4 * q] = v.x; g[4 * q + 1] = v.y; g[4 * q + 2] = v.z; g[4 * q + 3] = v.w;
            }
#pragma unroll
            for (int b = 0; b < 16; ++b)
                if ((m >> b) & 1u) atomicAdd(&group_counts[g[b]], 1);
        } else {
#pragma unroll 1
            for (unsigned r = m; r; r &= r - 1) atomicAdd(&group_counts[__ldg(group + i0 + __ffs(r) - 1)], 1);
        }
    }
    unsigned c = __popc(m);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t = 0;
#pragma unroll
        for (int w = 0; w < SEL_THREADS / 32; ++w) t += s_w[w];
        tile_counts[blockIdx.x] = t;
    }
}

// exclusive scan of `tiles` counts in place (one CTA), total to *count
__global__ void __launch_bounds__(1024) select_scan_kernel(unsigned* __restrict__ tile_counts, int64_t tiles,
                                                             long long* __restrict__ count) {
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t base = 0; base < tiles; base += 1024) {
        const int64_t i = base + threadIdx.x;
        const unsigned long long v = i < tiles ? tile_counts[i] : 0;
        unsigned long long x = v;                                   // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[w] = x;
        __syncthreads();
        if (w == 0) {
            unsigned long long z = s_w[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, z, o);
                if (lane >= o) z += y;
            }
            s_w[lane] = z;                                           // inclusive over warps
        }
        __syncthreads();
        const unsigned long long excl = s_carry + (w ? s_w[w - 1] : 0) + x - v;
        if (i < tiles) tile_counts[i] = (unsigned)excl;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += s_w[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) *count = (long long)s_carry;
}

__global__ void __launch_bounds__(SEL_THREADS) select_write_kernel(const uint8_t* __restrict__ flags, int64_t n,
                                                                     const unsigned* __restrict__ tile_offsets,
                                                                     int32_t* __restrict__ ids) {
    __shared__ unsigned s_w[SEL_THREADS / 32];
    __shared__ int32_t s_ids[SEL_THREADS / 32][32 * 16];              // a warp's ids in order, then copied out
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * SEL_TILE + (int64_t)threadIdx.x * 16;
    const unsigned m = valid_mask16(flags, n, i0);
    const unsigned c = __popc(m);
    unsigned x = c;                                                  // inclusive warp scan of counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    unsigned before = 0;
#pragma unroll
    for (int q = 0; q < SEL_THREADS / 32; ++q) before += q < w ? s_w[q] : 0u;
    // each lane's ids go to their ordered places in the warp's staging row (shared
    // memory takes the scattered writes), then the warp writes the row out coalesced
    int32_t* const row = s_ids[w];
    unsigned p = x - c;
#pragma unroll 1
    for (unsigned r = m; r; r &= r - 1) row[p++] = (int32_t)(i0 + __ffs(r) - 1);
    __syncwarp();
    const unsigned total = __shfl_sync(0xffffffffu, x, 31);
    const unsigned base = tile_offsets[blockIdx.x] + before;
#pragma unroll 1
    for (unsigned q = lane; q < total; q += 32) {
        HV_CHECK((int64_t)(base + q) < n);
        ids[base + q] = row[q];
    }
}

// ---------------------------------------------------------------------------
// NEXT-4: linear quadrangle (section 2.1).  det J is
// bilinear, its minimum is at a corner: VALID iff J1..J4 > 0.  One quad per
// thread, 8 coordinate planes (plane 2k+a); a corner value within its rounding
// bound of 0 is decided exactly: (b-a) x (c-a) = a x b + b x c + c x a is a sum
// of 6 products of input doubles, accumulated in the K5 long accumulator.
// ---------------------------------------------------------------------------
__device__ __noinline__ int exact_orient2d(double ax, double ay, double bx, double by, double cx, double cy) {
    uint64_t acc[KW];
#pragma unroll 1
    for (int q = 0; q < KW; ++q) acc[q] = 0;
    kulisch_add(acc, ax, by, 1.0, 1);
    kulisch_add(acc, ay, bx, 1.0, -1);
    kulisch_add(acc, bx, cy, 1.0, 1);
    kulisch_add(acc, by, cx, 1.0, -1);
    kulisch_add(acc, cx, ay, 1.0, 1);
    kulisch_add(acc, cy, ax, 1.0, -1);
    return kulisch_sign(acc);
}

__device__ __forceinline__ uint8_t quad_one(const double* q, double* J) {
    bool bad = false;
#pragma unroll
    for (int p = 0; p < 8; ++p) bad |= !(fabs(q[p]) <= 0x1p300);
    if (bad) {
#pragma unroll
        for (int k = 0; k < 4; ++k) J[k] = __longlong_as_double(0x7ff8000000000000ll);
        return HEXVAL_NONFINITE;
    }
    const double v12x = __dsub_rn(q[2], q[0]), v12y = __dsub_rn(q[3], q[1]);
    const double v43x = __dsub_rn(q[4], q[6]), v43y = __dsub_rn(q[5], q[7]);
    const double v14x = __dsub_rn(q[6], q[0]), v14y = __dsub_rn(q[7], q[1]);
    const double v23x = __dsub_rn(q[4], q[2]), v23y = __dsub_rn(q[5], q[3]);
    // corner k: J_k = u x w (reading Q1: J3 at (1,1) pairs v43 with v23)
    const double ux[4] = {v12x, v12x, v43x, v43x}, uy[4] = {v12y, v12y, v43y, v43y};
    const double wx[4] = {v14x, v23x, v23x, v14x}, wy[4] = {v14y, v23y, v23y, v14y};
    // (origin, xi-neighbour, eta-neighbour) of each corner as an orientation of input points
    const int o[4][3] = {{0, 1, 3}, {0, 1, 2}, {2, 3, 1}, {3, 0, 2}};
    bool valid = true;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double a = __dmul_rn(ux[k], wy[k]), b = __dmul_rn(uy[k], wx[k]);
        J[k] = __dsub_rn(a, b);
        // |fl(J) - J| <= 8 u (|a| + |b|) for inputs with rounded differences (+ underflow)
        const double tau = __fma_rn(8.0 * U_ROUND, __dadd_rn(fabs(a), fabs(b)), 0x1p-1060);
        if (J[k] < -tau) valid = false;
        else if (!(J[k] > tau) && valid)
            valid = exact_orient2d(q[2 * o[k][0]], q[2 * o[k][0] + 1], q[2 * o[k][1]], q[2 * o[k][1] + 1],
                                   q[2 * o[k][2]], q[2 * o[k][2] + 1]) > 0;
    }
    return valid ? HEXVAL_VALID : HEXVAL_INVALID;
}

// QPT quads per thread, their 8*QPT loads issued before any compute (bytes in
// flight: the kernel is HBM bound at 65 B/quad with ~30 FP64 ops)
constexpr int QPT = 4;

__global__ void __launch_bounds__(256) quad_kernel(const double* __restrict__ coords, int64_t n,
                                                    uint8_t* __restrict__ flags, double* __restrict__ J_out) {
    const int64_t i0 = (int64_t)blockIdx.x * (256 * QPT) + threadIdx.x;
    double q[QPT][8];
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int64_t i = i0 + j * 256;
        if (i < n)
#pragma unroll
            for (int p = 0; p < 8; ++p) q[j][p] = __ldcs(coords + (int64_t)p * n + i);
    }
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int64_t i = i0 + j * 256;
        if (i >= n) break;
        double J[4];
        const uint8_t f = quad_one(q[j], J);
        __stcs(flags + i, f);
        if (J_out)
#pragma unroll
            for (int k = 0; k < 4; ++k) __stcs(J_out + (int64_t)k * n + i, J[k]);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct DeviceInfo {
    int sms = 0;
    int k4_blocks_per_sm = 0;
    int p1_variant = 0;           // SoA pass 1: P1_LDG (plain), P1_WTMA or P1_CP
    int p1_ctas_per_sm = 1;
    int screen_ctas_per_sm = 1;   // the fused screening pass (its own block size)
    bool ok = false;
};

DeviceInfo g_info[64];
std::mutex g_info_mu;

int wtma_setup() {
    const void* fns[4] = {(const void*)pass1_soa_wtma_kernel<false, false>,
                          (const void*)pass1_soa_wtma_kernel<false, true>,
                          (const void*)pass1_soa_wtma_kernel<true, false>,
                          (const void*)pass1_soa_wtma_kernel<true, true>};
    for (const void* f : fns)
        if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WT_SMEM) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pass1_soa_wtma_kernel<false, false>, WT_THREADS,
                                                      WT_SMEM) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return occ;
}

template <class Body>
bool cp_attr(size_t smem_soa = cp_smem<Body::THREADS, Body::STAGES>(), size_t smem_idx = cpi_smem<Body::THREADS>()) {
    return cudaFuncSetAttribute((const void*)soa_cp_kernel<Body>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem_soa) == cudaSuccess &&
           cudaFuncSetAttribute((const void*)idx_cp_kernel<Body>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem_idx) == cudaSuccess;
}

int cp_setup(int* screen_ctas) {
    const bool ok = cp_attr<Pass1Body<false, false>>() && cp_attr<Pass1Body<false, true>>() &&
                    cp_attr<Pass1Body<true, false>>() && cp_attr<Pass1Body<true, true>>() &&
                    cp_attr<Pass1Body<false, false, true>>() && cp_attr<Pass1Body<false, true, true>>();
    if (!ok) {
        cudaGetLastError();
        return 0;
    }
    int occ = 0, socc = 0;
    using SB = Pass1Body<false, false, true>;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, soa_cp_kernel<Pass1Body<false, false>>, CP_THREADS,
                                                      cp_smem<CP_THREADS, HEXVAL_CP_STAGES>()) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&socc, soa_cp_kernel<SB>, SB::THREADS,
                                                      cp_smem<SB::THREADS, SB::STAGES>()) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    *screen_ctas = socc > 0 ? socc : 1;
    return occ;
}

template <class Body>
bool bulk_attr() {
    return cudaFuncSetAttribute((const void*)soa_bulk_kernel<Body>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)BK_SMEM) == cudaSuccess;
}
int bulk_setup() {
    if (!(bulk_attr<Pass1Body<false, false>>() && bulk_attr<Pass1Body<false, true>>() &&
          bulk_attr<Pass1Body<true, false>>() && bulk_attr<Pass1Body<true, true>>())) {
        cudaGetLastError();
        return 0;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, soa_bulk_kernel<Pass1Body<false, false>>, BK_THREADS,
                                                      BK_SMEM) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return occ;
}

// Pass-1 variant for SoA inputs: HEXVAL_PASS1 = ldg | wtma | cp | bulk (tuning knob
// for measurements).
enum { P1_LDG = 0, P1_WTMA = 1, P1_CP = 2, P1_BULK = 3 };
int pass1_variant_from_env() {
    const char* v = getenv("HEXVAL_PASS1");
    if (v && !strcmp(v, "wtma")) return P1_WTMA;
    if (v && !strcmp(v, "bulk")) return P1_BULK;
    if (v && !strcmp(v, "cp")) return P1_CP;
    if (v && !strcmp(v, "ldg")) return P1_LDG;
    return P1_CP;                 // measured best on B200 (profiles/r01)
}

template <class L>
const DeviceInfo& device_info(int dev) {
    std::lock_guard<std::mutex> lk(g_info_mu);
    DeviceInfo& d = g_info[dev & 63];
    if (!d.ok) {
        cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, subdiv_kernel<CoordRoot<SoaLoader>, false>, K4_THREADS,
                                                      0);
        d.k4_blocks_per_sm = occ > 0 ? occ : 1;
        const int want = pass1_variant_from_env();
        int ctas = want == P1_WTMA ? wtma_setup() : (want == P1_CP || want == P1_BULK ? cp_setup(&d.screen_ctas_per_sm) : 0);
        if (want == P1_BULK && ctas > 0) ctas = bulk_setup();
        d.p1_variant = ctas > 0 ? want : P1_LDG;
        d.p1_ctas_per_sm = ctas > 0 ? ctas : 1;
        d.ok = true;
    }
    return d;
}

}  // namespace

struct hexval_profile {
    static constexpr int CAP = 256;
    cudaEvent_t ev[CAP][HEXVAL_NUM_PHASES][2];
    int count = 0;
    double pending_ms[HEXVAL_NUM_PHASES] = {0, 0, 0};
    long long pending_launches[HEXVAL_NUM_PHASES] = {0, 0, 0};
};

namespace {

// The pass-1 body of a call: (coefficients, stats, fused screening outputs).
struct P1Args {
    int64_t n;
    uint8_t* flags;
    double* coeffs;
    Ctl* ctl;
    uint32_t* qsub;
    uint32_t* qex;
    hexval_stats* stats;
    double* sj;                   // fused NEXT-2 outputs (both set or both null)
    uint8_t* t1;
};

template <class F>
void with_pass1_body(const P1Args& a, F&& f) {
    if (a.sj) {
        if (a.stats) f(Pass1Body<false, true, true>{a.n, a.flags, a.coeffs, a.ctl, a.qsub, a.qex, a.stats, a.sj, a.t1, {}});
        else f(Pass1Body<false, false, true>{a.n, a.flags, a.coeffs, a.ctl, a.qsub, a.qex, a.stats, a.sj, a.t1, {}});
    } else if (a.coeffs) {
        if (a.stats) f(Pass1Body<true, true>{a.n, a.flags, a.coeffs, a.ctl, a.qsub, a.qex, a.stats, nullptr, nullptr, {}});
        else f(Pass1Body<true, false>{a.n, a.flags, a.coeffs, a.ctl, a.qsub, a.qex, a.stats, nullptr, nullptr, {}});
    } else {
        if (a.stats) f(Pass1Body<false, true>{a.n, a.flags, a.coeffs, a.ctl, a.qsub, a.qex, a.stats, nullptr, nullptr, {}});
        else f(Pass1Body<false, false>{a.n, a.flags, a.coeffs, a.ctl, a.qsub, a.qex, a.stats, nullptr, nullptr, {}});
    }
}

template <class L>
void launch_pass1_plain(const L& ld, const P1Args& a, cudaStream_t stream) {
    const unsigned blocks = (unsigned)((a.n + P1_THREADS - 1) / P1_THREADS);
    with_pass1_body(a, [&](auto body) { plain_kernel<<<blocks, P1_THREADS, 0, stream>>>(ld, a.n, body); });
}

template <class L>
void launch_pass1(const L& ld, const DeviceInfo& info, const P1Args& a, cudaStream_t stream);

// indexed: the cp.async gather pipeline when the connectivity rows are 16-B
// aligned (int4 loads), else the plain kernel
template <>
void launch_pass1<IdxLoader>(const IdxLoader& ld, const DeviceInfo& info, const P1Args& a, cudaStream_t stream) {
    if (info.p1_variant != P1_CP || (((uintptr_t)ld.idx) & 15) != 0) {
        launch_pass1_plain(ld, a, stream);
        return;
    }
    with_pass1_body(a, [&](auto body) {
        constexpr int T = decltype(body)::THREADS;
        const int64_t tiles = (a.n + T - 1) / T;
        const int64_t cap = (int64_t)info.sms * (T == CP_THREADS ? info.p1_ctas_per_sm : info.screen_ctas_per_sm);
        const unsigned grid = (unsigned)(tiles < cap ? tiles : cap);
        idx_cp_kernel<<<grid, T, cpi_smem<T>(), stream>>>(ld.verts, ld.idx, a.n, body);
    });
}

void launch_bulk(const SoaLoader& ld, const DeviceInfo& info, const P1Args& a, cudaStream_t stream) {
    const int64_t tiles = (a.n + BK_THREADS - 1) / BK_THREADS;
    const int64_t cap = (int64_t)info.sms * info.p1_ctas_per_sm;
    const unsigned grid = (unsigned)(tiles < cap ? tiles : cap);
    with_pass1_body(a, [&](auto body) { soa_bulk_kernel<<<grid, BK_THREADS, BK_SMEM, stream>>>(ld.coords, a.n, body); });
}

void launch_wtma(const SoaLoader& ld, const DeviceInfo& info, const P1Args& a, cudaStream_t stream) {
    const int64_t chunks = (a.n + 31) / 32;
    const int64_t cap = (int64_t)info.sms * info.p1_ctas_per_sm;
    const int64_t want = (chunks + WT_WARPS - 1) / WT_WARPS;
    const unsigned grid = (unsigned)(want < cap ? want : cap);
    const double* c = ld.coords;
    const int64_t n = a.n;
    if (a.coeffs) {
        if (a.stats) pass1_soa_wtma_kernel<true, true><<<grid, WT_THREADS, WT_SMEM, stream>>>(c, n, a.flags, a.coeffs, a.ctl, a.qsub, a.qex, a.stats);
        else pass1_soa_wtma_kernel<true, false><<<grid, WT_THREADS, WT_SMEM, stream>>>(c, n, a.flags, a.coeffs, a.ctl, a.qsub, a.qex, a.stats);
    } else {
        if (a.stats) pass1_soa_wtma_kernel<false, true><<<grid, WT_THREADS, WT_SMEM, stream>>>(c, n, a.flags, a.coeffs, a.ctl, a.qsub, a.qex, a.stats);
        else pass1_soa_wtma_kernel<false, false><<<grid, WT_THREADS, WT_SMEM, stream>>>(c, n, a.flags, a.coeffs, a.ctl, a.qsub, a.qex, a.stats);
    }
}

void launch_cp(const SoaLoader& ld, const DeviceInfo& info, const P1Args& a, cudaStream_t stream) {
    with_pass1_body(a, [&](auto body) {
        constexpr int T = decltype(body)::THREADS;
        const int64_t tiles = (a.n + T - 1) / T;
        const int64_t cap = (int64_t)info.sms * (T == CP_THREADS ? info.p1_ctas_per_sm : info.screen_ctas_per_sm);
        const unsigned grid = (unsigned)(tiles < cap ? tiles : cap);
        soa_cp_kernel<<<grid, T, cp_smem<T, decltype(body)::STAGES>(), stream>>>(ld.coords, a.n, body);
    });
}

// SoA: the selected variant (warp-TMA needs a 16-B aligned coordinate array
// and has no fused screening outputs).
template <>
void launch_pass1<SoaLoader>(const SoaLoader& ld, const DeviceInfo& info, const P1Args& a, cudaStream_t stream) {
    const bool aligned = (((uintptr_t)ld.coords) & 15) == 0;
    if (aligned && info.p1_variant == P1_WTMA && !a.sj) launch_wtma(ld, info, a, stream);
    else if (aligned && info.p1_variant == P1_BULK && !a.sj) launch_bulk(ld, info, a, stream);
    else if (info.p1_variant == P1_CP || info.p1_variant == P1_BULK) launch_cp(ld, info, a, stream);
    else launch_pass1_plain(ld, a, stream);
}

template <class R>
void launch_subdiv(const R& root, const DeviceInfo& info, unsigned blocks, uint8_t* flags, Ctl* ctl,
                   const uint32_t* qsub, const uint32_t* qex, const WarpStacks& fr, hexval_stats* stats,
                   cudaStream_t stream) {
    if (stats) subdiv_kernel<R, true><<<blocks, K4_THREADS, 0, stream>>>(root, flags, ctl, qsub, qex, fr, stats);
    else subdiv_kernel<R, false><<<blocks, K4_THREADS, 0, stream>>>(root, flags, ctl, qsub, qex, fr, stats);
}

// Persistent K4 / bounds grid: one block per SM slot, but no more warps than
// there can be batches of 32 queued hexes (the queue holds at most n), so a
// small call does not reserve (or page in) stacks for idle warps.
unsigned k4_grid(const DeviceInfo& info, int64_t n, int blocks_per_sm) {
    const int64_t full = (int64_t)info.sms * blocks_per_sm;
    const int64_t need = ((n + 31) / 32 + K4_WARPS - 1) / K4_WARPS;
    return (unsigned)(need < full ? (need > 0 ? need : 1) : full);
}

int collect_profile(hexval_profile* p) {
    for (int k = 0; k < p->count; ++k)
        for (int ph = 0; ph < HEXVAL_NUM_PHASES; ++ph) {
            if (ph == HEXVAL_PHASE_EXACT) continue;          // fused into the subdivision kernel
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, p->ev[k][ph][0], p->ev[k][ph][1]) != cudaSuccess) return HEXVAL_ERR_CUDA;
            p->pending_ms[ph] += ms;
            p->pending_launches[ph] += 1;
        }
    p->count = 0;
    return HEXVAL_OK;
}

template <class L>
int run_device(const L& ld, int64_t n, uint8_t* flags, double* coeffs, hexval_stats* stats,
               hexval_profile* prof, cudaStream_t stream, double* sj = nullptr, uint8_t* t1 = nullptr) {
    if (n == 0) return HEXVAL_OK;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return HEXVAL_ERR_CUDA;
    const DeviceInfo& info = device_info<L>(dev);
    const unsigned k4_blocks = k4_grid(info, n, info.k4_blocks_per_sm);
    const size_t warps = (size_t)k4_blocks * K4_WARPS;

    if (prof && prof->count >= hexval_profile::CAP) return HEXVAL_ERR_ARGUMENT;   // read it first
    const size_t ctl_bytes = 256;
    const size_t q_bytes = ((size_t)n * 4 + 255) & ~(size_t)255;
    const size_t sc_bytes = warps * 28 * K4_STRIDE * sizeof(double);
    const size_t total = ctl_bytes + 2 * q_bytes + sc_bytes;
    hexval_scratch::Lease lease;
    if (hexval_scratch::acquire(lease, total, stream) != cudaSuccess) {
        cudaGetLastError();
        return HEXVAL_ERR_ALLOC;
    }
    char* const base = lease.base;
    Ctl* ctl = reinterpret_cast<Ctl*>(base);
    uint32_t* qsub = reinterpret_cast<uint32_t*>(base + ctl_bytes);
    uint32_t* qex = reinterpret_cast<uint32_t*>(base + ctl_bytes + q_bytes);
    WarpStacks fr;
    fr.coef = reinterpret_cast<double*>(base + ctl_bytes + 2 * q_bytes);
    cudaMemsetAsync(ctl, 0, ctl_bytes, stream);

    const int slot = prof ? prof->count++ : -1;
    auto mark = [&](int ph, int which) {
        if (slot >= 0) cudaEventRecord(prof->ev[slot][ph][which], stream);
    };

    mark(HEXVAL_PHASE_PASS1, 0);
    launch_pass1(ld, info, P1Args{n, flags, coeffs, ctl, qsub, qex, stats, sj, t1}, stream);
    mark(HEXVAL_PHASE_PASS1, 1);
    // K5 (exact signs) is fused into K4's batch filling: no separate launch
    mark(HEXVAL_PHASE_SUBDIV, 0);
    const CoordRoot<L> root{ld};
    launch_subdiv(root, info, k4_blocks, flags, ctl, qsub, qex, fr, stats, stream);
    mark(HEXVAL_PHASE_SUBDIV, 1);
    hexval_scratch::release(lease, stream);
    if (cudaGetLastError() != cudaSuccess) return HEXVAL_ERR_CUDA;
    return HEXVAL_OK;
}

bool misaligned(const void* p, size_t a) { return p && (((uintptr_t)p) & (a - 1)) != 0; }

// Steps 4-5 on caller-supplied coefficients: Step 4 + enqueue, then K4.
template <bool STATS>
__global__ void __launch_bounds__(P1_THREADS) bezier_pass_kernel(const double* __restrict__ b, int64_t n,
                                                                 uint8_t* __restrict__ flags, Ctl* ctl,
                                                                 uint32_t* __restrict__ qsub, hexval_stats* stats) {
    const int64_t i = (int64_t)blockIdx.x * P1_THREADS + threadIdx.x;
    int st = -1;
    if (i < n) {
        bool finite = true;
        int m = 0x7fffffff;
#pragma unroll
        for (int sg = 0; sg < 27; ++sg) {
            const double v = __ldg(b + (int64_t)sg * n + i);
            finite &= isfinite(v);
            if (sg >= 8) m = min(m, key(v));
        }
        st = !finite ? ST_NONFINITE : (m > 0 ? ST_VALID : ST_SUB);
        flags[i] = st == ST_NONFINITE ? HEXVAL_NONFINITE : (st == ST_VALID ? HEXVAL_VALID : HEXVAL_FLAG_SUBDIVIDED);
    }
    warp_append(st == ST_SUB, (uint32_t)i, qsub, &ctl->n_sub);
    if (STATS) {
        const unsigned nv = __popc(__ballot_sync(0xffffffffu, st == ST_VALID));
        const unsigned nn = __popc(__ballot_sync(0xffffffffu, st == ST_NONFINITE));
        if ((threadIdx.x & 31) == 0) {
            if (nv) atomicAdd(&stats->n_valid, (unsigned long long)nv);
            if (nn) atomicAdd(&stats->n_nonfinite, (unsigned long long)nn);
        }
    }
}

int run_bezier(const double* b, int64_t n, uint8_t* flags, hexval_stats* stats, cudaStream_t stream) {
    if (n == 0) return HEXVAL_OK;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return HEXVAL_ERR_CUDA;
    const DeviceInfo& info = device_info<SoaLoader>(dev);
    const unsigned k4_blocks = k4_grid(info, n, info.k4_blocks_per_sm);
    const size_t warps = (size_t)k4_blocks * K4_WARPS;
    const size_t ctl_bytes = 256;
    const size_t q_bytes = ((size_t)n * 4 + 255) & ~(size_t)255;
    const size_t sc_bytes = warps * 28 * K4_STRIDE * sizeof(double);
    hexval_scratch::Lease lease;
    if (hexval_scratch::acquire(lease, ctl_bytes + q_bytes + sc_bytes, stream) != cudaSuccess) {
        cudaGetLastError();
        return HEXVAL_ERR_ALLOC;
    }
    char* const base = lease.base;
    Ctl* ctl = reinterpret_cast<Ctl*>(base);
    uint32_t* qsub = reinterpret_cast<uint32_t*>(base + ctl_bytes);
    WarpStacks fr;
    fr.coef = reinterpret_cast<double*>(base + ctl_bytes + q_bytes);
    cudaMemsetAsync(ctl, 0, ctl_bytes, stream);
    const unsigned p1_blocks = (unsigned)((n + P1_THREADS - 1) / P1_THREADS);
    if (stats) bezier_pass_kernel<true><<<p1_blocks, P1_THREADS, 0, stream>>>(b, n, flags, ctl, qsub, stats);
    else bezier_pass_kernel<false><<<p1_blocks, P1_THREADS, 0, stream>>>(b, n, flags, ctl, qsub, stats);
    const CoeffRoot root{b, n};
    launch_subdiv(root, info, k4_blocks, flags, ctl, qsub, qsub, fr, stats, stream);
    hexval_scratch::release(lease, stream);
    if (cudaGetLastError() != cudaSuccess) return HEXVAL_ERR_CUDA;
    return HEXVAL_OK;
}

// NEXT-1 root phase: the plain one-hex-per-thread kernel (measured: 0.853 vs
// 0.867 ms on config 1, 4.01 vs 4.14 ms on config 3 for the cp.async pipeline)
template <class L>
void launch_bounds_root(const L& ld, int64_t n, const BoundsRootBody& body, cudaStream_t stream) {
    plain_kernel<<<(unsigned)((n + P1_THREADS - 1) / P1_THREADS), P1_THREADS, 0, stream>>>(ld, n, body);
}

template <class L>
int run_bounds(const L& ld, int64_t n, double rel_tol, double* lower, double* upper, uint8_t* status,
               unsigned long long* nodes_dev_opt, cudaStream_t stream) {
    if (n == 0) return HEXVAL_OK;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return HEXVAL_ERR_CUDA;
    const DeviceInfo& info = device_info<SoaLoader>(dev);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bounds_kernel<L>, K4_THREADS, 0);
    if (occ < 1) occ = 1;
    const int64_t blocks = k4_grid(info, n, occ);
    const size_t warps = (size_t)blocks * K4_WARPS;
    const size_t q_bytes = ((size_t)n * 4 + 255) & ~(size_t)255;
    const size_t sc_bytes = warps * 28 * K4_STRIDE * sizeof(double);
    hexval_scratch::Lease lease;
    if (hexval_scratch::acquire(lease, 256 + q_bytes + sc_bytes, stream) != cudaSuccess) {
        cudaGetLastError();
        return HEXVAL_ERR_ALLOC;
    }
    char* const base = lease.base;
    unsigned* ctlq = reinterpret_cast<unsigned*>(base);          // [0] queue length, [1] fetch cursor
    uint32_t* q = reinterpret_cast<uint32_t*>(base + 256);
    WarpStacks ws;
    ws.coef = reinterpret_cast<double*>(base + 256 + q_bytes);
    cudaMemsetAsync(ctlq, 0, 256, stream);
    launch_bounds_root(ld, n, BoundsRootBody{rel_tol, lower, upper, status, ctlq, q}, stream);
    bounds_kernel<L><<<(unsigned)blocks, K4_THREADS, 0, stream>>>(ld, rel_tol, lower, upper, status, ctlq, q, ws,
                                                                    nodes_dev_opt);
    hexval_scratch::release(lease, stream);
    return cudaGetLastError() == cudaSuccess ? HEXVAL_OK : HEXVAL_ERR_CUDA;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int hexval_check_soa_ex(const double* coords, int64_t n, uint8_t* flags_out, double* coeffs_out_opt,
                        hexval_stats* stats_dev_opt, hexval_profile* profile_opt, cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX) return HEXVAL_ERR_ARGUMENT;
    if (n > 0 && (!coords || !flags_out)) return HEXVAL_ERR_ARGUMENT;
    if (misaligned(coords, 8) || misaligned(coeffs_out_opt, 8) || misaligned(stats_dev_opt, 8))
        return HEXVAL_ERR_ALIGNMENT;
    SoaLoader ld{coords, n};
    return run_device(ld, n, flags_out, coeffs_out_opt, stats_dev_opt, profile_opt, stream);
}

int hexval_check_indexed_ex(const double* vertices, const int32_t* hex_idx, int64_t n, uint8_t* flags_out,
                            double* coeffs_out_opt, hexval_stats* stats_dev_opt, hexval_profile* profile_opt,
                            cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX) return HEXVAL_ERR_ARGUMENT;
    if (n > 0 && (!vertices || !hex_idx || !flags_out)) return HEXVAL_ERR_ARGUMENT;
    if (misaligned(vertices, 8) || misaligned(hex_idx, 4) || misaligned(coeffs_out_opt, 8) ||
        misaligned(stats_dev_opt, 8))
        return HEXVAL_ERR_ALIGNMENT;
    IdxLoader ld{vertices, hex_idx};
    return run_device(ld, n, flags_out, coeffs_out_opt, stats_dev_opt, profile_opt, stream);
}

int hexval_classify_bezier(const double* coeffs, int64_t n, uint8_t* flags_out, hexval_stats* stats_dev_opt,
                           cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX) return HEXVAL_ERR_ARGUMENT;
    if (n > 0 && (!coeffs || !flags_out)) return HEXVAL_ERR_ARGUMENT;
    if (misaligned(coeffs, 8) || misaligned(stats_dev_opt, 8)) return HEXVAL_ERR_ALIGNMENT;
    return run_bezier(coeffs, n, flags_out, stats_dev_opt, stream);
}

int hexval_check_screen_soa(const double* coords, int64_t n, uint8_t* flags_out, double* sj_min_out,
                            uint8_t* test1_out, cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX) return HEXVAL_ERR_ARGUMENT;
    if (n > 0 && (!coords || !flags_out || !sj_min_out || !test1_out)) return HEXVAL_ERR_ARGUMENT;
    if (misaligned(coords, 8) || misaligned(sj_min_out, 8)) return HEXVAL_ERR_ALIGNMENT;
    SoaLoader ld{coords, n};
    return run_device(ld, n, flags_out, nullptr, nullptr, nullptr, stream, sj_min_out, test1_out);
}

int hexval_check_screen_indexed(const double* vertices, const int32_t* hex_idx, int64_t n, uint8_t* flags_out,
                                double* sj_min_out, uint8_t* test1_out, cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX) return HEXVAL_ERR_ARGUMENT;
    if (n > 0 && (!vertices || !hex_idx || !flags_out || !sj_min_out || !test1_out)) return HEXVAL_ERR_ARGUMENT;
    if (misaligned(vertices, 8) || misaligned(hex_idx, 4) || misaligned(sj_min_out, 8)) return HEXVAL_ERR_ALIGNMENT;
    IdxLoader ld{vertices, hex_idx};
    return run_device(ld, n, flags_out, nullptr, nullptr, nullptr, stream, sj_min_out, test1_out);
}

int hexval_corner_quality_soa(const double* coords, int64_t n, double* sj_min_out_opt, uint8_t* test1_out_opt,
                              cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX) return HEXVAL_ERR_ARGUMENT;
    if (n > 0 && !coords) return HEXVAL_ERR_ARGUMENT;
    if (misaligned(coords, 8) || misaligned(sj_min_out_opt, 8)) return HEXVAL_ERR_ALIGNMENT;
    if (n == 0) return HEXVAL_OK;
    quality_kernel<SoaLoader><<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(SoaLoader{coords, n}, n, sj_min_out_opt,
                                                                               test1_out_opt);
    return cudaGetLastError() == cudaSuccess ? HEXVAL_OK : HEXVAL_ERR_CUDA;
}

int hexval_corner_quality_indexed(const double* vertices, const int32_t* hex_idx, int64_t n, double* sj_min_out_opt,
                                  uint8_t* test1_out_opt, cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX) return HEXVAL_ERR_ARGUMENT;
    if (n > 0 && (!vertices || !hex_idx)) return HEXVAL_ERR_ARGUMENT;
    if (misaligned(vertices, 8) || misaligned(hex_idx, 4) || misaligned(sj_min_out_opt, 8)) return HEXVAL_ERR_ALIGNMENT;
    if (n == 0) return HEXVAL_OK;
    quality_kernel<IdxLoader><<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(IdxLoader{vertices, hex_idx}, n,
                                                                               sj_min_out_opt, test1_out_opt);
    return cudaGetLastError() == cudaSuccess ? HEXVAL_OK : HEXVAL_ERR_CUDA;
}

int hexval_min_detj_bounds_soa(const double* coords, int64_t n, double rel_tol, double* lower_out,
                               double* upper_out, uint8_t* status_out_opt, unsigned long long* nodes_dev_opt,
                               cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX || !(rel_tol >= 0.0)) return HEXVAL_ERR_ARGUMENT;
    if (n > 0 && (!coords || !lower_out || !upper_out)) return HEXVAL_ERR_ARGUMENT;
    if (misaligned(coords, 8) || misaligned(lower_out, 8) || misaligned(upper_out, 8) || misaligned(nodes_dev_opt, 8))
        return HEXVAL_ERR_ALIGNMENT;
    return run_bounds(SoaLoader{coords, n}, n, rel_tol, lower_out, upper_out, status_out_opt, nodes_dev_opt, stream);
}

int hexval_min_detj_bounds_indexed(const double* vertices, const int32_t* hex_idx, int64_t n, double rel_tol,
                                   double* lower_out, double* upper_out, uint8_t* status_out_opt,
                                   unsigned long long* nodes_dev_opt, cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX || !(rel_tol >= 0.0)) return HEXVAL_ERR_ARGUMENT;
    if (n > 0 && (!vertices || !hex_idx || !lower_out || !upper_out)) return HEXVAL_ERR_ARGUMENT;
    if (misaligned(vertices, 8) || misaligned(hex_idx, 4) || misaligned(lower_out, 8) || misaligned(upper_out, 8) ||
        misaligned(nodes_dev_opt, 8))
        return HEXVAL_ERR_ALIGNMENT;
    return run_bounds(IdxLoader{vertices, hex_idx}, n, rel_tol, lower_out, upper_out, status_out_opt, nodes_dev_opt,
                      stream);
}

int hexval_select_valid(const uint8_t* flags, int64_t n, const int32_t* group_opt, int64_t n_groups,
                        int32_t* ids_out_opt, long long* count_dev, int32_t* group_counts_opt, cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX || n_groups < 0 || !count_dev) return HEXVAL_ERR_ARGUMENT;
    if (misaligned(count_dev, 8)) return HEXVAL_ERR_ALIGNMENT;
    if (n == 0) {                                     // nothing to select (empty arrays may be NULL)
        cudaMemsetAsync(count_dev, 0, sizeof(long long), stream);
        return cudaGetLastError() == cudaSuccess ? HEXVAL_OK : HEXVAL_ERR_CUDA;
    }
    if (!flags || ((group_opt == nullptr) != (group_counts_opt == nullptr))) return HEXVAL_ERR_ARGUMENT;
    if (misaligned(ids_out_opt, 4) || misaligned(group_opt, 4) || misaligned(group_counts_opt, 4))
        return HEXVAL_ERR_ALIGNMENT;
    const int64_t tiles = (n + SEL_TILE - 1) / SEL_TILE;
    hexval_scratch::Lease lease;
    if (hexval_scratch::acquire(lease, (size_t)tiles * sizeof(unsigned), stream) != cudaSuccess) {
        cudaGetLastError();
        return HEXVAL_ERR_ALLOC;
    }
    unsigned* tc = reinterpret_cast<unsigned*>(lease.base);
    select_count_kernel<<<(unsigned)tiles, SEL_THREADS, 0, stream>>>(flags, n, group_opt, group_counts_opt, tc);
    select_scan_kernel<<<1, 1024, 0, stream>>>(tc, tiles, count_dev);
    if (ids_out_opt) select_write_kernel<<<(unsigned)tiles, SEL_THREADS, 0, stream>>>(flags, n, tc, ids_out_opt);
    hexval_scratch::release(lease, stream);
    return cudaGetLastError() == cudaSuccess ? HEXVAL_OK : HEXVAL_ERR_CUDA;
}

int hexval_check_quad_soa(const double* coords, int64_t n, uint8_t* flags_out, double* J_out_opt,
                          cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX) return HEXVAL_ERR_ARGUMENT;
    if (n > 0 && (!coords || !flags_out)) return HEXVAL_ERR_ARGUMENT;
    if (misaligned(coords, 8) || misaligned(J_out_opt, 8)) return HEXVAL_ERR_ALIGNMENT;
    if (n == 0) return HEXVAL_OK;
    quad_kernel<<<(unsigned)((n + 256 * QPT - 1) / (256 * QPT)), 256, 0, stream>>>(coords, n, flags_out, J_out_opt);
    return cudaGetLastError() == cudaSuccess ? HEXVAL_OK : HEXVAL_ERR_CUDA;
}

int hexval_check_soa(const double* coords, int64_t n, uint8_t* flags_out, double* coeffs_out_opt,
                     cudaStream_t stream) {
    return hexval_check_soa_ex(coords, n, flags_out, coeffs_out_opt, nullptr, nullptr, stream);
}

int hexval_check_indexed(const double* vertices, const int32_t* hex_idx, int64_t n, uint8_t* flags_out,
                         double* coeffs_out_opt, cudaStream_t stream) {
    return hexval_check_indexed_ex(vertices, hex_idx, n, flags_out, coeffs_out_opt, nullptr, nullptr, stream);
}

// ---- host-resident (end-to-end) calls ---------------------------------------
namespace {

struct HostPipe {
    cudaStream_t s[2] = {nullptr, nullptr};
    cudaEvent_t start = nullptr;
    bool ok = false;
};

int host_pipe_init(HostPipe& hp, cudaStream_t user) {
    for (int k = 0; k < 2; ++k)
        if (cudaStreamCreateWithFlags(&hp.s[k], cudaStreamNonBlocking) != cudaSuccess) return HEXVAL_ERR_CUDA;
    if (cudaEventCreateWithFlags(&hp.start, cudaEventDisableTiming) != cudaSuccess) return HEXVAL_ERR_CUDA;
    // order after prior work on the user's stream
    if (cudaEventRecord(hp.start, user) != cudaSuccess) return HEXVAL_ERR_CUDA;
    for (int k = 0; k < 2; ++k) cudaStreamWaitEvent(hp.s[k], hp.start, 0);
    hp.ok = true;
    return HEXVAL_OK;
}

void host_pipe_fini(HostPipe& hp) {
    for (int k = 0; k < 2; ++k)
        if (hp.s[k]) { cudaStreamSynchronize(hp.s[k]); cudaStreamDestroy(hp.s[k]); }
    if (hp.start) cudaEventDestroy(hp.start);
}

}  // namespace

int hexval_check_soa_host(const double* coords_host, int64_t n, uint8_t* flags_host, double* coeffs_host_opt,
                          int64_t chunk_hexes, cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX) return HEXVAL_ERR_ARGUMENT;
    if (n > 0 && (!coords_host || !flags_host)) return HEXVAL_ERR_ARGUMENT;
    if (n == 0) return HEXVAL_OK;
    const int64_t C = chunk_hexes > 0 ? (chunk_hexes < n ? chunk_hexes : n) : (n < (1 << 21) ? n : (1 << 21));
    HostPipe hp;
    int rc = host_pipe_init(hp, stream);
    double* dc[2] = {nullptr, nullptr};
    uint8_t* df[2] = {nullptr, nullptr};
    double* dk[2] = {nullptr, nullptr};
    for (int k = 0; k < 2 && rc == HEXVAL_OK; ++k) {
        if (hexval_scratch::alloc_async((void**)&dc[k], (size_t)24 * C * sizeof(double), hp.s[k]) != cudaSuccess ||
            hexval_scratch::alloc_async((void**)&df[k], (size_t)C, hp.s[k]) != cudaSuccess ||
            (coeffs_host_opt && hexval_scratch::alloc_async((void**)&dk[k], (size_t)27 * C * sizeof(double), hp.s[k]) != cudaSuccess))
            rc = HEXVAL_ERR_ALLOC;
    }
    for (int64_t off = 0, it = 0; off < n && rc == HEXVAL_OK; off += C, ++it) {
        const int k = (int)(it & 1);
        const int64_t m = (n - off) < C ? (n - off) : C;
        cudaStream_t s = hp.s[k];
        for (int p = 0; p < 24; ++p)
            cudaMemcpyAsync(dc[k] + (size_t)p * m, coords_host + (size_t)p * n + off, (size_t)m * sizeof(double),
                            cudaMemcpyHostToDevice, s);
        rc = hexval_check_soa_ex(dc[k], m, df[k], dk[k], nullptr, nullptr, s);
        cudaMemcpyAsync(flags_host + off, df[k], (size_t)m, cudaMemcpyDeviceToHost, s);
        if (coeffs_host_opt)
            for (int sg = 0; sg < 27; ++sg)
                cudaMemcpyAsync(coeffs_host_opt + (size_t)sg * n + off, dk[k] + (size_t)sg * m,
                                (size_t)m * sizeof(double), cudaMemcpyDeviceToHost, s);
    }
    for (int k = 0; k < 2; ++k) {
        if (dc[k]) cudaFreeAsync(dc[k], hp.s[k]);
        if (df[k]) cudaFreeAsync(df[k], hp.s[k]);
        if (dk[k]) cudaFreeAsync(dk[k], hp.s[k]);
    }
    host_pipe_fini(hp);
    if (cudaGetLastError() != cudaSuccess && rc == HEXVAL_OK) rc = HEXVAL_ERR_CUDA;
    return rc;
}

int hexval_check_indexed_host(const double* vertices_host, int64_t nv, const int32_t* hex_idx_host, int64_t n,
                              uint8_t* flags_host, double* coeffs_host_opt, int64_t chunk_hexes,
                              cudaStream_t stream) {
    if (n < 0 || n > INT32_MAX || nv < 0) return HEXVAL_ERR_ARGUMENT;
    if (n > 0 && (!vertices_host || !hex_idx_host || !flags_host)) return HEXVAL_ERR_ARGUMENT;
    if (n == 0) return HEXVAL_OK;
    const int64_t C = chunk_hexes > 0 ? (chunk_hexes < n ? chunk_hexes : n) : (n < (1 << 22) ? n : (1 << 22));
    HostPipe hp;
    int rc = host_pipe_init(hp, stream);
    double* dv = nullptr;
    int32_t* di[2] = {nullptr, nullptr};
    uint8_t* df[2] = {nullptr, nullptr};
    double* dk[2] = {nullptr, nullptr};
    cudaEvent_t vready = nullptr;
    if (rc == HEXVAL_OK) {
        if (hexval_scratch::alloc_async((void**)&dv, (size_t)3 * nv * sizeof(double) + 8, hp.s[0]) != cudaSuccess) rc = HEXVAL_ERR_ALLOC;
        else {
            cudaMemcpyAsync(dv, vertices_host, (size_t)3 * nv * sizeof(double), cudaMemcpyHostToDevice, hp.s[0]);
            cudaEventCreateWithFlags(&vready, cudaEventDisableTiming);
            cudaEventRecord(vready, hp.s[0]);
            cudaStreamWaitEvent(hp.s[1], vready, 0);
        }
    }
    for (int k = 0; k < 2 && rc == HEXVAL_OK; ++k) {
        if (hexval_scratch::alloc_async((void**)&di[k], (size_t)8 * C * sizeof(int32_t), hp.s[k]) != cudaSuccess ||
            hexval_scratch::alloc_async((void**)&df[k], (size_t)C, hp.s[k]) != cudaSuccess ||
            (coeffs_host_opt && hexval_scratch::alloc_async((void**)&dk[k], (size_t)27 * C * sizeof(double), hp.s[k]) != cudaSuccess))
            rc = HEXVAL_ERR_ALLOC;
    }
    for (int64_t off = 0, it = 0; off < n && rc == HEXVAL_OK; off += C, ++it) {
        const int k = (int)(it & 1);
        const int64_t m = (n - off) < C ? (n - off) : C;
        cudaStream_t s = hp.s[k];
        cudaMemcpyAsync(di[k], hex_idx_host + (size_t)8 * off, (size_t)8 * m * sizeof(int32_t),
                        cudaMemcpyHostToDevice, s);
        rc = hexval_check_indexed_ex(dv, di[k], m, df[k], dk[k], nullptr, nullptr, s);
        cudaMemcpyAsync(flags_host + off, df[k], (size_t)m, cudaMemcpyDeviceToHost, s);
        if (coeffs_host_opt)
            for (int sg = 0; sg < 27; ++sg)
                cudaMemcpyAsync(coeffs_host_opt + (size_t)sg * n + off, dk[k] + (size_t)sg * m,
                                (size_t)m * sizeof(double), cudaMemcpyDeviceToHost, s);
    }
    // the vertex buffer is freed after both pipelines finish
    if (vready) {
        cudaEventRecord(vready, hp.s[1]);
        cudaStreamWaitEvent(hp.s[0], vready, 0);
    }
    for (int k = 0; k < 2; ++k) {
        if (di[k]) cudaFreeAsync(di[k], hp.s[k]);
        if (df[k]) cudaFreeAsync(df[k], hp.s[k]);
        if (dk[k]) cudaFreeAsync(dk[k], hp.s[k]);
    }
    if (dv) cudaFreeAsync(dv, hp.s[0]);
    host_pipe_fini(hp);
    if (vready) cudaEventDestroy(vready);
    if (cudaGetLastError() != cudaSuccess && rc == HEXVAL_OK) rc = HEXVAL_ERR_CUDA;
    return rc;
}

// ---- profiling ------------------------------------------------------------
hexval_profile* hexval_profile_create(void) {
    hexval_profile* p = new hexval_profile();
    for (int k = 0; k < hexval_profile::CAP; ++k)
        for (int ph = 0; ph < HEXVAL_NUM_PHASES; ++ph)
            for (int w = 0; w < 2; ++w)
                if (cudaEventCreate(&p->ev[k][ph][w]) != cudaSuccess) {
                    delete p;
                    return nullptr;
                }
    return p;
}

void hexval_profile_destroy(hexval_profile* p) {
    if (!p) return;
    for (int k = 0; k < hexval_profile::CAP; ++k)
        for (int ph = 0; ph < HEXVAL_NUM_PHASES; ++ph)
            for (int w = 0; w < 2; ++w) cudaEventDestroy(p->ev[k][ph][w]);
    delete p;
}

int hexval_profile_read(hexval_profile* p, double* ms_out, long long* launches_out) {
    if (!p) return HEXVAL_ERR_ARGUMENT;
    const int rc = collect_profile(p);
    for (int ph = 0; ph < HEXVAL_NUM_PHASES; ++ph) {
        if (ms_out) ms_out[ph] = p->pending_ms[ph];
        if (launches_out) launches_out[ph] = p->pending_launches[ph];
        p->pending_ms[ph] = 0;
        p->pending_launches[ph] = 0;
    }
    return rc;
}

const char* hexval_status_string(int status) {
    switch (status) {
        case HEXVAL_OK: return "ok";
        case HEXVAL_ERR_ARGUMENT: return "invalid argument (n < 0, n > INT32_MAX, NULL buffer, or a profile holding 256 unread calls)";
        case HEXVAL_ERR_ALIGNMENT: return "misaligned pointer";
        case HEXVAL_ERR_CUDA: return "CUDA launch or copy error";
        case HEXVAL_ERR_ALLOC: return "scratch allocation failed";
        default: return "unknown status";
    }
}

int hexval_scratch_info(int device, size_t* bytes_reserved_out, int* arenas_out) {
    if (device < 0 || device >= 64) return HEXVAL_ERR_ARGUMENT;
    hexval_scratch::info(device, bytes_reserved_out, arenas_out);
    return HEXVAL_OK;
}

int hexval_scratch_release(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return HEXVAL_ERR_CUDA;
    hexval_scratch::release_all(dev);
    return cudaGetLastError() == cudaSuccess ? HEXVAL_OK : HEXVAL_ERR_CUDA;
}

int hexval_version(void) { return 200; }

int hexval_kernel_launches_per_call(void) { return 2; }

}  // extern "C"
