// hexval.cu -- kernels and C ABI of the B200 hot path for the robust validity
// check of linear hexahedra (section 6).
//
//   K1/K2 pass1_kernel   one hex per thread: coalesced fp64 loads (SoA planes,
//                        or int32 connectivity + vertex gather), 20 tet
//                        determinants, Step 2, 27 Bezier coefficients, Step 4,
//                        flags, optional coefficients, and (K3) warp-ballot +
//                        block-scan compaction of undecided / ambiguous hexes.
//   K5    exact_kernel   exact signs of root samples within their rounding
//                        bound of 0 (Kulisch accumulator), then Steps 3-4.
//   K4    subdiv_kernel  persistent grid, dynamic hex fetch, per-thread
//                        depth-first recursive_subdivision with a depth-20
//                        frame stack in a global scratch buffer.
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

using namespace hexval;

namespace {

constexpr int P1_THREADS = 256;
constexpr int K5_THREADS = 128;
constexpr int K4_THREADS = 256;

// flags placeholders written by pass 1 for hexes that later kernels finish
constexpr uint8_t PENDING_EXACT = 0xFF;

struct Ctl {                 // per-call control block (device scratch)
    unsigned int n_sub;      // subdivision queue length
    unsigned int n_exact;    // exact-sign queue length
    unsigned int k4_next;    // dynamic fetch cursor of the subdivision kernel
    unsigned int pad[5];
};

// ---------------------------------------------------------------------------
// loaders: SoA planes or indexed gather
// ---------------------------------------------------------------------------
struct SoaLoader {
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
};

struct IdxLoader {
    const double* __restrict__ verts;
    const int32_t* __restrict__ idx;
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
};

// NONFINITE (reading G13): a coordinate is NaN/Inf or |x| > 2^300
__device__ __forceinline__ bool out_of_range(const double* X) {
    int mk = 0;
#pragma unroll
    for (int p = 0; p < 24; ++p) mk = max(mk, abskey(X[p]));
    if (mk < 0x52B00000) return false;                 // every |x| < 2^300
    bool bad = false;
#pragma unroll
    for (int p = 0; p < 24; ++p) bad |= !(fabs(X[p]) <= 0x1p300);
    return bad;
}

// Step 2 classification shared by pass 1 and the exact kernel.
enum : int { ST_INVALID = 0, ST_VALID = 1, ST_NONFINITE = 3, ST_SUB = 4, ST_EXACT = 5 };

__device__ __forceinline__ int step2_class(const Samples& s, double tau2) {
    int km = key(s.c[0]);
#pragma unroll
    for (int k = 1; k < 8; ++k) km = min(km, key(s.c[k]));
#pragma unroll
    for (int e = 0; e < 12; ++e) km = min(km, key(s.d[e]));
    if (km > key(tau2)) return ST_VALID;               // every sample > tau2 > 0: robustly positive
    bool neg = false, amb = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) { neg |= s.c[k] < -tau2; amb |= fabs(s.c[k]) <= tau2; }
#pragma unroll
    for (int e = 0; e < 12; ++e) { neg |= s.d[e] < -tau2; amb |= fabs(s.d[e]) <= tau2; }
    if (neg) return ST_INVALID;                        // some sample robustly negative
    return amb ? ST_EXACT : ST_VALID;
}

__device__ __forceinline__ void write_coeffs(double* __restrict__ coeffs, int64_t n, int64_t i,
                                             const Samples& s, const Coeffs& t) {
    double P[27];
    root_coeffs(s, t, P);
#pragma unroll
    for (int sg = 0; sg < 27; ++sg) __stcs(coeffs + (int64_t)sg * n + i, P[kSigmaToSlot[sg]]);
}

// K3: warp ballot + block exclusive scan + one atomic per block
template <int NW>
__device__ __forceinline__ void block_append(bool pred, uint32_t val, uint32_t* __restrict__ q,
                                             unsigned int* counter, unsigned int* s_warp) {
    const int total = __syncthreads_count(pred);
    if (total == 0) return;                            // block-uniform
    const unsigned bal = __ballot_sync(0xffffffffu, pred);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned run = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const unsigned c = s_warp[w];
            s_warp[w] = run;
            run += c;
        }
        s_warp[32] = atomicAdd(counter, run);
    }
    __syncthreads();
    if (pred) q[s_warp[32] + s_warp[warp] + __popc(bal & ((1u << lane) - 1u))] = val;
}

// ---------------------------------------------------------------------------
// K1 / K2: pass 1
// ---------------------------------------------------------------------------
template <class L, bool COEFFS, bool STATS>
__global__ void __launch_bounds__(P1_THREADS) pass1_kernel(L ld, int64_t n, uint8_t* __restrict__ flags,
                                                           double* __restrict__ coeffs, Ctl* ctl,
                                                           uint32_t* __restrict__ qsub,
                                                           uint32_t* __restrict__ qexact,
                                                           hexval_stats* stats) {
    __shared__ unsigned int s_sub[33], s_ex[33];
    const int64_t i = (int64_t)blockIdx.x * P1_THREADS + threadIdx.x;
    const bool active = i < n;
    int st = -1;
    if (active) {
        double X[24];
        ld.load_stream(i, X);
        if (out_of_range(X)) {
            st = ST_NONFINITE;
        } else {
            Samples s;
            samples20(X, s);                                  // S1 + S2
            st = step2_class(s, step2_tau(s.ekey));           // S3 (Step 2)
            Coeffs t;
            transform(s, t);                                  // S4 (Step 3)
            if (st == ST_VALID && !step4_positive(t)) st = ST_SUB;   // S5 (Step 4)
            if (COEFFS) write_coeffs(coeffs, n, i, s, t);
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
    }
    // S6: compaction into the two work queues
    block_append<P1_THREADS / 32>(st == ST_SUB, (uint32_t)i, qsub, &ctl->n_sub, s_sub);
    block_append<P1_THREADS / 32>(st == ST_EXACT, (uint32_t)i, qexact, &ctl->n_exact, s_ex);
    if (STATS) {
        const int nv = __syncthreads_count(st == ST_VALID);
        const int ni = __syncthreads_count(st == ST_INVALID);
        const int nn = __syncthreads_count(st == ST_NONFINITE);
        if (threadIdx.x == 0) {
            if (nv) atomicAdd(&stats->n_valid, (unsigned long long)nv);
            if (ni) atomicAdd(&stats->n_invalid, (unsigned long long)ni);
            if (nn) atomicAdd(&stats->n_nonfinite, (unsigned long long)nn);
        }
    }
}

// ---------------------------------------------------------------------------
// K5: exact signs for ambiguous root samples, then Steps 3-4
// ---------------------------------------------------------------------------
template <class L, bool STATS>
__global__ void __launch_bounds__(K5_THREADS) exact_kernel(L ld, uint8_t* __restrict__ flags, Ctl* ctl,
                                                           const uint32_t* __restrict__ qexact,
                                                           uint32_t* __restrict__ qsub, hexval_stats* stats) {
    const unsigned cnt = *((volatile unsigned*)&ctl->n_exact);
    for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += gridDim.x * blockDim.x) {
        const uint32_t h = qexact[q];
        double X[24];
        ld.load(h, X);
        Samples s;
        samples20(X, s);
        const double tau2 = step2_tau(s.ekey);
        bool invalid = false;
        for (int j = 0; j < 20 && !invalid; ++j) {
            const double x = j < 8 ? s.c[j] : s.d[j - 8];
            if (x < -tau2) invalid = true;
            else if (fabs(x) <= tau2) invalid = exact_sample_sign(X, j) <= 0;
        }
        uint8_t f;
        if (invalid) {
            f = HEXVAL_INVALID;
        } else {
            Coeffs t;
            transform(s, t);
            if (step4_positive(t)) {
                f = HEXVAL_VALID;
            } else {
                f = HEXVAL_FLAG_SUBDIVIDED;
                qsub[atomicAdd(&ctl->n_sub, 1u)] = h;
            }
        }
        flags[h] = f;
        if (STATS) {
            atomicAdd(&stats->n_exact, 1ull);
            if (f == HEXVAL_INVALID) atomicAdd(&stats->n_invalid, 1ull);
            if (f == HEXVAL_VALID) atomicAdd(&stats->n_valid, 1ull);
        }
    }
}

// ---------------------------------------------------------------------------
// K4: recursive_subdivision, depth-first per thread
// ---------------------------------------------------------------------------
// Test the 8 children of node P; returns -1 if some child corner <= 0
// (INVALID) else the bit mask (bit hx + 2 hy + 4 hz) of undecided children.
__device__ __forceinline__ int test_children(const double* P) {
    int pend = 0;
    bool bad = false;
    double G1[45];
    both_split<0>(P, G1);
#pragma unroll
    for (int hx = 0; hx < 2; ++hx) {
        double A[27];
        take_half<0>(G1, hx, A);
        double G2[45];
        both_split<1>(A, G2);
#pragma unroll
        for (int hy = 0; hy < 2; ++hy) {
            double B[27];
            take_half<1>(G2, hy, B);
            // zeta split of the 9 lines of B, classifying both children as the
            // lines are produced (child hz takes points 2hz..2hz+2 of each line)
            int mc0 = 0x7fffffff, mc1 = 0x7fffffff, mi0 = 0x7fffffff, mi1 = 0x7fffffff;
#pragma unroll
            for (int u = 0; u < 3; ++u)
#pragma unroll
                for (int w = 0; w < 3; ++w) {
                    const double p0 = B[u + 3 * w], p1 = B[u + 3 * w + 9], p2 = B[u + 3 * w + 18];
                    const double m01 = half_sum(p0, p1), m12 = half_sum(p1, p2), m = half_sum(m01, m12);
                    const bool corner_line = (u != 1) && (w != 1);
                    // child 0: (p0, m01, m); child 1: (m, m12, p2); points 0 and 2 of a
                    // child line are corners iff the line itself is a corner line
                    if (corner_line) {
                        mc0 = min(mc0, min(key(p0), key(m)));
                        mc1 = min(mc1, min(key(m), key(p2)));
                    } else {
                        mi0 = min(mi0, min(key(p0), key(m)));
                        mi1 = min(mi1, min(key(m), key(p2)));
                    }
                    mi0 = min(mi0, key(m01));
                    mi1 = min(mi1, key(m12));
                }
            bad |= (mc0 <= 0) | (mc1 <= 0);
            const int b0 = hx + 2 * hy;
            if (mi0 <= 0) pend |= 1 << b0;
            if (mi1 <= 0) pend |= 1 << (b0 + 4);
        }
    }
    return bad ? -1 : pend;
}

struct Frames {
    double* coef;        // [lvl][27][T]
    unsigned char* mask; // [lvl][T]
    unsigned T;
};

// Root coefficients of queued item h: recomputed from the coordinates with
// the pass-1 arithmetic (bit-identical), or read from caller-supplied Bezier
// coefficients (hexval_classify_bezier).
template <class L>
struct CoordRoot {
    L ld;
    __device__ __forceinline__ void operator()(uint32_t h, double* P) const {
        double X[24];
        ld.load(h, X);
        Samples s;
        samples20(X, s);
        Coeffs t;
        transform(s, t);
        root_coeffs(s, t, P);
    }
};

struct CoeffRoot {
    const double* __restrict__ b;   // coefficient-major, b[sigma*n + h]
    int64_t n;
    __device__ __forceinline__ void operator()(uint32_t h, double* P) const {
#pragma unroll
        for (int sg = 0; sg < 27; ++sg) P[kSigmaToSlot[sg]] = __ldg(b + (int64_t)sg * n + h);
    }
};

template <class R, bool STATS>
__global__ void __launch_bounds__(K4_THREADS, 1) subdiv_kernel(R root, uint8_t* __restrict__ flags, Ctl* ctl,
                                                               const uint32_t* __restrict__ qsub, Frames fr,
                                                               hexval_stats* stats) {
    const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned T = fr.T;
    const unsigned total = *((volatile unsigned*)&ctl->n_sub);
    double* const fc = fr.coef + tid;
    unsigned char* const fm = fr.mask + tid;
    for (;;) {
        const unsigned q = atomicAdd(&ctl->k4_next, 1u);
        if (q >= total) break;
        const uint32_t h = qsub[q];
        double P[27];
        root(h, P);                                      // bit-identical to pass 1
        unsigned long long nodes = 0;
        int maxd = 0;
        bool undet = false, invalid = false;
        unsigned levels = 0;                             // bit d: frame d has pending children
        int d = 0;                                       // depth of node P
        for (;;) {
            ++nodes;
            // keep the node: its other undecided children are extracted from it later
#pragma unroll
            for (int c = 0; c < 27; ++c) fc[(size_t)(d * 27 + c) * T] = P[c];
            int pend = test_children(P);
            maxd = max(maxd, d + 1);
            if (pend < 0) { invalid = true; break; }
            if (pend && d + 1 >= MAX_DEPTH) { undet = true; pend = 0; }   // depth cap (reading G5)
            int o;
            if (pend) {
                o = __ffs(pend) - 1;
                pend &= pend - 1;
                if (pend) { fm[(size_t)d * T] = (unsigned char)pend; levels |= 1u << d; }
            } else {
                // backtrack to the deepest frame with pending children
                if (levels == 0) break;
                d = 31 - __clz(levels);
                unsigned m = fm[(size_t)d * T];
                o = __ffs(m) - 1;
                m &= m - 1;
                if (m) fm[(size_t)d * T] = (unsigned char)m;
                else levels &= ~(1u << d);
            }
            double Pp[27];
#pragma unroll
            for (int c = 0; c < 27; ++c) Pp[c] = fc[(size_t)(d * 27 + c) * T];
            extract_child(Pp, o & 1, (o >> 1) & 1, o >> 2, P);
            ++d;
        }
        const uint8_t verdict = invalid ? HEXVAL_INVALID : (undet ? HEXVAL_UNDETERMINED : HEXVAL_VALID);
        flags[h] = verdict | HEXVAL_FLAG_SUBDIVIDED;
        if (STATS) {
            atomicAdd(&stats->n_subdivided, 1ull);
            atomicAdd(&stats->n_nodes, nodes);
            atomicMax(&stats->max_depth, (unsigned long long)maxd);
            atomicAdd(verdict == HEXVAL_INVALID ? &stats->n_invalid
                      : (verdict == HEXVAL_VALID ? &stats->n_valid : &stats->n_undetermined), 1ull);
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct DeviceInfo {
    int sms = 0;
    int k4_blocks_per_sm = 0;
    bool ok = false;
};

DeviceInfo g_info[64];
std::mutex g_info_mu;

template <class L>
const DeviceInfo& device_info(int dev) {
    std::lock_guard<std::mutex> lk(g_info_mu);
    DeviceInfo& d = g_info[dev & 63];
    if (!d.ok) {
        cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, subdiv_kernel<CoordRoot<SoaLoader>, false>, K4_THREADS, 0);
        d.k4_blocks_per_sm = occ > 0 ? occ : 1;
        // keep freed stream-ordered scratch in the pool between calls
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
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

int collect_profile(hexval_profile* p) {
    for (int k = 0; k < p->count; ++k)
        for (int ph = 0; ph < HEXVAL_NUM_PHASES; ++ph) {
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
               hexval_profile* prof, cudaStream_t stream) {
    if (n == 0) return HEXVAL_OK;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return HEXVAL_ERR_CUDA;
    const DeviceInfo& info = device_info<L>(dev);
    const unsigned T = (unsigned)(info.sms * info.k4_blocks_per_sm * K4_THREADS);

    if (prof && prof->count >= hexval_profile::CAP) return HEXVAL_ERR_ARGUMENT;   // read it first
    const size_t ctl_bytes = 256;
    const size_t q_bytes = ((size_t)n * 4 + 255) & ~(size_t)255;
    const size_t fc_bytes = (size_t)MAX_DEPTH * 27 * T * sizeof(double);
    const size_t fm_bytes = ((size_t)MAX_DEPTH * T + 255) & ~(size_t)255;
    const size_t total = ctl_bytes + 2 * q_bytes + fc_bytes + fm_bytes;
    char* base = nullptr;
    if (cudaMallocAsync((void**)&base, total, stream) != cudaSuccess) {
        cudaGetLastError();
        return HEXVAL_ERR_ALLOC;
    }
    Ctl* ctl = reinterpret_cast<Ctl*>(base);
    uint32_t* qsub = reinterpret_cast<uint32_t*>(base + ctl_bytes);
    uint32_t* qex = reinterpret_cast<uint32_t*>(base + ctl_bytes + q_bytes);
    Frames fr;
    fr.coef = reinterpret_cast<double*>(base + ctl_bytes + 2 * q_bytes);
    fr.mask = reinterpret_cast<unsigned char*>(base + ctl_bytes + 2 * q_bytes + fc_bytes);
    fr.T = T;
    cudaMemsetAsync(ctl, 0, ctl_bytes, stream);

    const int slot = prof ? prof->count++ : -1;
    auto mark = [&](int ph, int which) {
        if (slot >= 0) cudaEventRecord(prof->ev[slot][ph][which], stream);
    };

    const unsigned p1_blocks = (unsigned)((n + P1_THREADS - 1) / P1_THREADS);
    mark(HEXVAL_PHASE_PASS1, 0);
    if (coeffs) {
        if (stats) pass1_kernel<L, true, true><<<p1_blocks, P1_THREADS, 0, stream>>>(ld, n, flags, coeffs, ctl, qsub, qex, stats);
        else pass1_kernel<L, true, false><<<p1_blocks, P1_THREADS, 0, stream>>>(ld, n, flags, coeffs, ctl, qsub, qex, stats);
    } else {
        if (stats) pass1_kernel<L, false, true><<<p1_blocks, P1_THREADS, 0, stream>>>(ld, n, flags, coeffs, ctl, qsub, qex, stats);
        else pass1_kernel<L, false, false><<<p1_blocks, P1_THREADS, 0, stream>>>(ld, n, flags, coeffs, ctl, qsub, qex, stats);
    }
    mark(HEXVAL_PHASE_PASS1, 1);
    mark(HEXVAL_PHASE_EXACT, 0);
    const unsigned k5_blocks = (unsigned)info.sms * 4;
    if (stats) exact_kernel<L, true><<<k5_blocks, K5_THREADS, 0, stream>>>(ld, flags, ctl, qex, qsub, stats);
    else exact_kernel<L, false><<<k5_blocks, K5_THREADS, 0, stream>>>(ld, flags, ctl, qex, qsub, stats);
    mark(HEXVAL_PHASE_EXACT, 1);
    mark(HEXVAL_PHASE_SUBDIV, 0);
    const unsigned k4_blocks = (unsigned)(info.sms * info.k4_blocks_per_sm);
    const CoordRoot<L> root{ld};
    if (stats) subdiv_kernel<CoordRoot<L>, true><<<k4_blocks, K4_THREADS, 0, stream>>>(root, flags, ctl, qsub, fr, stats);
    else subdiv_kernel<CoordRoot<L>, false><<<k4_blocks, K4_THREADS, 0, stream>>>(root, flags, ctl, qsub, fr, stats);
    mark(HEXVAL_PHASE_SUBDIV, 1);
    cudaFreeAsync(base, stream);
    if (cudaGetLastError() != cudaSuccess) return HEXVAL_ERR_CUDA;
    return HEXVAL_OK;
}

bool misaligned(const void* p, size_t a) { return p && (((uintptr_t)p) & (a - 1)) != 0; }

// Steps 4-5 on caller-supplied coefficients: Step 4 + enqueue, then K4.
template <bool STATS>
__global__ void __launch_bounds__(P1_THREADS) bezier_pass_kernel(const double* __restrict__ b, int64_t n,
                                                                 uint8_t* __restrict__ flags, Ctl* ctl,
                                                                 uint32_t* __restrict__ qsub, hexval_stats* stats) {
    __shared__ unsigned int s_sub[33];
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
    block_append<P1_THREADS / 32>(st == ST_SUB, (uint32_t)i, qsub, &ctl->n_sub, s_sub);
    if (STATS) {
        const int nv = __syncthreads_count(st == ST_VALID);
        const int nn = __syncthreads_count(st == ST_NONFINITE);
        if (threadIdx.x == 0) {
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
    const unsigned T = (unsigned)(info.sms * info.k4_blocks_per_sm * K4_THREADS);
    const size_t ctl_bytes = 256;
    const size_t q_bytes = ((size_t)n * 4 + 255) & ~(size_t)255;
    const size_t fc_bytes = (size_t)MAX_DEPTH * 27 * T * sizeof(double);
    const size_t fm_bytes = ((size_t)MAX_DEPTH * T + 255) & ~(size_t)255;
    char* base = nullptr;
    if (cudaMallocAsync((void**)&base, ctl_bytes + q_bytes + fc_bytes + fm_bytes, stream) != cudaSuccess) {
        cudaGetLastError();
        return HEXVAL_ERR_ALLOC;
    }
    Ctl* ctl = reinterpret_cast<Ctl*>(base);
    uint32_t* qsub = reinterpret_cast<uint32_t*>(base + ctl_bytes);
    Frames fr;
    fr.coef = reinterpret_cast<double*>(base + ctl_bytes + q_bytes);
    fr.mask = reinterpret_cast<unsigned char*>(base + ctl_bytes + q_bytes + fc_bytes);
    fr.T = T;
    cudaMemsetAsync(ctl, 0, ctl_bytes, stream);
    const unsigned p1_blocks = (unsigned)((n + P1_THREADS - 1) / P1_THREADS);
    if (stats) bezier_pass_kernel<true><<<p1_blocks, P1_THREADS, 0, stream>>>(b, n, flags, ctl, qsub, stats);
    else bezier_pass_kernel<false><<<p1_blocks, P1_THREADS, 0, stream>>>(b, n, flags, ctl, qsub, stats);
    const CoeffRoot root{b, n};
    const unsigned k4_blocks = (unsigned)(info.sms * info.k4_blocks_per_sm);
    if (stats) subdiv_kernel<CoeffRoot, true><<<k4_blocks, K4_THREADS, 0, stream>>>(root, flags, ctl, qsub, fr, stats);
    else subdiv_kernel<CoeffRoot, false><<<k4_blocks, K4_THREADS, 0, stream>>>(root, flags, ctl, qsub, fr, stats);
    cudaFreeAsync(base, stream);
    if (cudaGetLastError() != cudaSuccess) return HEXVAL_ERR_CUDA;
    return HEXVAL_OK;
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
        if (cudaMallocAsync((void**)&dc[k], (size_t)24 * C * sizeof(double), hp.s[k]) != cudaSuccess ||
            cudaMallocAsync((void**)&df[k], (size_t)C, hp.s[k]) != cudaSuccess ||
            (coeffs_host_opt && cudaMallocAsync((void**)&dk[k], (size_t)27 * C * sizeof(double), hp.s[k]) != cudaSuccess))
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
        if (cudaMallocAsync((void**)&dv, (size_t)3 * nv * sizeof(double) + 8, hp.s[0]) != cudaSuccess) rc = HEXVAL_ERR_ALLOC;
        else {
            cudaMemcpyAsync(dv, vertices_host, (size_t)3 * nv * sizeof(double), cudaMemcpyHostToDevice, hp.s[0]);
            cudaEventCreateWithFlags(&vready, cudaEventDisableTiming);
            cudaEventRecord(vready, hp.s[0]);
            cudaStreamWaitEvent(hp.s[1], vready, 0);
        }
    }
    for (int k = 0; k < 2 && rc == HEXVAL_OK; ++k) {
        if (cudaMallocAsync((void**)&di[k], (size_t)8 * C * sizeof(int32_t), hp.s[k]) != cudaSuccess ||
            cudaMallocAsync((void**)&df[k], (size_t)C, hp.s[k]) != cudaSuccess ||
            (coeffs_host_opt && cudaMallocAsync((void**)&dk[k], (size_t)27 * C * sizeof(double), hp.s[k]) != cudaSuccess))
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
        case HEXVAL_ERR_ARGUMENT: return "invalid argument (n < 0, n > INT32_MAX, or NULL buffer)";
        case HEXVAL_ERR_ALIGNMENT: return "misaligned pointer";
        case HEXVAL_ERR_CUDA: return "CUDA launch or copy error";
        case HEXVAL_ERR_ALLOC: return "scratch allocation failed";
        default: return "unknown status";
    }
}

int hexval_version(void) { return 100; }

int hexval_kernel_launches_per_call(void) { return 3; }

}  // extern "C"
