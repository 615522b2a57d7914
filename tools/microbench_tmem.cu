// TMEM as a per-thread scratchpad (tooling, not product): can K4 park part of a
// node's split (the 45-value xi split G1) in tensor memory to free registers?
// Measures, per SM, the throughput of tcgen05.st / tcgen05.ld in the 32x32b
// shape (thread t <-> TMEM lane 32*(warp%4)+t) at 4..16 warps per SM, and the
// round-trip latency of one ld + wait::ld.  Verifies the data read back.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mbt tools/microbench_tmem.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

#define LD16(r, a)                                                                                           \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),  \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) \
                 : "r"(a))
#define ST16(a, r)                                                                                           \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
                 ::"r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), \
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory")
#define WAIT_LD() asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory")
#define WAIT_ST() asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory")

template <int COLS>
__device__ uint32_t tmem_alloc() {
    __shared__ uint32_t base;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&base)), "n"(COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    return base;
}
template <int COLS>
__device__ void tmem_free(uint32_t base) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(COLS));
}

// MODE 0: st 64 cols + ld 64 cols per iteration (round trip, 512 B/thread moved)
// MODE 1: ld 64 cols per iteration (4 x16 loads, one wait)
// MODE 2: ld 16 cols + wait per iteration (latency bound)
template <int COLS, int MODE>
__global__ void __launch_bounds__(128) k_tmem(int iters, unsigned* out, long long* cyc) {
    const uint32_t base = tmem_alloc<COLS>();
    const uint32_t lane_base = (uint32_t)((threadIdx.x / 32) * 32) << 16;
    const uint32_t t = base + lane_base;
    uint32_t r[4][16];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int j = 0; j < 16; ++j) r[q][j] = threadIdx.x * 1000 + q * 16 + j;
#pragma unroll
    for (int q = 0; q < 4; ++q) ST16(t + 16 * q, r[q]);
    WAIT_ST();
    unsigned acc = 0;
    __syncwarp();
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) ST16(t + 16 * q, r[q]);
            WAIT_ST();
        }
        if (MODE <= 1) {
#pragma unroll
            for (int q = 0; q < 4; ++q) LD16(r[q], t + 16 * q);
            WAIT_LD();
#pragma unroll
            for (int q = 0; q < 4; ++q) acc ^= r[q][i & 15];
        } else {
            LD16(r[0], t + 16 * (i & 3));
            WAIT_LD();
            acc += r[0][0];
        }
    }
    const long long c1 = clock64();
    unsigned bad = 0;
    if (MODE <= 1) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int j = 0; j < 16; ++j) bad |= r[q][j] != (unsigned)(threadIdx.x * 1000 + q * 16 + j);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ (bad << 31);
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    if (bad) printf("TMEM readback mismatch block %d thread %d\n", blockIdx.x, threadIdx.x);
    tmem_free<COLS>(base);
}

template <int COLS, int MODE>
void run(int ctas_per_sm, int sms, double clk_ghz) {
    const int blocks = ctas_per_sm * sms, iters = 4096;
    unsigned* out;
    long long* cyc;
    cudaMalloc(&out, blocks * 128 * sizeof(unsigned));
    cudaMalloc(&cyc, blocks * sizeof(long long));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_tmem<COLS, MODE><<<blocks, 128>>>(16, out, cyc);
    cudaEventRecord(e0);
    k_tmem<COLS, MODE><<<blocks, 128>>>(iters, out, cyc);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long hc[4096];
    cudaMemcpy(hc, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    double mc = 0;
    for (int b = 0; b < blocks; ++b) mc += hc[b];
    mc /= blocks;
    const double bytes_per_iter_thread = MODE == 0 ? 512.0 : (MODE == 1 ? 256.0 : 64.0);
    const double total = bytes_per_iter_thread * iters * 128.0 * blocks;
    printf("mode %d (%s) cols %d ctas/SM %d warps/SM %2d: %.3f ms, %.1f B/clk/SM (event), %.1f B/clk/SM (clock64), "
           "%.1f cycles/iter/warp  [%s]\n",
           MODE, MODE == 0 ? "st64+ld64" : (MODE == 1 ? "ld64     " : "ld16+wait"), COLS, ctas_per_sm, 4 * ctas_per_sm,
           ms, total / (ms * 1e-3) / sms / (clk_ghz * 1e9), bytes_per_iter_thread * iters * 128.0 * ctas_per_sm / mc,
           mc / iters, cudaGetErrorString(err));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double ghz = clk_khz * 1e-6;
    printf("%s, %d SMs, %.3f GHz\n", p.name, p.multiProcessorCount, ghz);
    const int sms = p.multiProcessorCount;
    run<128, 0>(1, sms, ghz); run<128, 0>(2, sms, ghz); run<128, 0>(4, sms, ghz);
    run<128, 1>(1, sms, ghz); run<128, 1>(2, sms, ghz); run<128, 1>(4, sms, ghz);
    run<128, 2>(1, sms, ghz); run<128, 2>(4, sms, ghz);
    return 0;
}
