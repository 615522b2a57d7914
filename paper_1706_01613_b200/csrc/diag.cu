// diag.cu -- roofline denominators measured on the device the library runs on
// (not part of the hot path).  hexval_diag_fp64_peak times a DFMA-only kernel:
// every thread runs 8 independent __fma_rn chains, grid = 8 blocks of 256
// threads per SM, best of 5 launches between CUDA events.  The result is the
// FP64 pipe's throughput in DFMA lane-instructions per second, the unit in
// which the subdivision kernel's algorithmic work (294 FP64
// operations per node) and pass 1's (381 per hex) are counted.
#include <cuda_runtime.h>
#include <stdint.h>

#include "hexval.h"

namespace {

constexpr int DIAG_ILP = 8;

__global__ void __launch_bounds__(256) dfma_probe_kernel(double* out, double a, double b, int iters) {
    double x[DIAG_ILP];
#pragma unroll
    for (int j = 0; j < DIAG_ILP; ++j) x[j] = threadIdx.x + j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < DIAG_ILP; ++j) x[j] = __fma_rn(x[j], a, b);
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < DIAG_ILP; ++j) s = __dadd_rn(s, x[j]);
    if (s == 0.123456789) out[0] = s;                      // keeps the chains live, never true
}

}  // namespace

extern "C" int hexval_diag_fp64_peak(int iters, double* dfma_per_s_out, float* best_ms_out, cudaStream_t stream) {
    if (iters <= 0 || !dfma_per_s_out) return HEXVAL_ERR_ARGUMENT;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return HEXVAL_ERR_CUDA;
    double* out = nullptr;
    if (cudaMallocAsync((void**)&out, sizeof(double), stream) != cudaSuccess) return HEXVAL_ERR_ALLOC;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256;
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {                          // first launch warms up
        cudaEventRecord(e0, stream);
        dfma_probe_kernel<<<blocks, threads, 0, stream>>>(out, 0.999, 1e-3, iters);
        cudaEventRecord(e1, stream);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    cudaFreeAsync(out, stream);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (cudaStreamSynchronize(stream) != cudaSuccess || cudaGetLastError() != cudaSuccess) return HEXVAL_ERR_CUDA;
    *dfma_per_s_out = (double)blocks * threads * iters * DIAG_ILP / (best * 1e-3);
    if (best_ms_out) *best_ms_out = best;
    return HEXVAL_OK;
}
