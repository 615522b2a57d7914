// Pipe-throughput microbenchmark (tooling, not product): per-SM issue rates of
// the instructions a pass-1 design could use on sm_100a: DFMA/DADD (FP64 pipe),
// FFMA / FFMA2 (FP32 pipe), F2F.F32.F64 (conversion), IMNMX (integer).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb tools/microbench_pipes.cu
#include <cuda_runtime.h>
#include <stdio.h>

constexpr int ITERS = 4096;
constexpr int ILP = 8;

__global__ void k_dfma(double* out, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = threadIdx.x + j;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int j = 0; j < ILP; ++j) x[j] = __fma_rn(x[j], a, b);
    double s = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(float* out, float a, float b) {
    float x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = threadIdx.x + j;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int j = 0; j < ILP; ++j) x[j] = __fmaf_rn(x[j], a, b);
    float s = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
    float2 x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = make_float2(threadIdx.x + j, j);
    const float2 A = make_float2(a, a), B = make_float2(b, b);
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int j = 0; j < ILP; ++j) x[j] = __ffma2_rn(x[j], A, B);
    float s = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += x[j].x + x[j].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_f2f(float* out, double a) {
    double x[ILP];
    float acc[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) { x[j] = a * (threadIdx.x + j); acc[j] = 0.f; }
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int j = 0; j < ILP; ++j) {
            const float f = __double2float_rn(x[j]);
            acc[j] = __int_as_float(__float_as_int(acc[j]) ^ __float_as_int(f));   // LOP3, keeps F2F live
            x[j] = __longlong_as_double(__double_as_longlong(x[j]) ^ (long long)i);
        }
    float s = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imnmx(int* out, int a) {
    int x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = threadIdx.x * (j + 1);
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int j = 0; j < ILP; ++j) x[j] = min(x[j] + a, x[(j + 1) % ILP]);
    int s = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F>
void run(const char* name, F launch, double ops_per_thread) {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256;
    launch(blocks, threads);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch(blocks, threads);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ops = 5.0 * blocks * threads * ops_per_thread;
    const double rate = ops / (ms * 1e-3);
    printf("%-8s %8.3f ms  %10.3f Gop/s  %7.2f ops/clk/SM at %d MHz (max clock)\n", name, ms, rate / 1e9,
           rate / sms / (clk * 1e3), clk / 1000);
}

int main() {
    double* dd;
    float* df;
    int* di;
    cudaMalloc(&dd, 1 << 24);
    cudaMalloc(&df, 1 << 24);
    cudaMalloc(&di, 1 << 24);
    const double per = (double)ITERS * ILP;
    run("DFMA", [&](int b, int t) { k_dfma<<<b, t>>>(dd, 0.999, 1e-3); }, per);
    run("FFMA", [&](int b, int t) { k_ffma<<<b, t>>>(df, 0.999f, 1e-3f); }, per);
    run("FFMA2x", [&](int b, int t) { k_ffma2<<<b, t>>>(df, 0.999f, 1e-3f); }, 2 * per);
    run("F2F.64>32", [&](int b, int t) { k_f2f<<<b, t>>>(df, 1.0001); }, per);
    run("IMNMX+IADD", [&](int b, int t) { k_imnmx<<<b, t>>>(di, 3); }, 2 * per);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
