/*
 * check_hexes.c -- the C ABI from plain C (no Python, no torch): validate a few
 * hexahedra given as 8 points each through the host-buffer
 * entry point, then the same batch from device memory.
 *
 *   gcc -std=c99 -Wall -I include -I /usr/local/cuda/include examples/check_hexes.c \
 *       -L paper_1706_01613_b200 -lhexval -Wl,-rpath,$PWD/paper_1706_01613_b200 \
 *       -L /usr/local/cuda/lib64 -lcudart -o check_hexes
 *   ./check_hexes            (needs a CUDA device)
 *
 * Prints one line per hex: its verdict and whether it was subdivided.
 */
#include <stdio.h>
#include <string.h>
#include <cuda_runtime_api.h>
#include "hexval.h"

enum { N = 4 };

/* unit cube in the paper's node order (Fig. 3): bottom face counter-clockwise, then top */
static const double CUBE[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                  {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

static void put_hex(double* soa, int i, double X[8][3]) {
    for (int k = 0; k < 8; ++k)
        for (int a = 0; a < 3; ++a) soa[(3 * k + a) * N + i] = X[k][a];   /* plane 3*node + axis */
}

static const char* verdict(uint8_t f) {
    static const char* names[4] = {"INVALID", "VALID", "UNDETERMINED", "NONFINITE"};
    return names[f & 3];
}

int main(void) {
    double soa[24 * N];
    double X[8][3];
    /* 0: unit cube (VALID) */
    memcpy(X, CUBE, sizeof X);
    put_hex(soa, 0, X);
    /* 1: node 7 pushed through the opposite face (INVALID at a corner) */
    memcpy(X, CUBE, sizeof X);
    X[6][0] = -0.5; X[6][1] = -0.5; X[6][2] = -0.5;
    put_hex(soa, 1, X);
    /* 2: mirrored cube (negative orientation: INVALID) */
    memcpy(X, CUBE, sizeof X);
    for (int k = 0; k < 8; ++k) X[k][0] = -X[k][0];
    put_hex(soa, 2, X);
    /* 3: a NaN coordinate (NONFINITE) */
    memcpy(X, CUBE, sizeof X);
    X[3][1] = 0.0 / 0.0;
    put_hex(soa, 3, X);

    uint8_t flags[N];
    int rc = hexval_check_soa_host(soa, N, flags, NULL, 0, 0);
    if (rc != HEXVAL_OK) {
        fprintf(stderr, "hexval_check_soa_host: %s\n", hexval_status_string(rc));
        return 1;
    }
    for (int i = 0; i < N; ++i) printf("host   hex %d: %s%s\n", i, verdict(flags[i]),
                                       (flags[i] & HEXVAL_FLAG_SUBDIVIDED) ? " (subdivided)" : "");

    /* the same batch from device memory on a stream */
    double* d_soa = NULL;
    uint8_t* d_flags = NULL;
    cudaStream_t s;
    if (cudaStreamCreate(&s) != cudaSuccess || cudaMalloc((void**)&d_soa, sizeof soa) != cudaSuccess ||
        cudaMalloc((void**)&d_flags, N) != cudaSuccess) {
        fprintf(stderr, "CUDA setup failed\n");
        return 1;
    }
    cudaMemcpyAsync(d_soa, soa, sizeof soa, cudaMemcpyHostToDevice, s);
    rc = hexval_check_soa(d_soa, N, d_flags, NULL, s);
    if (rc != HEXVAL_OK) {
        fprintf(stderr, "hexval_check_soa: %s\n", hexval_status_string(rc));
        return 1;
    }
    uint8_t dflags[N];
    cudaMemcpyAsync(dflags, d_flags, N, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    for (int i = 0; i < N; ++i) printf("device hex %d: %s\n", i, verdict(dflags[i]));
    cudaFree(d_soa);
    cudaFree(d_flags);
    cudaStreamDestroy(s);
    return memcmp(flags, dflags, N) != 0;
}
