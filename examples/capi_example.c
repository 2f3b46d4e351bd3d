/*
 * capi_example.c -- the C ABI (include/ariann_fss.h) used from plain C, with
 * no Python and no torch: draw a DCF tape from a PCG64 state on the device,
 * generate 2^20 comparison keys (n = 32), evaluate both parties on x = alpha +
 * y for small signed y, and check that the shares reconstruct to 1[x <= alpha]
 * for every element. Build and run (needs a GPU):
 *
 *   gcc -O2 -std=c11 examples/capi_example.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2006_04593_b200 -lariann_fss -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2006_04593_b200 -o capi_example && ./capi_example
 *
 * This is what a non-Python host (the cgo / JNI / N-API binding of
 * INTEGRATION.md) drives: device pointers, counts, n, a stream, int status.
 */
#include <cuda_runtime_api.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "ariann_fss.h"

#define CHECK_FSS(call)                                                          \
    do {                                                                         \
        int rc_ = (call);                                                        \
        if (rc_ != FSS_OK) {                                                     \
            fprintf(stderr, "%s -> %d: %s\n", #call, rc_, fss_last_error());     \
            return 1;                                                            \
        }                                                                        \
    } while (0)
#define CHECK_CUDA(call)                                                         \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) {                                                 \
            fprintf(stderr, "%s -> %s\n", #call, cudaGetErrorString(e_));        \
            return 1;                                                            \
        }                                                                        \
    } while (0)

int main(void) {
    const int n = 32;
    const uint64_t N = 1u << 20;
    void* stream = NULL; /* legacy default stream */
    if (fss_abi_version() != FSS_ABI_VERSION) {
        fprintf(stderr, "library ABI %d, header %d\n", fss_abi_version(), FSS_ABI_VERSION);
        return 1;
    }
    /* any PCG64 state (numpy's Generator(PCG64(seed)).bit_generator.state) */
    fss_pcg64_state st = {0x0123456789abcdefULL, 0x0fedcba987654321ULL, 0x5851f42d4c957f2dULL | 1,
                          0x14057b7ef767814fULL, 0, 0, 0};
    fss_pcg64_state st_out;

    uint64_t *alpha, *alpha0, *alpha1, *sigma_cw, *leaf_cw, *x, *y0, *y1;
    uint8_t *s0, *s1, *scw, *tcw;
    CHECK_CUDA(cudaMalloc((void**)&alpha, N * 8));
    CHECK_CUDA(cudaMalloc((void**)&alpha0, N * 8));
    CHECK_CUDA(cudaMalloc((void**)&alpha1, N * 8));
    CHECK_CUDA(cudaMalloc((void**)&s0, N * 16));
    CHECK_CUDA(cudaMalloc((void**)&s1, N * 16));
    CHECK_CUDA(cudaMalloc((void**)&scw, (uint64_t)n * N * 16));
    CHECK_CUDA(cudaMalloc((void**)&tcw, (uint64_t)n * N));
    CHECK_CUDA(cudaMalloc((void**)&sigma_cw, (uint64_t)n * N * 8));
    CHECK_CUDA(cudaMalloc((void**)&leaf_cw, (uint64_t)(n + 1) * N * 8));
    CHECK_CUDA(cudaMalloc((void**)&x, N * 8));
    CHECK_CUDA(cudaMalloc((void**)&y0, N * 8));
    CHECK_CUDA(cudaMalloc((void**)&y1, N * 8));

    /* dealer: tape (alpha, alpha0, s0, s1) -> keys (CWs shared by both parties) */
    CHECK_FSS(fss_pcg64_tape(&st, n, N, 1, alpha, alpha0, s0, s1, &st_out, stream));
    CHECK_FSS(fss_dcf_keygen(n, n, N, alpha, alpha0, s0, s1, scw, tcw, sigma_cw, leaf_cw, alpha1, stream));

    /* public inputs x = alpha + y, y in [-1000, 1000) */
    uint64_t* a_host = (uint64_t*)malloc(N * 8);
    uint64_t* x_host = (uint64_t*)malloc(N * 8);
    uint64_t* r0 = (uint64_t*)malloc(N * 8);
    uint64_t* r1 = (uint64_t*)malloc(N * 8);
    CHECK_CUDA(cudaMemcpy(a_host, alpha, N * 8, cudaMemcpyDeviceToHost));
    uint64_t lcg = 12345;
    for (uint64_t e = 0; e < N; e++) {
        lcg = lcg * 6364136223846793005ULL + 1442695040888963407ULL;
        const int64_t yv = (int64_t)((lcg >> 33) % 2000) - 1000;
        x_host[e] = (a_host[e] + (uint64_t)yv) & 0xFFFFFFFFULL;
    }
    CHECK_CUDA(cudaMemcpy(x, x_host, N * 8, cudaMemcpyHostToDevice));

    /* the two parties: party 0 holds seed s0, party 1 seed s1 (ld = N) */
    CHECK_FSS(fss_dcf_eval(0, n, n, N, N, s0, scw, tcw, sigma_cw, leaf_cw, x, y0, NULL, stream));
    CHECK_FSS(fss_dcf_eval(1, n, n, N, N, s1, scw, tcw, sigma_cw, leaf_cw, x, y1, NULL, stream));
    CHECK_CUDA(cudaMemcpy(r0, y0, N * 8, cudaMemcpyDeviceToHost));
    CHECK_CUDA(cudaMemcpy(r1, y1, N * 8, cudaMemcpyDeviceToHost));

    uint64_t bad = 0;
    for (uint64_t e = 0; e < N; e++) {
        const uint64_t rec = (r0[e] + r1[e]) & 0xFFFFFFFFULL;
        const uint64_t want = x_host[e] <= a_host[e] ? 1 : 0;
        bad += rec != want;
    }
    printf("capi_example: %llu DCF comparisons (n=%d), %llu mismatches, rng advanced by %llu outputs\n",
           (unsigned long long)N, n, (unsigned long long)bad, (unsigned long long)st_out.advance);
    free(a_host);
    free(x_host);
    free(r0);
    free(r1);
    return bad != 0;
}
