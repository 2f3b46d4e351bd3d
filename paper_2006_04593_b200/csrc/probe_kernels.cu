// On-box peak probes for the roofline denominators of the AES work
// (diagnostics, not part of the reference surface):
//   * shared-memory lookup rate -- the exact access pattern of aes_ttable.cuh
//     (lane-replicated table, address built by one PRMT, LDS.32), 8 independent
//     lookup chains per thread, one 512-thread CTA per SM;
//   * LOP3 lane-op rate -- 8 independent lop3.b32 chains per thread (the unit
//     of the bitsliced-AES estimate in SURVEY.md §8d);
//   * the SM clock seen by the probe (clock64 cycles / %globaltimer ns).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ariann_fss.h"
#include "common.cuh"

namespace {

constexpr int kProbeThreads = 512;
constexpr int kTabWords = 256 * 64;  // two interleaved lane-replicated tables (64 KiB)

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(kProbeThreads, 1)
lds_probe_kernel(int iters, uint32_t seed, uint32_t* sink, unsigned long long* cycles,
                 unsigned long long* ns) {
    extern __shared__ uint32_t tab[];
    for (int i = threadIdx.x; i < kTabWords; i += blockDim.x) tab[i] = (uint32_t)(i * 2654435761u);
    __syncthreads();
    const uint32_t lo = (threadIdx.x & 31) * 4;
    const unsigned char* base = reinterpret_cast<const unsigned char*>(tab);
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; j++) v[j] = seed * (threadIdx.x + 1) + j * 0x9E3779B9u;
    const long long c0 = clock64();
    const uint64_t t0 = gtimer();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            // table index = byte 1 of v; address = PRMT(v, lo): byte1 -> byte1, lo -> byte0
            const uint32_t addr = __byte_perm(v[j], lo, 0x5514);
            v[j] = *reinterpret_cast<const uint32_t*>(base + addr);
        }
    }
    const long long c1 = clock64();
    const uint64_t t1 = gtimer();
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) acc ^= v[j];
    if (acc == 0x12345678u) sink[blockIdx.x] = acc;
    if (threadIdx.x == 0) {
        atomicMax(cycles, (unsigned long long)(c1 - c0));
        atomicMax(ns, (unsigned long long)(t1 - t0));
    }
}

__global__ void __launch_bounds__(kProbeThreads, 2)
lop3_probe_kernel(int iters, uint32_t seed, uint32_t* sink) {
    uint32_t v[8];
    const uint32_t y = seed ^ threadIdx.x, z = seed * 3u + blockIdx.x;
#pragma unroll
    for (int j = 0; j < 8; j++) v[j] = seed + j * 0x01000193u + threadIdx.x;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[j]) : "r"(y), "r"(z));
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) acc ^= v[j];
    if (acc == 0x12345678u) sink[blockIdx.x] = acc;
}

}  // namespace

extern "C" int fss_probe_peaks(fss_peaks* out) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t* sink = nullptr;
    unsigned long long* meta = nullptr;
    cudaEvent_t e0, e1;
    if (cudaMalloc(&sink, 4096 * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&meta, 2 * sizeof(unsigned long long)) != cudaSuccess)
        return fssb::set_error(FSS_ECUDA, "probe allocation failed");
    cudaFuncSetAttribute(lds_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTabWords * 4);
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int lds_iters = 80000, lop_iters = 100000;
    float ms_lds = 0.f, ms_lop = 0.f;
    unsigned long long host_meta[2] = {0, 0};
    for (int rep = 0; rep < 3; rep++) {  // first rep warms clocks up; keep the best
        cudaMemset(meta, 0, 2 * sizeof(unsigned long long));
        cudaEventRecord(e0);
        lds_probe_kernel<<<sms, kProbeThreads, kTabWords * 4>>>(lds_iters, 7u + rep, sink, meta, meta + 1);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float t = 0.f;
        cudaEventElapsedTime(&t, e0, e1);
        if (rep == 0 || t < ms_lds) {
            ms_lds = t;
            cudaMemcpy(host_meta, meta, sizeof(host_meta), cudaMemcpyDeviceToHost);
        }
        cudaEventRecord(e0);
        lop3_probe_kernel<<<2 * sms, kProbeThreads>>>(lop_iters, 11u + rep, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&t, e0, e1);
        if (rep == 0 || t < ms_lop) ms_lop = t;
    }
    cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    cudaFree(meta);
    if (err != cudaSuccess) return fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
    const double warps = (double)sms * (kProbeThreads / 32);
    out->lds_wavefronts_per_s = warps * lds_iters * 8 / (ms_lds * 1e-3);
    out->lop3_lane_ops_per_s = 2.0 * sms * kProbeThreads * (double)lop_iters * 8 / (ms_lop * 1e-3);
    out->sm_clock_hz = host_meta[1] ? (double)host_meta[0] / ((double)host_meta[1] * 1e-9) : 0.0;
    out->sms = sms;
    return FSS_OK;
}
