// Experiment: can a second lookup path add table-lookup bandwidth next to
// conflict-free shared memory (the bound of the T-table AES)?
//   lds  : 8 lookup chains per thread into a lane-replicated shared table
//   ldg  : 8 chains into a lane-replicated GLOBAL table (L1-resident, LDG.CONSTANT)
//   tex  : 8 chains via tex1Dfetch on a texture object (texture path)
//   mix1 : 7 LDS chains + 1 LDG chain;  mix2 : 7 LDS + 1 TEX
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lookup_probe lookup_paths_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int kThreads = 512;
constexpr int kWords = 256 * 64;   // 64 KiB: two interleaved lane-replicated tables

template <int NLDS, int NLDG, int NTEX>
__global__ void __launch_bounds__(kThreads, 1)
probe(int iters, const uint32_t* __restrict__ gtab, cudaTextureObject_t tex, uint32_t* sink) {
    extern __shared__ uint32_t tab[];
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) tab[i] = gtab[i];
    __syncthreads();
    const uint32_t lo = (threadIdx.x & 31) * 4;
    const unsigned char* base = reinterpret_cast<const unsigned char*>(tab);
    const unsigned char* gbase = reinterpret_cast<const unsigned char*>(gtab);
    uint32_t v[NLDS + NLDG + NTEX];
#pragma unroll
    for (int j = 0; j < NLDS + NLDG + NTEX; j++) v[j] = threadIdx.x * 2654435761u + j;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int j = 0; j < NLDS; j++) {
            const uint32_t addr = __byte_perm(v[j], lo, 0x5514);
            v[j] = *reinterpret_cast<const uint32_t*>(base + addr);
        }
#pragma unroll
        for (int j = NLDS; j < NLDS + NLDG; j++) {
            const uint32_t addr = __byte_perm(v[j], lo, 0x5514);
            v[j] = __ldg(reinterpret_cast<const uint32_t*>(gbase + addr));
        }
#pragma unroll
        for (int j = NLDS + NLDG; j < NLDS + NLDG + NTEX; j++) {
            const uint32_t idx = __byte_perm(v[j], lo, 0x5514) >> 2;
            v[j] = tex1Dfetch<uint32_t>(tex, (int)idx);
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < NLDS + NLDG + NTEX; j++) acc ^= v[j];
    if (acc == 0x12345678u) sink[blockIdx.x] = acc;
}

template <int A, int B, int C>
void run(const char* name, int sms, const uint32_t* g, cudaTextureObject_t tex, uint32_t* sink) {
    const int iters = 40000;
    cudaFuncSetAttribute(probe<A, B, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        probe<A, B, C><<<sms, kThreads, kWords * 4>>>(iters, g, tex, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double lookups = (double)sms * kThreads * iters * (A + B + C);
    printf("{\"probe\": \"%s\", \"lds\": %d, \"ldg\": %d, \"tex\": %d, \"ms\": %.3f, "
           "\"lookups_per_s\": %.4g, \"lookups_per_clk_sm_at_1.965GHz\": %.2f}\n",
           name, A, B, C, best, lookups / (best * 1e-3),
           lookups / (best * 1e-3) / sms / 1.965e9);
    if (cudaGetLastError() != cudaSuccess) printf("error\n");
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *g, *sink;
    cudaMalloc(&g, kWords * 4);
    cudaMalloc(&sink, 4096 * 4);
    uint32_t h[kWords];
    for (int i = 0; i < kWords; i++) h[i] = (uint32_t)(i * 2246822519u + 0x9E3779B9u);
    cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = g;
    rd.res.linear.desc = cudaCreateChannelDesc<uint32_t>();
    rd.res.linear.sizeInBytes = kWords * 4;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex;
    cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    run<8, 0, 0>("lds", sms, g, tex, sink);
    run<0, 8, 0>("ldg", sms, g, tex, sink);
    run<0, 0, 8>("tex", sms, g, tex, sink);
    run<7, 1, 0>("mix_lds_ldg", sms, g, tex, sink);
    run<7, 0, 1>("mix_lds_tex", sms, g, tex, sink);
    run<6, 0, 2>("mix_lds_tex2", sms, g, tex, sink);
    run<8, 0, 1>("mix_lds8_tex1", sms, g, tex, sink);
    return 0;
}
