// RESEARCH RECORD, not part of the product library: bitsliced AES-MMO expand
// (prg.expand, prg.py:43-60) -- the measured alternative to the T-table
// expand_kernel (7x slower on B200, 255 registers).
// Built on demand into scripts/_variants/libfss_bitsliced.so by
// scripts/research/bitsliced/build.py for tests/test_gpu_fss.py and
// scripts/aes_variants.py. One thread owns 32 consecutive
// seeds; for each output block it transposes them into 128 bit-slices,
// runs the fixed-key bitsliced AES (aes_bitsliced.cuh), transposes back and
// applies the MMO feed-forward. Pure ALU work (LOP3 / SHF): no tables.
#include <cuda_runtime.h>
#include <stdint.h>

#include "aes_bitsliced.cuh"

// status codes of include/ariann_fss.h (this library is standalone)
#define BS_OK 0
#define BS_EINVAL 1
#define BS_ECUDA 2

namespace {

constexpr int kBsThreads = 128;

template <int KEY>
__device__ __forceinline__ void mmo_group(const uint4* __restrict__ in, uint8_t* __restrict__ out,
                                          int blocks) {
    uint32_t x[128];
#pragma unroll
    for (int j = 0; j < 32; j++) {
        const uint4 v = __ldg(in + j);
        x[j] = v.x;
        x[32 + j] = v.y;
        x[64 + j] = v.z;
        x[96 + j] = v.w;
    }
#pragma unroll
    for (int c = 0; c < 4; c++) fssb::bs::transpose32(x + 32 * c);
    fssb::bs::encrypt<KEY>(x);
#pragma unroll
    for (int c = 0; c < 4; c++) fssb::bs::transpose32(x + 32 * c);
#pragma unroll
    for (int j = 0; j < 32; j++) {
        const uint4 v = __ldg(in + j);
        *reinterpret_cast<uint4*>(out + (size_t)j * 16 * blocks + 16 * KEY) =
            make_uint4(x[j] ^ v.x, x[32 + j] ^ v.y, x[64 + j] ^ v.z, x[96 + j] ^ v.w);
    }
}

__global__ void __launch_bounds__(kBsThreads)
bs_expand_kernel(const uint8_t* __restrict__ seeds, uint64_t groups, int blocks,
                 uint8_t* __restrict__ out) {
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint4* in = reinterpret_cast<const uint4*>(seeds + g * 512);
        uint8_t* o = out + g * 512 * blocks;
        mmo_group<0>(in, o, blocks);
        mmo_group<1>(in, o, blocks);
        if (blocks == 3) mmo_group<2>(in, o, blocks);
    }
}

}  // namespace

extern "C" int fss_aes_mmo_expand_bitsliced(const uint8_t* seeds, uint64_t count, int out_blocks,
                                            uint8_t* out, void* stream) {
    if (out_blocks < 2 || out_blocks > 3) return BS_EINVAL;
    if (count % 32) return BS_EINVAL;   // 32 seeds per thread
    if (count == 0) return BS_OK;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t groups = count / 32;
    uint64_t grid = (groups + kBsThreads - 1) / kBsThreads;
    const uint64_t cap = (uint64_t)sms * 8;
    if (grid > cap) grid = cap;
    bs_expand_kernel<<<(unsigned)grid, kBsThreads, 0, (cudaStream_t)stream>>>(seeds, groups, out_blocks,
                                                                               out);
    const cudaError_t err = cudaGetLastError();
    return err == cudaSuccess ? BS_OK : BS_ECUDA;
}
