// ARNK key-container payloads (reference LAYOUT.md:48-71, fss.py:498-602) on
// device: level-major SoA keys <-> element-major per-party byte payloads.
//
// Element layout (w = ceil(n/8) little-endian bytes per ring value):
//   eq : alpha_share[w] | seed0[16] | n x (scw[16] | flags[1])           | cw_final[w]
//   cmp: alpha_share[w] | seed0[16] | n x (scw[16] | flags[1] | sigma[w]) | (n+1) x leaf[w]
// Grid: x over elements, y over "slots" (slot i < n = level i's record,
// slot n = head + eq tail, slot n+1 = cmp leaf block). Each thread moves one
// slot of one element.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/ariann_fss.h"
#include "common.cuh"

namespace {

__device__ __forceinline__ void put_le(uint8_t* p, uint64_t v, int w) {
    for (int b = 0; b < w; b++) p[b] = (uint8_t)(v >> (8 * b));
}

__device__ __forceinline__ uint64_t get_le(const uint8_t* p, int w) {
    uint64_t v = 0;
    for (int b = 0; b < w; b++) v |= (uint64_t)p[b] << (8 * b);
    return v;
}

__host__ __device__ __forceinline__ uint64_t elem_bytes(int kind, int n) {
    const int w = (n + 7) / 8;
    return kind == 0 ? (uint64_t)(w + 16 + 17 * n + w) : (uint64_t)(w + 16 + n * (17 + w) + (n + 1) * w);
}

struct Keys {
    uint64_t* alpha_share;
    uint8_t* seed0;
    uint8_t* scw;
    uint8_t* tcw;
    uint64_t* cw_final;  // eq
    uint64_t* sigma_cw;  // cmp
    uint64_t* leaf_cw;   // cmp
};

template <bool PACK>
__global__ void arnk_kernel(int kind, int n, uint64_t count, uint64_t ld, Keys k, uint8_t* buf) {
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (e >= count) return;
    const int slot = blockIdx.y;
    const int w = (n + 7) / 8;
    const int rec = kind == 0 ? 17 : 17 + w;
    uint8_t* p = buf + e * elem_bytes(kind, n);
    if (slot < n) {
        const uint64_t off = (uint64_t)slot * ld + e;
        uint8_t* q = p + w + 16 + (uint64_t)slot * rec;
        if (PACK) {
            const uint4 v = *reinterpret_cast<const uint4*>(k.scw + 16 * off);
            const uint32_t words[4] = {v.x, v.y, v.z, v.w};
            for (int b = 0; b < 16; b++) q[b] = (uint8_t)(words[b >> 2] >> (8 * (b & 3)));
            q[16] = k.tcw[off];
            if (kind == 1) put_le(q + 17, k.sigma_cw[off], w);
        } else {
            uint32_t words[4] = {0, 0, 0, 0};
            for (int b = 0; b < 16; b++) words[b >> 2] |= (uint32_t)q[b] << (8 * (b & 3));
            *reinterpret_cast<uint4*>(k.scw + 16 * off) = make_uint4(words[0], words[1], words[2], words[3]);
            k.tcw[off] = q[16];
            if (kind == 1) k.sigma_cw[off] = get_le(q + 17, w);
        }
    } else if (slot == n) {
        uint8_t* tail = p + w + 16 + (uint64_t)n * rec;
        if (PACK) {
            put_le(p, k.alpha_share[e], w);
            for (int b = 0; b < 16; b++) p[w + b] = k.seed0[16 * e + b];
            if (kind == 0) put_le(tail, k.cw_final[e], w);
        } else {
            k.alpha_share[e] = get_le(p, w);
            for (int b = 0; b < 16; b++) k.seed0[16 * e + b] = p[w + b];
            if (kind == 0) k.cw_final[e] = get_le(tail, w);
        }
    } else {  // cmp leaf block
        uint8_t* tail = p + w + 16 + (uint64_t)n * rec;
        for (int i = 0; i <= n; i++) {
            const uint64_t off = (uint64_t)i * ld + e;
            if (PACK)
                put_le(tail + (uint64_t)i * w, k.leaf_cw[off], w);
            else
                k.leaf_cw[off] = get_le(tail + (uint64_t)i * w, w);
        }
    }
}

int launch(bool pack, int kind, int n, uint64_t count, uint64_t ld, Keys k, uint8_t* buf, void* stream) {
    if ((kind != 0 && kind != 1) || n < 1 || n > 64 || (kind == 1 && n > 63))
        return fssb::set_error(FSS_EINVAL, "ARNK: bad kind or n");
    if (count == 0) return FSS_OK;
    const int bs = 256;
    dim3 grid((unsigned)((count + bs - 1) / bs), kind == 0 ? n + 1 : n + 2);
    if (pack)
        arnk_kernel<true><<<grid, bs, 0, (cudaStream_t)stream>>>(kind, n, count, ld, k, buf);
    else
        arnk_kernel<false><<<grid, bs, 0, (cudaStream_t)stream>>>(kind, n, count, ld, k, buf);
    const cudaError_t err = cudaGetLastError();
    return err == cudaSuccess ? FSS_OK : fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
}

}  // namespace

extern "C" {

uint64_t fss_arnk_elem_bytes(int kind, int n) { return elem_bytes(kind, n); }

int fss_arnk_pack(int kind, int n, uint64_t count, uint64_t ld, const uint64_t* alpha_share,
                  const uint8_t* seed0, const uint8_t* scw, const uint8_t* tcw,
                  const uint64_t* cw_final, const uint64_t* sigma_cw, const uint64_t* leaf_cw,
                  uint8_t* payload, void* stream) {
    Keys k{const_cast<uint64_t*>(alpha_share), const_cast<uint8_t*>(seed0), const_cast<uint8_t*>(scw),
           const_cast<uint8_t*>(tcw), const_cast<uint64_t*>(cw_final), const_cast<uint64_t*>(sigma_cw),
           const_cast<uint64_t*>(leaf_cw)};
    return launch(true, kind, n, count, ld, k, payload, stream);
}

int fss_arnk_unpack(int kind, int n, uint64_t count, const uint8_t* payload, uint64_t* alpha_share,
                    uint8_t* seed0, uint8_t* scw, uint8_t* tcw, uint64_t* cw_final,
                    uint64_t* sigma_cw, uint64_t* leaf_cw, void* stream) {
    Keys k{alpha_share, seed0, scw, tcw, cw_final, sigma_cw, leaf_cw};
    return launch(false, kind, n, count, count, k, const_cast<uint8_t*>(payload), stream);
}

}  // extern "C"
