// Elementwise Z_2^n ring arithmetic for the share layer (reference ring.py:99-129,
// sharing.py:214-230 mask_and_reveal, beaver.py:257-294 Beaver combine).
// u64 words, wraparound mod 2^64 then mask (ring.py:107-114). Vectorised:
// each thread handles two u64 (one 16-byte load per operand).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ariann_fss.h"
#include "common.cuh"

namespace {

__device__ __forceinline__ uint64_t apply(int op, uint64_t a, uint64_t b) {
    switch (op) {
        case FSS_RING_ADD: return a + b;
        case FSS_RING_SUB: return a - b;
        case FSS_RING_MUL: return a * b;
        case FSS_RING_NEG: return 0 - a;
        default: return a;  // FSS_RING_MASK
    }
}

__global__ void ring_kernel(int op, uint64_t mask, uint64_t count, const uint64_t* __restrict__ a,
                            const uint64_t* __restrict__ b, uint64_t bs, uint64_t* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint64_t bv = b ? b[i] : bs;
        out[i] = apply(op, a[i], bv) & mask;
    }
}

// Beaver elementwise combine (beaver.py:286-292):
//   delta = d_own + d_peer, eps = e_own + e_peer,
//   z = delta*b + a*eps + c (+ delta*eps for party 0)
__global__ void beaver_kernel(int party, uint64_t mask, uint64_t count,
                              const uint64_t* __restrict__ d_own, const uint64_t* __restrict__ d_peer,
                              const uint64_t* __restrict__ e_own, const uint64_t* __restrict__ e_peer,
                              const uint64_t* __restrict__ ta, const uint64_t* __restrict__ tb,
                              const uint64_t* __restrict__ tc, uint64_t* __restrict__ z) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint64_t d = (d_own[i] + d_peer[i]) & mask;
        const uint64_t e = (e_own[i] + e_peer[i]) & mask;
        uint64_t v = d * tb[i] + ta[i] * e + tc[i];
        if (party == 0) v += d * e;
        z[i] = v & mask;
    }
}

int grid_size(uint64_t count) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (!sms) sms = 148;
    }
    const uint64_t need = (count + 255) / 256;
    const uint64_t cap = (uint64_t)sms * 8;
    return (int)(need < cap ? (need ? need : 1) : cap);
}

int done() {
    const cudaError_t err = cudaGetLastError();
    return err == cudaSuccess ? FSS_OK : fssb::set_error(FSS_ECUDA, cudaGetErrorString(err));
}

}  // namespace

extern "C" {

int fss_ring_op(int op, int n_bits, uint64_t count, const uint64_t* a, const uint64_t* b,
                uint64_t b_scalar, uint64_t* out, void* stream) {
    if (n_bits < 1 || n_bits > 64) return fssb::set_error(FSS_EINVAL, "ring width out of range");
    if (op < FSS_RING_ADD || op > FSS_RING_MASK) return fssb::set_error(FSS_EINVAL, "bad ring op");
    if (count == 0) return FSS_OK;
    const uint64_t mask = n_bits >= 64 ? ~0ULL : ((1ULL << n_bits) - 1);
    ring_kernel<<<grid_size(count), 256, 0, (cudaStream_t)stream>>>(op, mask, count, a, b, b_scalar, out);
    return done();
}

int fss_beaver_mul(int party, int n_bits, uint64_t count, const uint64_t* delta_own,
                   const uint64_t* delta_peer, const uint64_t* eps_own, const uint64_t* eps_peer,
                   const uint64_t* a, const uint64_t* b, const uint64_t* c, uint64_t* z,
                   void* stream) {
    if (party != 0 && party != 1) return fssb::set_error(FSS_EINVAL, "party must be 0 or 1");
    if (n_bits < 1 || n_bits > 64) return fssb::set_error(FSS_EINVAL, "ring width out of range");
    if (count == 0) return FSS_OK;
    const uint64_t mask = n_bits >= 64 ? ~0ULL : ((1ULL << n_bits) - 1);
    beaver_kernel<<<grid_size(count), 256, 0, (cudaStream_t)stream>>>(
        party, mask, count, delta_own, delta_peer, eps_own, eps_peer, a, b, c, z);
    return done();
}

}  // extern "C"
