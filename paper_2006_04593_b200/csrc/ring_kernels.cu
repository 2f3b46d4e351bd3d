// Elementwise Z_2^n ring arithmetic for the share layer (reference ring.py:99-129),
// the wire packing of the one masked message (sharing.py:191-230) and the
// Beaver combine (beaver.py:257-294).
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

// Wire format of the share layer (sharing.py:191-207 pack_ring/_wire_dtype):
// ring values travel at the smallest power-of-two byte width covering n_bits.
using fssb::wire_get;

__device__ __forceinline__ void wire_put(int wb, void* p, uint64_t i, uint64_t v) {
    switch (wb) {
        case 1: reinterpret_cast<uint8_t*>(p)[i] = (uint8_t)v; break;
        case 2: reinterpret_cast<uint16_t*>(p)[i] = (uint16_t)v; break;
        case 4: reinterpret_cast<uint32_t*>(p)[i] = (uint32_t)v; break;
        default: reinterpret_cast<uint64_t*>(p)[i] = v;
    }
}

// wire = (a op b) & mask  (mask_and_reveal's y + alpha, Beaver's x - a / y - b)
__global__ void wire_pack_kernel(int op, int wb, uint64_t mask, uint64_t count,
                                 const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                                 void* __restrict__ wire) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint64_t bv = b ? b[i] : 0;
        wire_put(wb, wire, i, apply(op, a[i], bv) & mask);
    }
}

// out = (own + peer) & mask: the public value both parties reconstruct
__global__ void wire_open_kernel(int wb, uint64_t mask, uint64_t count, const void* __restrict__ own,
                                 const void* __restrict__ peer, uint64_t* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint64_t p = peer ? wire_get(wb, peer, i) : 0;
        out[i] = (wire_get(wb, own, i) + p) & mask;
    }
}

// Beaver elementwise combine (beaver.py:281-292) fused with the opening of
// delta and eps from the two parties' wire messages:
//   delta = d_own + d_peer, eps = e_own + e_peer,
//   z = delta*b + a*eps + c (+ delta*eps for party 0)
__global__ void beaver_kernel(int party, int wb, uint64_t mask, uint64_t count,
                              const void* __restrict__ d_own, const void* __restrict__ d_peer,
                              const void* __restrict__ e_own, const void* __restrict__ e_peer,
                              const uint64_t* __restrict__ ta, const uint64_t* __restrict__ tb,
                              const uint64_t* __restrict__ tc, uint64_t* __restrict__ z) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint64_t d = (wire_get(wb, d_own, i) + wire_get(wb, d_peer, i)) & mask;
        const uint64_t e = (wire_get(wb, e_own, i) + wire_get(wb, e_peer, i)) & mask;
        uint64_t v = d * tb[i] + ta[i] * e + tc[i];
        if (party == 0) v += d * e;
        z[i] = v & mask;
    }
}

// argmax's pairwise differences (reference nn_ops.py:111-114): for each row of
// m values, out[j][k] = v[i] - v[j] over the m-1 indices i != j in ascending
// order (k = i for i < j, i - 1 for i > j), mod 2^n. One thread per output;
// the row's m values are re-read from L1/L2.
__global__ void pairwise_kernel(uint64_t mask, uint64_t rows, uint32_t m, const uint64_t* __restrict__ v,
                                uint64_t* __restrict__ out) {
    const uint32_t per = m * (m - 1);
    const uint64_t total = rows * per;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < total; o += stride) {
        const uint64_t r = o / per;
        const uint32_t w = (uint32_t)(o - r * per);
        const uint32_t j = w / (m - 1), k = w - j * (m - 1);
        const uint32_t i = k + (k >= j);
        const uint64_t* row = v + r * m;
        out[o] = (__ldg(row + i) - __ldg(row + j)) & mask;
    }
}

// out[q] = (sum of the g values in[q*g .. q*g+g) + add) mod 2^n: the per-row
// counts of argmax (nn_ops.py:115-116, with the public -(m-1) of party 0)
// and maxpool's window sums (nn_ops.py:174).
__global__ void group_sum_kernel(uint64_t mask, uint64_t groups, uint32_t g, const uint64_t* __restrict__ in,
                                 uint64_t add, uint64_t* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < groups; q += stride) {
        const uint64_t* p = in + q * g;
        uint64_t acc = add;
        for (uint32_t t = 0; t < g; t++) acc += __ldg(p + t);
        out[q] = acc & mask;
    }
}

int grid_size(uint64_t count) {
    static int sms_of[64] = {0};  // per device; benign race (same value written)
    int dev = 0;
    cudaGetDevice(&dev);
    int& sms = sms_of[dev & 63];
    if (!sms) {
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
    if (!a || !out) return fssb::set_error(FSS_EINVAL, "null device pointer");
    const uint64_t mask = n_bits >= 64 ? ~0ULL : ((1ULL << n_bits) - 1);
    ring_kernel<<<grid_size(count), 256, 0, (cudaStream_t)stream>>>(op, mask, count, a, b, b_scalar, out);
    return done();
}

int fss_wire_bytes(int n_bits) {
    if (n_bits < 1 || n_bits > 64) return 0;
    return fssb::wire_bytes(n_bits);
}

int fss_wire_pack(int op, int n_bits, uint64_t count, const uint64_t* a, const uint64_t* b,
                  void* wire, void* stream) {
    if (n_bits < 1 || n_bits > 64) return fssb::set_error(FSS_EINVAL, "ring width out of range");
    if (op != FSS_RING_ADD && op != FSS_RING_SUB)
        return fssb::set_error(FSS_EINVAL, "wire pack supports add/sub only");
    if (count == 0) return FSS_OK;
    if (!a || !wire) return fssb::set_error(FSS_EINVAL, "null device pointer");
    const uint64_t mask = n_bits >= 64 ? ~0ULL : ((1ULL << n_bits) - 1);
    wire_pack_kernel<<<grid_size(count), 256, 0, (cudaStream_t)stream>>>(
        op, fss_wire_bytes(n_bits), mask, count, a, b, wire);
    return done();
}

int fss_wire_open(int n_bits, uint64_t count, const void* own, const void* peer, uint64_t* out,
                  void* stream) {
    if (n_bits < 1 || n_bits > 64) return fssb::set_error(FSS_EINVAL, "ring width out of range");
    if (count == 0) return FSS_OK;
    if (!own || !out) return fssb::set_error(FSS_EINVAL, "null device pointer");
    const uint64_t mask = n_bits >= 64 ? ~0ULL : ((1ULL << n_bits) - 1);
    wire_open_kernel<<<grid_size(count), 256, 0, (cudaStream_t)stream>>>(
        fss_wire_bytes(n_bits), mask, count, own, peer, out);
    return done();
}

int fss_beaver_mul(int party, int n_bits, uint64_t count, const void* delta_own,
                   const void* delta_peer, const void* eps_own, const void* eps_peer,
                   const uint64_t* a, const uint64_t* b, const uint64_t* c, uint64_t* z,
                   void* stream) {
    if (party != 0 && party != 1) return fssb::set_error(FSS_EINVAL, "party must be 0 or 1");
    if (n_bits < 1 || n_bits > 64) return fssb::set_error(FSS_EINVAL, "ring width out of range");
    if (count == 0) return FSS_OK;
    if (!delta_own || !delta_peer || !eps_own || !eps_peer || !a || !b || !c || !z)
        return fssb::set_error(FSS_EINVAL, "null device pointer");
    const uint64_t mask = n_bits >= 64 ? ~0ULL : ((1ULL << n_bits) - 1);
    beaver_kernel<<<grid_size(count), 256, 0, (cudaStream_t)stream>>>(
        party, fss_wire_bytes(n_bits), mask, count, delta_own, delta_peer, eps_own, eps_peer, a, b,
        c, z);
    return done();
}

int fss_ring_pairwise(int n_bits, uint64_t rows, int m, const uint64_t* v, uint64_t* out, void* stream) {
    if (n_bits < 1 || n_bits > 64) return fssb::set_error(FSS_EINVAL, "ring width out of range");
    if (m < 2 || m > 65536) return fssb::set_error(FSS_EINVAL, "pairwise: m must be in [2, 65536]");
    if (rows == 0) return FSS_OK;
    if (!v || !out) return fssb::set_error(FSS_EINVAL, "null device pointer");
    const uint64_t mask = n_bits >= 64 ? ~0ULL : ((1ULL << n_bits) - 1);
    pairwise_kernel<<<grid_size(rows * (uint64_t)m * (m - 1)), 256, 0, (cudaStream_t)stream>>>(
        mask, rows, (uint32_t)m, v, out);
    return done();
}

int fss_ring_group_sum(int n_bits, uint64_t groups, int g, const uint64_t* in, uint64_t add, uint64_t* out,
                       void* stream) {
    if (n_bits < 1 || n_bits > 64) return fssb::set_error(FSS_EINVAL, "ring width out of range");
    if (g < 1) return fssb::set_error(FSS_EINVAL, "group sum: group size must be >= 1");
    if (groups == 0) return FSS_OK;
    if (!in || !out) return fssb::set_error(FSS_EINVAL, "null device pointer");
    const uint64_t mask = n_bits >= 64 ? ~0ULL : ((1ULL << n_bits) - 1);
    group_sum_kernel<<<grid_size(groups), 256, 0, (cudaStream_t)stream>>>(mask, groups, (uint32_t)g, in,
                                                                           add, out);
    return done();
}

}  // extern "C"
