// ARNK key-container payloads (reference LAYOUT.md:48-71, fss.py:498-602) on
// device: level-major SoA keys <-> element-major per-party byte payloads.
//
// Element layout (w = ceil(n/8) little-endian bytes per ring value):
//   eq : alpha_share[w] | seed0[16] | n x (scw[16] | flags[1])           | cw_final[w]
//   cmp: alpha_share[w] | seed0[16] | n x (scw[16] | flags[1] | sigma[w]) | (n+1) x leaf[w]
//
// Tiled transpose through shared memory. A CTA owns a tile of E consecutive
// elements: their payload records are one contiguous byte range of HBM
// (E * elem bytes), moved between HBM and shared memory with 16-byte vector
// accesses; the level-major key rows of the tile (scw[i][e0 .. e0+E), tcw,
// sigma, leaf, ...) are read / written with consecutive threads on consecutive
// elements, i.e. coalesced. All byte-level (re)assembly happens in shared
// memory, so HBM traffic is the algorithmic bytes: the payload once plus the
// key arrays once.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../../include/ariann_fss.h"
#include "common.cuh"

#ifndef FSSB_ARNK_NAIVE
#define FSSB_ARNK_NAIVE 0
#endif

namespace {

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

#if FSSB_ARNK_NAIVE
__device__ __forceinline__ void put_le(uint8_t* p, uint64_t v, int w) {
    for (int b = 0; b < w; b++) p[b] = (uint8_t)(v >> (8 * b));
}

__device__ __forceinline__ uint64_t get_le(const uint8_t* p, int w) {
    uint64_t v = 0;
    for (int b = 0; b < w; b++) v |= (uint64_t)p[b] << (8 * b);
    return v;
}

// Round-1 first cut, kept for the variant sweep (scripts/aes_variants.py):
// one thread per (element, slot), byte loads / stores straight to the
// element-major payload in HBM -- a warp's 32 lanes touch 32 different lines
// per byte instruction.
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
#endif

constexpr int kArnkThreads = 256;

__device__ __forceinline__ uint32_t sld32(const uint8_t* s, uint32_t off) {
    return *reinterpret_cast<const uint32_t*>(s + off);
}

// NB (<= 8) little-endian bytes at any byte offset of the shared tile (the
// tile buffer has 16 bytes of slack so the covering word reads stay in bounds).
template <int NB>
__device__ __forceinline__ uint64_t sget(const uint8_t* s, uint32_t off) {
    const uint32_t a = off & ~3u, sh = (off & 3u) * 8u;
    const uint32_t w0 = sld32(s, a), w1 = sld32(s, a + 4);
    uint64_t v = __funnelshift_r(w0, w1, sh);
    if (NB > 4) v |= (uint64_t)__funnelshift_r(w1, sld32(s, a + 8), sh) << 32;
    return NB >= 8 ? v : v & ((1ULL << (8 * NB)) - 1);
}

__device__ __forceinline__ uint4 sget16(const uint8_t* s, uint32_t off) {
    const uint32_t a = off & ~3u, sh = (off & 3u) * 8u;
    const uint32_t w0 = sld32(s, a), w1 = sld32(s, a + 4), w2 = sld32(s, a + 8), w3 = sld32(s, a + 12),
                   w4 = sld32(s, a + 16);
    return make_uint4(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh), __funnelshift_r(w2, w3, sh),
                      __funnelshift_r(w3, w4, sh));
}

// Store the NB (<= 28) bytes of the little-endian byte stream R[0..6] at tile
// offset A + r (A word-aligned, r = offset mod 4, both layouts compile-time
// after unrolling): whole aligned words as 32-bit stores, only the partial
// words at either end byte by byte (their other bytes belong to neighbouring
// fields written by other threads). Aligned word k holds stream bytes
// [4k - r, 4k - r + 4).
template <int r, int NB>
__device__ __forceinline__ void sput_stream_r(uint8_t* s, uint32_t A, const uint32_t (&R)[7]) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const int lo = 4 * k - r;
        if (lo >= NB) break;
        const uint32_t prev = k > 0 ? R[k - 1] : 0u;
        const uint32_t cur = k < 7 ? R[k] : 0u;
        const uint32_t v = r ? __funnelshift_l(prev, cur, 8 * r) : cur;
        if (lo >= 0 && lo + 4 <= NB) {
            *reinterpret_cast<uint32_t*>(s + A + 4 * k) = v;
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++)
                if (lo + j >= 0 && lo + j < NB) s[A + 4 * k + j] = (uint8_t)(v >> (8 * j));
        }
    }
}

template <int NB>
__device__ __forceinline__ void sput_stream(uint8_t* s, uint32_t o, const uint32_t (&R)[7]) {
    const uint32_t A = o & ~3u;
    switch (o & 3u) {   // uniform across a warp whenever the record stride is word-aligned
        case 0: sput_stream_r<0, NB>(s, A, R); break;
        case 1: sput_stream_r<1, NB>(s, A, R); break;
        case 2: sput_stream_r<2, NB>(s, A, R); break;
        default: sput_stream_r<3, NB>(s, A, R); break;
    }
}

template <int NB>
__device__ __forceinline__ void sput_u64(uint8_t* s, uint32_t o, uint64_t v) {
    const uint32_t R[7] = {(uint32_t)v, (uint32_t)(v >> 32), 0, 0, 0, 0, 0};
    sput_stream<NB>(s, o, R);
}

__device__ __forceinline__ void sput16(uint8_t* s, uint32_t o, uint4 v) {
    const uint32_t R[7] = {v.x, v.y, v.z, v.w, 0, 0, 0};
    sput_stream<16>(s, o, R);
}

// Cooperative byte-range copy with the widest access both ends allow.
__device__ __forceinline__ void copy_range(uint8_t* dst, const uint8_t* src, uint64_t nbytes) {
    const uintptr_t mis = ((uintptr_t)dst | (uintptr_t)src);
    if ((mis & 15) == 0) {
        const uint64_t n16 = nbytes / 16;
        for (uint64_t i = threadIdx.x; i < n16; i += blockDim.x)
            reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
        for (uint64_t i = 16 * n16 + threadIdx.x; i < nbytes; i += blockDim.x) dst[i] = src[i];
    } else if ((mis & 3) == 0) {
        const uint64_t n4 = nbytes / 4;
        for (uint64_t i = threadIdx.x; i < n4; i += blockDim.x)
            reinterpret_cast<uint32_t*>(dst)[i] = reinterpret_cast<const uint32_t*>(src)[i];
        for (uint64_t i = 4 * n4 + threadIdx.x; i < nbytes; i += blockDim.x) dst[i] = src[i];
    } else {
        for (uint64_t i = threadIdx.x; i < nbytes; i += blockDim.x) dst[i] = src[i];
    }
}

// Work-item mapping for `rows` level-major rows x the E elements of a tile
// (E = 16 << lnb): each half-warp takes 16 consecutive elements of one row and
// the two half-warps of a warp take rows r and r + d (d = 1 << ld_). Row
// accesses in HBM stay coalesced (16 consecutive elements). In shared memory
// the 16 elements of one row, EB bytes apart, spread over 16 banks, and d is
// chosen so that d * rowbytes = 4 (mod 8) -- an odd number of words: the
// second row lands on the other 16 banks at the same byte alignment, so all
// 32 lanes take the same store path. Shifts only, no divisions.
__host__ __device__ __forceinline__ int row_step_log2(uint32_t rowbytes) {
    for (int l = 0; l <= 2; l++)
        if (((rowbytes << l) & 7u) == 4u) return l;
    return 0;
}

struct Item {
    uint32_t row, e;
};

__device__ __forceinline__ uint32_t pair_items(uint32_t rows, int lnb, int ld_) {
    const uint32_t blocks = (rows + (2u << ld_) - 1) >> (ld_ + 1);
    return (blocks << (ld_ + lnb)) * 32u;
}

__device__ __forceinline__ Item pair_item(uint32_t idx, int lnb, int ld_) {
    const uint32_t q = idx >> 5;
    const uint32_t pr = q >> lnb, eb = q & ((1u << lnb) - 1);
    const uint32_t blk = pr >> ld_, r0 = pr & ((1u << ld_) - 1);
    Item it;
    it.row = (blk << (ld_ + 1)) + r0 + (((idx >> 4) & 1u) << ld_);
    it.e = (eb << 4) + (idx & 15u);
    return it;
}

// ---- bulk asynchronous copies (TMA engine, cp.async.bulk) -------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

#ifndef FSSB_ARNK_BATCH
#define FSSB_ARNK_BATCH 4
#endif
constexpr int kBatch = FSSB_ARNK_BATCH;   // row loads in flight per thread (pack)

// Tiles are double-buffered per CTA: while the threads transpose tile j in one
// buffer, the TMA engine moves tile j+1 in (unpack) or tile j-1 out (pack) of
// the other, so the payload side of the transfer costs no thread time. A tile
// whose byte range is not 16-byte aligned (only the last, partial tile can be)
// falls back to a cooperative copy. KIND and the ring width W are template
// parameters so every record layout is compile-time.
template <bool PACK, int KIND, int W, int THREADS = kArnkThreads>
__global__ void __launch_bounds__(THREADS)
arnk_tile_kernel(int n, uint64_t count, uint64_t ld, int lnb, uint32_t stride, int use_tma, Keys k,
                 uint8_t* buf) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr uint32_t rec = KIND == 0 ? 17 : 17 + W;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);       // 2 mbarriers
    uint8_t* tiles_base = smem + 128;
    const uint32_t E = 16u << lnb;
    const uint32_t EB = (uint32_t)elem_bytes(KIND, n);
    const uint32_t tail = W + 16 + n * rec;   // cw_final (eq) / leaf block (cmp)
    const int d_lv = row_step_log2(rec), d_leaf = row_step_log2(W);
    const uint64_t tiles = (count + E - 1) / E;
    if (threadIdx.x == 0) {
        mbar_init(&bars[0]);
        mbar_init(&bars[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t parity = 0;   // bit b: phase of buffer b's mbarrier

    auto tile_m = [&](uint64_t t) { return (uint32_t)(count - t * E < (uint64_t)E ? count - t * E : E); };
    auto aligned = [&](uint32_t bytes, const uint8_t* gp) {
        return use_tma && (bytes & 15u) == 0 && ((uintptr_t)gp & 15u) == 0;
    };
    // unpack: bring tile t into buffer b (async when aligned)
    auto fetch = [&](uint64_t t, int b) {
        const uint32_t bytes = tile_m(t) * EB;
        const uint8_t* gp = buf + t * E * EB;
        uint8_t* dst = tiles_base + b * stride;
        if (aligned(bytes, gp)) {
            if (threadIdx.x == 0) bulk_load(dst, gp, bytes, &bars[b]);
        } else {
            copy_range(dst, gp, bytes);
        }
    };

    int j = 0;
    if (!PACK && blockIdx.x < tiles) fetch(blockIdx.x, 0);
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, j++) {
        const int cur = j & 1;
        uint8_t* tile = tiles_base + cur * stride;
        const uint32_t m = tile_m(t);
        const uint64_t e0 = t * E;
        uint8_t* gp = buf + e0 * EB;
        const bool async_io = aligned(m * EB, gp);
        if (!PACK) {
            const uint64_t tn = t + gridDim.x;
            if (tn < tiles) fetch(tn, cur ^ 1);    // buffer cur^1 was released at the end of j-1
            if (async_io) {
                mbar_wait(&bars[cur], (parity >> cur) & 1u);
                parity ^= 1u << cur;
            } else {
                __syncthreads();
            }
        } else {
            // the bulk store issued from this buffer two tiles ago must have
            // finished reading it (only the newest group may still be in flight)
            if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncthreads();
        }
        // per-level records (scw | flags | sigma)
        const uint32_t items = pair_items((uint32_t)n, lnb, d_lv);
        if (PACK) {
            for (uint32_t base = threadIdx.x; base < items; base += kBatch * THREADS) {
                uint4 v[kBatch];
                uint32_t f[kBatch], so[kBatch];
                uint64_t sg[kBatch];
                bool ok[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; u++) {   // all loads first: kBatch rows in flight
                    const uint32_t idx = base + u * THREADS;
                    const Item it = pair_item(idx, lnb, d_lv);
                    ok[u] = idx < items && it.row < (uint32_t)n && it.e < m;
                    if (ok[u]) {
                        const uint64_t off = (uint64_t)it.row * ld + e0 + it.e;
                        v[u] = *reinterpret_cast<const uint4*>(k.scw + 16 * off);
                        f[u] = k.tcw[off];
                        sg[u] = KIND == 1 ? k.sigma_cw[off] : 0;
                        so[u] = it.e * EB + W + 16 + it.row * rec;
                    }
                }
#pragma unroll
                for (int u = 0; u < kBatch; u++) {
                    if (!ok[u]) continue;
                    const uint32_t R[7] = {v[u].x, v[u].y, v[u].z, v[u].w, f[u] | ((uint32_t)sg[u] << 8),
                                           (uint32_t)(sg[u] >> 24), (uint32_t)(sg[u] >> 56)};
                    sput_stream<rec>(tile, so[u], R);
                }
            }
        } else {
            for (uint32_t idx = threadIdx.x; idx < items; idx += THREADS) {
                const Item it = pair_item(idx, lnb, d_lv);
                if (it.row >= (uint32_t)n || it.e >= m) continue;
                const uint64_t off = (uint64_t)it.row * ld + e0 + it.e;
                const uint32_t so = it.e * EB + W + 16 + it.row * rec;
                *reinterpret_cast<uint4*>(k.scw + 16 * off) = sget16(tile, so);
                k.tcw[off] = tile[so + 16];
                if (KIND == 1) k.sigma_cw[off] = sget<W>(tile, so + 17);
            }
        }
        // element head (alpha share, seed) and the eq tail (cw_final)
        for (uint32_t e = threadIdx.x; e < m; e += THREADS) {
            const uint32_t so = e * EB;
            if (PACK) {
                sput_u64<W>(tile, so, k.alpha_share[e0 + e]);
                sput16(tile, so + W, *reinterpret_cast<const uint4*>(k.seed0 + 16 * (e0 + e)));
                if (KIND == 0) sput_u64<W>(tile, so + tail, k.cw_final[e0 + e]);
            } else {
                k.alpha_share[e0 + e] = sget<W>(tile, so);
                *reinterpret_cast<uint4*>(k.seed0 + 16 * (e0 + e)) = sget16(tile, so + W);
                if (KIND == 0) k.cw_final[e0 + e] = sget<W>(tile, so + tail);
            }
        }
        // cmp leaf block: n + 1 rows of W-byte values
        if (KIND == 1) {
            const uint32_t leaf_items = pair_items((uint32_t)n + 1, lnb, d_leaf);
            if (PACK) {
                for (uint32_t base = threadIdx.x; base < leaf_items; base += kBatch * THREADS) {
                    uint64_t v[kBatch];
                    uint32_t so[kBatch];
                    bool ok[kBatch];
#pragma unroll
                    for (int u = 0; u < kBatch; u++) {
                        const uint32_t idx = base + u * THREADS;
                        const Item it = pair_item(idx, lnb, d_leaf);
                        ok[u] = idx < leaf_items && it.row <= (uint32_t)n && it.e < m;
                        if (ok[u]) {
                            v[u] = k.leaf_cw[(uint64_t)it.row * ld + e0 + it.e];
                            so[u] = it.e * EB + tail + it.row * W;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kBatch; u++)
                        if (ok[u]) sput_u64<W>(tile, so[u], v[u]);
                }
            } else {
                for (uint32_t idx = threadIdx.x; idx < leaf_items; idx += THREADS) {
                    const Item it = pair_item(idx, lnb, d_leaf);
                    if (it.row > (uint32_t)n || it.e >= m) continue;
                    k.leaf_cw[(uint64_t)it.row * ld + e0 + it.e] = sget<W>(tile, it.e * EB + tail + it.row * W);
                }
            }
        }
        if (PACK) {
            // generic-proxy smem writes -> visible to the TMA (async proxy) read
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (async_io) {
                if (threadIdx.x == 0) bulk_store(gp, tile, m * EB);
            } else {
                copy_range(gp, tile, (uint64_t)m * EB);
                if (threadIdx.x == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else {
            __syncthreads();   // tile consumed: its buffer may be refilled
        }
    }
    if (PACK && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- pack with asynchronously staged key rows ------------------------------
// The pack kernel above loads each thread's key rows with plain loads, so its
// warps stall on HBM latency and at the tile barriers (ncu r01f: long
// scoreboard + barrier stalls, 27 % issue-active). Here every row segment of
// tile j+1 -- scw, tcw, sigma, leaf, alpha, seed, cw_final -- is copied into
// a shared-memory staging buffer with cp.async (LDGSTS: global -> shared, no
// register round trip, all in flight at once) while the threads assemble tile
// j from the other staging buffer; the assembled payload leaves through the
// TMA bulk store as before. Needs ld % 4 == 0 (4-byte cp.async of the tcw
// rows, tcw / scw / seed bases aligned); other layouts take the kernel above.
__device__ __forceinline__ void cp_async(void* dst, const void* src, int bytes) {
    const uint32_t d = smem_u32(dst);
    if (bytes == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    else if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}

struct Stage {   // byte offsets of the row blocks inside one staging buffer (E elements)
    uint32_t scw, sig, leaf, alpha, cwf, seed, tcw, bytes;
};

__host__ __device__ __forceinline__ Stage stage_layout(int kind, int n, uint32_t E) {
    Stage g;
    g.scw = 0;
    g.sig = g.scw + (uint32_t)n * E * 16;
    g.leaf = g.sig + (kind == 1 ? (uint32_t)n * E * 8 : 0);
    g.alpha = g.leaf + (kind == 1 ? (uint32_t)(n + 1) * E * 8 : 0);
    g.cwf = g.alpha + E * 8;
    g.seed = g.cwf + (kind == 0 ? E * 8 : 0);
    g.tcw = g.seed + E * 16;
    g.bytes = (g.tcw + (uint32_t)n * E + 127) / 128 * 128;
    return g;
}

// Assemble the element-major payload records of one tile (m <= E elements)
// from its staged level-major key rows S (layout G) into the tile buffer.
template <int KIND, int W, int THREADS>
__device__ __forceinline__ void assemble_stage(uint8_t* tile, const uint8_t* S, const Stage& G, int n, int lnb,
                                               uint32_t m) {
    constexpr uint32_t rec = KIND == 0 ? 17 : 17 + W;
    const uint32_t E = 16u << lnb;
    const uint32_t EB = (uint32_t)elem_bytes(KIND, n);
    const uint32_t tail = W + 16 + n * rec;
    const int d_lv = row_step_log2(rec), d_leaf = row_step_log2(W);
    const uint32_t items = pair_items((uint32_t)n, lnb, d_lv);
    for (uint32_t idx = threadIdx.x; idx < items; idx += THREADS) {
        const Item it = pair_item(idx, lnb, d_lv);
        if (it.row >= (uint32_t)n || it.e >= m) continue;
        const uint32_t so = it.e * EB + W + 16 + it.row * rec;
        const uint4 v = *reinterpret_cast<const uint4*>(S + G.scw + (it.row * E + it.e) * 16);
        const uint32_t f = S[G.tcw + it.row * E + it.e];
        const uint64_t sg = KIND == 1 ? *reinterpret_cast<const uint64_t*>(S + G.sig + (it.row * E + it.e) * 8)
                                      : 0;
        const uint32_t R[7] = {v.x, v.y, v.z, v.w, f | ((uint32_t)sg << 8), (uint32_t)(sg >> 24),
                               (uint32_t)(sg >> 56)};
        sput_stream<rec>(tile, so, R);
    }
    for (uint32_t e = threadIdx.x; e < m; e += THREADS) {
        const uint32_t so = e * EB;
        sput_u64<W>(tile, so, *reinterpret_cast<const uint64_t*>(S + G.alpha + e * 8));
        sput16(tile, so + W, *reinterpret_cast<const uint4*>(S + G.seed + e * 16));
        if (KIND == 0) sput_u64<W>(tile, so + tail, *reinterpret_cast<const uint64_t*>(S + G.cwf + e * 8));
    }
    if (KIND == 1) {
        const uint32_t leaf_items = pair_items((uint32_t)n + 1, lnb, d_leaf);
        for (uint32_t idx = threadIdx.x; idx < leaf_items; idx += THREADS) {
            const Item it = pair_item(idx, lnb, d_leaf);
            if (it.row > (uint32_t)n || it.e >= m) continue;
            sput_u64<W>(tile, it.e * EB + tail + it.row * W,
                        *reinterpret_cast<const uint64_t*>(S + G.leaf + (it.row * E + it.e) * 8));
        }
    }
}

template <int KIND, int W>
__global__ void __launch_bounds__(kArnkThreads)
arnk_pack_async_kernel(int n, uint64_t count, uint64_t ld, int lnb, uint32_t stride, uint32_t sstride,
                       int use_tma, Keys k, uint8_t* buf) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* tiles_base = smem;                    // 2 payload buffers
    uint8_t* stage_base = smem + 2 * stride;       // 2 staging buffers
    const uint32_t E = 16u << lnb;
    const uint32_t EB = (uint32_t)elem_bytes(KIND, n);
    const Stage G = stage_layout(KIND, n, E);
    const uint64_t tiles = (count + E - 1) / E;
    auto tile_m = [&](uint64_t t) { return (uint32_t)(count - t * E < (uint64_t)E ? count - t * E : E); };

    // issue the copies of tile t's key rows into staging buffer b (one group)
    auto stage_in = [&](uint64_t t, int b) {
        uint8_t* S = stage_base + b * sstride;
        const uint64_t e0 = t * E;
        const uint32_t m = tile_m(t);
        const uint32_t q16 = m;                             // 16-B pieces per scw row
        // scw rows (16 B per key) and seeds
        for (uint32_t i = threadIdx.x; i < (uint32_t)n * q16; i += kArnkThreads) {
            const uint32_t row = i / q16, e = i - row * q16;
            cp_async(S + G.scw + (row * E + e) * 16, k.scw + 16 * ((uint64_t)row * ld + e0 + e), 16);
        }
        for (uint32_t e = threadIdx.x; e < m; e += kArnkThreads) {
            cp_async(S + G.seed + e * 16, k.seed0 + 16 * (e0 + e), 16);
            cp_async(S + G.alpha + e * 8, k.alpha_share + e0 + e, 8);
            if (KIND == 0) cp_async(S + G.cwf + e * 8, k.cw_final + e0 + e, 8);
        }
        if (KIND == 1) {
            // sigma / leaf rows (8 B per key): 16-byte pieces of key pairs when
            // the rows are 16-byte aligned (ld even; e0 is a multiple of 16),
            // the odd last key of a ragged tile on its own
            const bool a16 = !(ld & 1) && !(((uintptr_t)k.sigma_cw | (uintptr_t)k.leaf_cw) & 15);
            const uint32_t pairs = a16 ? m / 2 : 0, singles = m - 2 * pairs;
            const uint32_t q = pairs + singles;
            for (uint32_t i = threadIdx.x; i < (uint32_t)(2 * n + 1) * q; i += kArnkThreads) {
                const uint32_t r = i / q, c = i - r * q;
                const bool leaf = r >= (uint32_t)n;
                const uint32_t row = leaf ? r - n : r;
                const uint32_t e = c < pairs ? 2 * c : 2 * pairs + (c - pairs);
                const uint64_t* src = (leaf ? k.leaf_cw : k.sigma_cw) + (uint64_t)row * ld + e0 + e;
                cp_async(S + (leaf ? G.leaf : G.sig) + (row * E + e) * 8, src, c < pairs ? 16 : 8);
            }
        }
        // tcw rows: one 16-byte piece per 16 keys when ld % 16 == 0, else
        // 4-byte pieces (ld % 4 == 0); a ragged tail of the last tile by plain
        // byte copies
        const uint32_t pw = ((ld & 15) || ((uintptr_t)k.tcw & 15)) ? 4 : 16;
        const uint32_t qw = m / pw;
        for (uint32_t i = threadIdx.x; i < (uint32_t)n * qw; i += kArnkThreads) {
            const uint32_t row = i / qw, w = i - row * qw;
            cp_async(S + G.tcw + row * E + pw * w, k.tcw + (uint64_t)row * ld + e0 + pw * w, (int)pw);
        }
        const uint32_t rag = m - pw * qw;
        for (uint32_t i = threadIdx.x; i < (uint32_t)n * rag; i += kArnkThreads) {
            const uint32_t row = i / rag, e = pw * qw + (i - row * rag);
            S[G.tcw + row * E + e] = k.tcw[(uint64_t)row * ld + e0 + e];
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    int j = 0;
    if (blockIdx.x < tiles) stage_in(blockIdx.x, 0);
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, j++) {
        const int cur = j & 1;
        uint8_t* tile = tiles_base + cur * stride;
        const uint8_t* S = stage_base + cur * sstride;
        const uint32_t m = tile_m(t);
        uint8_t* gp = buf + t * E * EB;
        const bool async_io = use_tma && ((m * EB) & 15u) == 0 && ((uintptr_t)gp & 15u) == 0;
        // staging buffer cur^1 was consumed by tile j-1 (barrier at its end)
        const uint64_t tn = t + gridDim.x;
        if (tn < tiles) {
            stage_in(tn, cur ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");   // tile j's rows have landed
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        // the bulk store issued from this payload buffer two tiles ago has read it
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        assemble_stage<KIND, W, kArnkThreads>(tile, S, G, n, lnb, m);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();   // payload assembled; staging buffer cur fully read
        if (async_io) {
            if (threadIdx.x == 0) bulk_store(gp, tile, m * EB);
        } else {
            copy_range(gp, tile, (uint64_t)m * EB);
            if (threadIdx.x == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- pack with the key rows staged by TMA tensor copies -------------------
// Each level-major key array is a 2-D tensor (rows = levels, row pitch ld
// elements): the rows of a tile are ONE box [E elements x n rows], so a tile's
// whole staging buffer arrives with seven cp.async.bulk.tensor copies issued
// by one thread (completion on the buffer's mbarrier), instead of every thread
// issuing 16-byte LDGSTS pieces (the tcw rows of a 16-key tile are 16-byte
// pieces from n different lines: 7.3 M excess L1 wavefronts per 2^22 keys,
// profiles/ncu_arnk_pack.json) plus the index arithmetic of the stage-in
// loops. Elements past `count` are zero-filled by the TMA unit and skipped by
// the assembly. The staging layout is stage_layout's, so the assembly is
// shared with the LDGSTS kernel above. Needs ld % 16 == 0 (tcw row pitch) and
// 16-byte aligned bases; other layouts take the kernels above.
struct PackMaps {
    CUtensorMap scw, tcw, sig, leaf, alpha, seed, cwf;
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const CUtensorMap* map, int c0, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(smem_u32(bar))
        : "memory");
}

#ifndef FSSB_ARNK_TMA_THREADS
#define FSSB_ARNK_TMA_THREADS 512
#endif

// Staging buffers per CTA (loads run STAGES - 1 tiles ahead) and CTA size,
// measured at n = 32 with round-robin timing (scripts/arnk_bench.py,
// profiles/r02_arnk_tma_pack.json): cmp 3 stages (0.909 of HBM vs 0.885 with
// 2), eq 2 stages (0.933 vs 0.824 with 3), 512 threads for both.
#ifndef FSSB_ARNK_TMA_STAGES_CMP
#define FSSB_ARNK_TMA_STAGES_CMP 3
#endif
#ifndef FSSB_ARNK_TMA_STAGES_EQ
#define FSSB_ARNK_TMA_STAGES_EQ 2
#endif

template <int KIND, int W, int THREADS, int kTmaStages>
__global__ void __launch_bounds__(THREADS)
arnk_pack_tma_kernel(const __grid_constant__ PackMaps M, int n, uint64_t count, int lnb, uint32_t stride,
                     uint32_t sstride, int use_tma_store, uint8_t* buf) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);   // full barriers of the staging buffers
    uint8_t* tiles_base = smem + 128;                      // 2 payload buffers
    uint8_t* stage_base = tiles_base + 2 * stride;         // kTmaStages staging buffers
    const uint32_t E = 16u << lnb;
    const uint32_t EB = (uint32_t)elem_bytes(KIND, n);
    const Stage G = stage_layout(KIND, n, E);
    const uint64_t tiles = (count + E - 1) / E;
    auto tile_m = [&](uint64_t t) { return (uint32_t)(count - t * E < (uint64_t)E ? count - t * E : E); };
    // box bytes of one tile (out-of-range elements are delivered as zeros and count)
    const uint32_t tx = (uint32_t)n * E * (16 + 1) + E * (8 + 16) +
                        (KIND == 1 ? (uint32_t)(2 * n + 1) * E * 8 : E * 8);
    auto issue = [&](uint64_t t, int b) {   // thread 0 only
        uint8_t* S = stage_base + b * sstride;
        const int e0 = (int)(t * E);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[b])), "r"(tx)
                     : "memory");
        tma_load_2d(S + G.scw, &M.scw, 4 * e0, 0, &bars[b]);
        tma_load_2d(S + G.tcw, &M.tcw, e0, 0, &bars[b]);
        tma_load_1d(S + G.alpha, &M.alpha, e0, &bars[b]);
        tma_load_1d(S + G.seed, &M.seed, 4 * e0, &bars[b]);
        if (KIND == 1) {
            tma_load_2d(S + G.sig, &M.sig, e0, 0, &bars[b]);
            tma_load_2d(S + G.leaf, &M.leaf, e0, 0, &bars[b]);
        } else {
            tma_load_1d(S + G.cwf, &M.cwf, e0, &bars[b]);
        }
    };
    if (threadIdx.x == 0) {
        for (int b = 0; b < kTmaStages; b++) mbar_init(&bars[b]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int b = 0; b + 1 < kTmaStages; b++)
            if (blockIdx.x + (uint64_t)b * gridDim.x < tiles) issue(blockIdx.x + (uint64_t)b * gridDim.x, b);
    }
    __syncthreads();
    uint32_t parity = 0;   // bit b: phase of staging buffer b's mbarrier
    int j = 0, sb = 0;     // sb = j mod kTmaStages
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, j++, sb = sb + 1 == kTmaStages ? 0 : sb + 1) {
        uint8_t* tile = tiles_base + (j & 1) * stride;
        const uint8_t* S = stage_base + sb * sstride;
        const uint32_t m = tile_m(t);
        uint8_t* gp = buf + t * E * EB;
        const bool async_io = use_tma_store && ((m * EB) & 15u) == 0 && ((uintptr_t)gp & 15u) == 0;
        if (threadIdx.x == 0) {
            // the staging buffer of tile j + kTmaStages - 1 held tile j - 1, fully
            // read before the barrier that ended iteration j - 1
            const uint64_t tn = t + (uint64_t)(kTmaStages - 1) * gridDim.x;
            if (tn < tiles) issue(tn, sb == 0 ? kTmaStages - 1 : sb - 1);
            // the bulk store issued from this payload buffer two tiles ago has read it
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        mbar_wait(&bars[sb], (parity >> sb) & 1u);
        parity ^= 1u << sb;
        __syncthreads();   // payload buffer j & 1 is free (thread 0's wait above)
        assemble_stage<KIND, W, THREADS>(tile, S, G, n, lnb, m);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();   // payload assembled; staging buffer sb fully read
        if (async_io) {
            if (threadIdx.x == 0) bulk_store(gp, tile, m * EB);
        } else {
            copy_range(gp, tile, (uint64_t)m * EB);
            if (threadIdx.x == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Tile of E = 16 << lnb elements, two tile buffers per CTA. Pack (the
// fallback tile kernel): 64 only up to 100 KiB, i.e. 32 for cmp n = 32 (four
// CTAs per SM hide its row-load latency better) -- measured,
// profiles/r01_arnk_variants.json. Largest record: cmp n = 63, 2,111 B.
#ifndef FSSB_ARNK_TILE_KB
#define FSSB_ARNK_TILE_KB 100
#endif
// Unpack: 128-key tiles (two buffers of 103 KB for DCF at n = 32, one CTA
// of 512 threads per SM) write longer level-row segments per tile than 64-key
// tiles at two CTAs per SM: DCF 0.873 -> 0.897, DPF 0.884 -> 0.920 of HBM
// (scripts/arnk_bench.py variants un_t128*, profiles/r02_arnk_unpack_tiles.json);
// 32-key tiles were worse, the thread count (128-1024) hardly matters.
#ifndef FSSB_ARNK_UNPACK_TILE_KB
#define FSSB_ARNK_UNPACK_TILE_KB 215
#endif
int arnk_tile_lnb(bool pack, int kind, int n) {
    // the largest tile (16 << lnb keys, lnb <= 3) whose two buffers fit the budget
    const uint64_t kb = pack ? FSSB_ARNK_TILE_KB : FSSB_ARNK_UNPACK_TILE_KB;
    int lnb = 1;
    while (lnb < 3 && 2 * elem_bytes(kind, n) * (16u << (lnb + 1)) <= kb * 1024) lnb++;
    return lnb;
}

#ifndef FSSB_ARNK_UNPACK_THREADS
#define FSSB_ARNK_UNPACK_THREADS 512
#endif
#ifndef FSSB_ARNK_ASYNC_PACK
#define FSSB_ARNK_ASYNC_PACK 1
#endif

template <int KIND, int W>
cudaError_t launch_pack_async(int n, uint64_t count, uint64_t ld, Keys k, uint8_t* buf, cudaStream_t st) {
    // 32-key tiles when two CTAs (2 payload + 2 staging buffers each) fit an
    // SM, else 16-key tiles: the assembly needs the warps of several CTAs
    // (cmp n = 32: 32 keys = 122 KB per CTA, one CTA per SM measured 30 %
    // slower than 16 keys at three CTAs per SM)
    auto smem_for = [&](uint32_t E) {
        return 2 * (size_t)((elem_bytes(KIND, n) * E + 16 + 127) / 128 * 128) +
               2 * (size_t)stage_layout(KIND, n, E).bytes;
    };
    const int lnb = 2 * smem_for(32) <= 200 * 1024 ? 1 : 0;
    const uint32_t E = 16u << lnb;
    const uint32_t stride = (uint32_t)((elem_bytes(KIND, n) * E + 16 + 127) / 128 * 128);
    const uint32_t sstride = stage_layout(KIND, n, E).bytes;
    const size_t smem = smem_for(E);
    int dev = 0, sms = 0, per_sm = 1;
    auto kern = arnk_pack_async_kernel<KIND, W>;
    cudaError_t err = cudaGetDevice(&dev);
    if (err == cudaSuccess) err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err == cudaSuccess) err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err == cudaSuccess) err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kArnkThreads, smem);
    if (err != cudaSuccess) return err;
    const uint64_t tiles = (count + E - 1) / E;
    const uint64_t cap = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
    static const int use_tma = getenv("FSSB_ARNK_NO_TMA") ? 0 : 1;
    kern<<<(unsigned)(tiles < cap ? tiles : cap), kArnkThreads, smem, st>>>(n, count, ld, lnb, stride, sstride,
                                                                           use_tma, k, buf);
    return cudaGetLastError();
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda
// link dependency); NULL when the driver does not provide it.
#ifndef FSSB_ARNK_TMA_L2PROMO
#define FSSB_ARNK_TMA_L2PROMO 3   // CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// rows x dim0 tensor (row pitch `pitch` bytes; rows == 0: 1-D) read in boxes of
// box0 x rows elements
bool encode_map(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t dim0, uint32_t rows,
                uint64_t pitch, uint32_t box0) {
    const cuuint64_t dims[2] = {dim0, rows ? rows : 1};
    const cuuint64_t strides[1] = {pitch};
    const cuuint32_t box[2] = {box0, rows ? rows : 1};
    const cuuint32_t estr[2] = {1, 1};
    return encode_fn()(map, dt, rows ? 2 : 1, const_cast<void*>(base), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)FSSB_ARNK_TMA_L2PROMO,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#ifndef FSSB_ARNK_TMA_PACK
#define FSSB_ARNK_TMA_PACK 1
#endif
// Keys per TMA pack tile = 16 << lnb, per kind (scripts/arnk_bench.py, r02):
// cmp 32-key tiles move the tile's rows in half as many TMA boxes per key and
// pack at 1.20 vs 1.35 ms per 2^22 keys (6.67 TB/s, above the 1:1 copy peak:
// the mix is read-heavy); eq stays at 16 (0.79 vs 0.84 ms).
#ifdef FSSB_ARNK_TMA_LNB
#define FSSB_ARNK_TMA_LNB_CMP FSSB_ARNK_TMA_LNB
#define FSSB_ARNK_TMA_LNB_EQ FSSB_ARNK_TMA_LNB
#endif
#ifndef FSSB_ARNK_TMA_LNB_CMP
#define FSSB_ARNK_TMA_LNB_CMP 1
#endif
#ifndef FSSB_ARNK_TMA_LNB_EQ
#define FSSB_ARNK_TMA_LNB_EQ 0
#endif

// The TMA-staged pack when the layout allows it (returns false otherwise and
// launches nothing): tcw row pitch ld a multiple of 16 bytes, sigma / leaf
// pitch (8 ld) too, every base 16-byte aligned, 4 count within a tensor
// dimension, and an even count: the TMA unit moves the inner dimension in
// 16-byte units, so a tensor of u64 values must end on a 16-byte boundary
// (measured on the store side, r02r: an odd-count 1-D u64 tensor got one
// element written past its end; the load side reads the same units).
template <int KIND, int W>
bool try_pack_tma(int n, uint64_t count, uint64_t ld, const Keys& k, uint8_t* buf, cudaStream_t st,
                  cudaError_t* err) {
    if (!FSSB_ARNK_TMA_PACK || ld % 16 || count % 2 || 4 * count >= (1ull << 32) || !encode_fn()) return false;
    const uintptr_t bases = (uintptr_t)k.scw | (uintptr_t)k.tcw | (uintptr_t)k.seed0 | (uintptr_t)k.alpha_share |
                            (uintptr_t)(KIND == 1 ? ((uintptr_t)k.sigma_cw | (uintptr_t)k.leaf_cw)
                                                  : (uintptr_t)k.cw_final);
    if (bases & 15) return false;
    const int lnb = KIND == 1 ? FSSB_ARNK_TMA_LNB_CMP : FSSB_ARNK_TMA_LNB_EQ;
    const uint32_t E = 16u << lnb;
    PackMaps M;
    memset(&M, 0, sizeof(M));
    bool ok = encode_map(&M.scw, CU_TENSOR_MAP_DATA_TYPE_UINT32, k.scw, 4 * count, n, 16 * ld, 4 * E) &&
              encode_map(&M.tcw, CU_TENSOR_MAP_DATA_TYPE_UINT8, k.tcw, count, n, ld, E) &&
              encode_map(&M.alpha, CU_TENSOR_MAP_DATA_TYPE_UINT64, k.alpha_share, count, 0, 8, E) &&
              encode_map(&M.seed, CU_TENSOR_MAP_DATA_TYPE_UINT32, k.seed0, 4 * count, 0, 16, 4 * E);
    if (KIND == 1)
        ok = ok && encode_map(&M.sig, CU_TENSOR_MAP_DATA_TYPE_UINT64, k.sigma_cw, count, n, 8 * ld, E) &&
             encode_map(&M.leaf, CU_TENSOR_MAP_DATA_TYPE_UINT64, k.leaf_cw, count, n + 1, 8 * ld, E);
    else
        ok = ok && encode_map(&M.cwf, CU_TENSOR_MAP_DATA_TYPE_UINT64, k.cw_final, count, 0, 8, E);
    if (!ok) return false;
    const uint32_t stride = (uint32_t)((elem_bytes(KIND, n) * E + 16 + 127) / 128 * 128);
    const uint32_t sstride = stage_layout(KIND, n, E).bytes;
    constexpr int kStages = KIND == 1 ? FSSB_ARNK_TMA_STAGES_CMP : FSSB_ARNK_TMA_STAGES_EQ;
    const size_t smem = 128 + 2 * (size_t)stride + kStages * (size_t)sstride;
    if (smem > 220 * 1024) return false;
    constexpr int kThr = FSSB_ARNK_TMA_THREADS;
    auto kern = arnk_pack_tma_kernel<KIND, W, kThr, kStages>;
    int dev = 0, sms = 0, per_sm = 1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThr, smem);
    if (e == cudaSuccess) {
        const uint64_t tiles = (count + E - 1) / E;
        const uint64_t cap = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
        static const int use_tma = getenv("FSSB_ARNK_NO_TMA") ? 0 : 1;
        kern<<<(unsigned)(tiles < cap ? tiles : cap), kThr, smem, st>>>(M, n, count, lnb, stride, sstride, use_tma,
                                                                         buf);
        e = cudaGetLastError();
    }
    *err = e;
    return true;
}

template <bool PACK, int KIND, int W>
cudaError_t launch_tile(int n, uint64_t count, uint64_t ld, Keys k, uint8_t* buf, cudaStream_t st) {
    // cp.async needs naturally aligned pieces: tcw rows 4-byte aligned, scw /
    // seed rows 16-byte aligned (sigma / leaf pick 16 or 8 in the kernel)
    if (PACK) {
        cudaError_t e = cudaSuccess;
        if (try_pack_tma<KIND, W>(n, count, ld, k, buf, st, &e)) return e;
    }
    if (PACK && FSSB_ARNK_ASYNC_PACK && ld % 4 == 0 && !((uintptr_t)k.tcw & 3) &&
        !(((uintptr_t)k.scw | (uintptr_t)k.seed0) & 15) && !((uintptr_t)k.alpha_share & 7) &&
        2 * (elem_bytes(KIND, n) * 16 + 144) + 2 * stage_layout(KIND, n, 16).bytes <= 220 * 1024)
        return launch_pack_async<KIND, W>(n, count, ld, k, buf, st);
    const int lnb = arnk_tile_lnb(PACK, KIND, n);
    const uint32_t E = 16u << lnb;
    // per buffer: the tile + 16 bytes of slack for the covering word reads,
    // rounded to 128 bytes; plus 128 bytes for the two mbarriers
    const uint32_t stride = (uint32_t)((elem_bytes(KIND, n) * E + 16 + 127) / 128 * 128);
    const size_t smem = 128 + 2 * (size_t)stride;
    int dev = 0, sms = 0, per_sm = 1;
    constexpr int kThr = PACK ? kArnkThreads : FSSB_ARNK_UNPACK_THREADS;
    auto kern = arnk_tile_kernel<PACK, KIND, W, kThr>;
    cudaError_t err = cudaGetDevice(&dev);
    if (err == cudaSuccess) err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err == cudaSuccess) err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err == cudaSuccess) err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThr, smem);
    if (err != cudaSuccess) return err;
    const uint64_t tiles = (count + E - 1) / E;
    const uint64_t cap = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
    // FSSB_ARNK_NO_TMA=1 (environment): cooperative copies instead of the bulk
    // engine -- for compute-sanitizer initcheck, which does not see TMA writes
    static const int use_tma = getenv("FSSB_ARNK_NO_TMA") ? 0 : 1;
    kern<<<(unsigned)(tiles < cap ? tiles : cap), kThr, smem, st>>>(n, count, ld, lnb, stride, use_tma,
                                                                           k, buf);
    return cudaGetLastError();
}

template <bool PACK, int KIND>
cudaError_t launch_kind(int n, uint64_t count, uint64_t ld, Keys k, uint8_t* buf, cudaStream_t st) {
    switch ((n + 7) / 8) {
        case 1: return launch_tile<PACK, KIND, 1>(n, count, ld, k, buf, st);
        case 2: return launch_tile<PACK, KIND, 2>(n, count, ld, k, buf, st);
        case 3: return launch_tile<PACK, KIND, 3>(n, count, ld, k, buf, st);
        case 4: return launch_tile<PACK, KIND, 4>(n, count, ld, k, buf, st);
        case 5: return launch_tile<PACK, KIND, 5>(n, count, ld, k, buf, st);
        case 6: return launch_tile<PACK, KIND, 6>(n, count, ld, k, buf, st);
        case 7: return launch_tile<PACK, KIND, 7>(n, count, ld, k, buf, st);
        default: return launch_tile<PACK, KIND, 8>(n, count, ld, k, buf, st);
    }
}

int launch(bool pack, int kind, int n, uint64_t count, uint64_t ld, Keys k, uint8_t* buf, void* stream) {
    if ((kind != 0 && kind != 1) || n < 1 || n > 64 || (kind == 1 && n > 63))
        return fssb::set_error(FSS_EINVAL, "ARNK: bad kind or n");
    if (ld < count) return fssb::set_error(FSS_EINVAL, "ARNK: level stride ld < count");
    if (count == 0) return FSS_OK;
    if (!buf || !k.alpha_share || !k.seed0 || !k.scw || !k.tcw ||
        (kind == 0 ? !k.cw_final : (!k.sigma_cw || !k.leaf_cw)))
        return fssb::set_error(FSS_EINVAL, "ARNK: null device pointer");
    cudaStream_t st = (cudaStream_t)stream;
#if FSSB_ARNK_NAIVE
    const int bs = 256;
    dim3 grid((unsigned)((count + bs - 1) / bs), kind == 0 ? n + 1 : n + 2);
    if (pack)
        arnk_kernel<true><<<grid, bs, 0, st>>>(kind, n, count, ld, k, buf);
    else
        arnk_kernel<false><<<grid, bs, 0, st>>>(kind, n, count, ld, k, buf);
    const cudaError_t err = cudaGetLastError();
#else
    const cudaError_t err = pack ? (kind ? launch_kind<true, 1>(n, count, ld, k, buf, st)
                                         : launch_kind<true, 0>(n, count, ld, k, buf, st))
                                 : (kind ? launch_kind<false, 1>(n, count, ld, k, buf, st)
                                         : launch_kind<false, 0>(n, count, ld, k, buf, st));
#endif
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

int fss_arnk_unpack(int kind, int n, uint64_t count, uint64_t ld, const uint8_t* payload,
                    uint64_t* alpha_share, uint8_t* seed0, uint8_t* scw, uint8_t* tcw,
                    uint64_t* cw_final, uint64_t* sigma_cw, uint64_t* leaf_cw, void* stream) {
    Keys k{alpha_share, seed0, scw, tcw, cw_final, sigma_cw, leaf_cw};
    return launch(false, kind, n, count, ld, k, const_cast<uint8_t*>(payload), stream);
}

}  // extern "C"
