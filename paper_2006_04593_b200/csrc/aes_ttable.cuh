// AES-128 (fixed MMO keys) on sm_100a: T-tables in shared memory, one lane
// replica per bank so every lookup of a warp is bank-conflict free.
//
// Shared-memory layout (128 KiB, one CTA per SM):
//   byte address = region*64K + x*256 + tsel*128 + lane*4,   x = table index byte
//   region 0 holds Te0 (tsel 0) and Te1 (tsel 1), region 1 holds Te2 / Te3,
//   Te_j[x] = rotl(Te0[x], 8j).
// Lane l always hits bank l, so a warp's 32 random lookups cost one wavefront.
// The address of a lookup is ONE PRMT: byte k of the state column goes to
// address byte 1, the lane/table offset (lo0 = 4*lane, lo1 = 4*lane + 128) to
// address byte 0, and zero bytes of lo* fill bytes 2..3.
//
// Round keys of the three fixed cipher keys (reference prg.py:24-28) are
// compile-time constants (aes_consts.h), so AddRoundKey folds into LOP3
// immediates. For the tree walk the key of the selected child block depends on
// a per-element input bit; a per-thread mask m (0 or ~0) selects
// rk = RK1 ^ (m & (RK1 ^ RK2)) -- one extra LOP3 per column.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "aes_consts.h"

#ifndef FSSB_IMAD_ADDR
#define FSSB_IMAD_ADDR 0
#endif

namespace fssb {

#if FSSB_IMAD_ADDR
// Multipliers read from the constant bank so ptxas cannot strength-reduce the
// IMADs below into ALU shifts: the address arithmetic of table bytes 0 and 3
// runs on the (otherwise idle) FMA pipe instead of the ALU pipe.
static __constant__ uint32_t kAddrMul[3] = {1u << 24, 1u << 16, 1u << 8};
#endif

constexpr int kTableWords = 32768;            // 4 tables x 256 entries x 32 lanes
constexpr int kTableBytes = kTableWords * 4;  // 128 KiB dynamic shared memory
constexpr uint32_t kRegion1 = 65536;

struct U4 {
    uint32_t x, y, z, w;
};

// Fill the replicated tables (once per CTA; kernels are persistent).
__device__ __forceinline__ void fill_tables(uint32_t* tab) {
    for (int idx = threadIdx.x; idx < kTableWords; idx += blockDim.x) {
        const int tsel = (idx >> 5) & 1;
        const int x = (idx >> 6) & 255;
        const int region = idx >> 14;
        const uint32_t v = kTe0[x];
        tab[idx] = __funnelshift_l(v, v, 8 * (2 * region + tsel));
    }
}

// The replicated tables are the same bytes for every CTA of every kernel, so
// they are built ONCE per device into a global image (table_image_upload, at
// the first launch on the device) and each CTA pulls its copy with four TMA
// bulk copies (cp.async.bulk, 32 KiB each, completion on an mbarrier) instead
// of computing 32768 words with its own threads: ~1 us from L2 whatever the
// thread count, where the computed fill took up to tens of us for the
// small-thread-count launches of small batches.
#ifndef FSSB_TMA_TABLES
#define FSSB_TMA_TABLES 1
#endif
// (static: one image per translation unit; fss_kernels.cu is the only unit
// that launches table kernels, and its prep_launch uploads its image)
static __device__ __align__(128) uint32_t g_tab_img[kTableWords];

__device__ __forceinline__ void load_tables(uint32_t* tab) {
#if FSSB_TMA_TABLES
    __shared__ __align__(8) uint64_t bar;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kTableBytes)
                     : "memory");
#pragma unroll
        for (int c = 0; c < 4; c++)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    (uint32_t)__cvta_generic_to_shared(tab + c * (kTableWords / 4))),
                "l"(g_tab_img + c * (kTableWords / 4)), "r"(kTableBytes / 4), "r"(b)
                : "memory");
    }
    __syncthreads();   // the barrier is initialised before anyone waits on it
    asm volatile(
        "{\n .reg .pred p;\n TAB_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        " @!p bra TAB_WAIT_%=;\n}" ::"r"(b)
        : "memory");
#else
    fill_tables(tab);
    __syncthreads();
#endif
}

// Host side: build the image from kTe0 and upload it to the current device
// (synchronous; once per device, before the first table-using launch).
inline cudaError_t table_image_upload() {
    static thread_local uint32_t te0[256];
    cudaError_t err = cudaMemcpyFromSymbol(te0, kTe0, sizeof(te0));
    if (err != cudaSuccess) return err;
    uint32_t* img = new uint32_t[kTableWords];
    for (int idx = 0; idx < kTableWords; idx++) {
        const int tsel = (idx >> 5) & 1, x = (idx >> 6) & 255, region = idx >> 14;
        const uint32_t v = te0[x];
        const int r = 8 * (2 * region + tsel);
        img[idx] = r ? (v << r) | (v >> (32 - r)) : v;
    }
    err = cudaMemcpyToSymbol(g_tab_img, img, sizeof(uint32_t) * kTableWords);
    delete[] img;
    // From pageable memory the copy returns once the bytes are staged, not
    // when they reach HBM, and the legacy stream it ran on does not order the
    // party / torch streams (non-blocking): wait for it before any kernel that
    // pulls the image can be launched.
    if (err == cudaSuccess) err = cudaStreamSynchronize(cudaStreamLegacy);
    return err;
}

struct Tab {
    const unsigned char* base;  // shared-memory table base
    uint32_t lo0, lo1;          // 4*lane and 4*lane+128
};

__device__ __forceinline__ Tab make_tab(const uint32_t* tab) {
    Tab t;
    t.base = reinterpret_cast<const unsigned char*>(tab);
    const uint32_t lane = threadIdx.x & 31;
    t.lo0 = lane * 4;
    t.lo1 = lane * 4 + 128;
    return t;
}

// Table J (0..3) looked up at byte K (0..3) of column c.
template <int J, int K>
__device__ __forceinline__ uint32_t T(const Tab& tb, uint32_t c) {
    const uint32_t lo = (J & 1) ? tb.lo1 : tb.lo0;
    uint32_t addr;
#if FSSB_IMAD_ADDR
    // FSSB_IMAD_ADDR: 1 = bytes 0 and 3 on the FMA pipe, 2 = byte 0 only, 3 = byte 3 only
    if (K == 0 && FSSB_IMAD_ADDR != 3) {   // addr = ((c << 24) * 2^16) >> 32 + lo = byte0 << 8 | lo
        uint32_t t;
        asm("mul.lo.u32 %0, %1, %2;" : "=r"(t) : "r"(c), "r"(kAddrMul[0]));
        asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(addr) : "r"(t), "r"(kAddrMul[1]), "r"(lo));
    } else if (K == 3 && FSSB_IMAD_ADDR != 2) {  // addr = (c * 2^8) >> 32 = byte3, then * 2^8 + lo
        uint32_t t;
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(t) : "r"(c), "r"(kAddrMul[2]));
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(addr) : "r"(t), "r"(kAddrMul[2]), "r"(lo));
    } else
#endif
    {
        addr = __byte_perm(c, lo, 0x5504 + 0x10 * K);
    }
    return *reinterpret_cast<const uint32_t*>(tb.base + (J >> 1) * kRegion1 + addr);
}

// Round-key word w for a fixed key KEY (0..2), or for the key selected per
// element between KEY=0 (k1, m=0) and KEY=1 (k2, m=~0) when SEL.
template <int KEY, bool SEL>
__device__ __forceinline__ uint32_t rk(int w, uint32_t m) {
    if (SEL) return kRK[0][w] ^ (m & (kRK[0][w] ^ kRK[1][w]));
    return kRK[KEY][w];
}

#ifndef FSSB_LOP3_COMBINE
#define FSSB_LOP3_COMBINE 1
#endif

__device__ __forceinline__ uint32_t lop3_xor3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ uint32_t lop3_xor_and(uint32_t a, uint32_t b, uint32_t c) {  // a ^ (b & c)
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// Column mix of one round: t0 ^ t1 ^ t2 ^ t3 ^ rk. For a per-element selected
// key, rk = RK1 ^ (m & (RK1 ^ RK2)); written as three explicit LOP3s
// ((t0^t1^t2), (^t3^RK1), (^(m&D))) -- left to itself the compiler emits four.
template <int KEY, bool SEL>
__device__ __forceinline__ uint32_t mixcol(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3, int w,
                                           uint32_t m) {
#if FSSB_LOP3_COMBINE
    if (SEL) {
        const uint32_t x = lop3_xor3(t0, t1, t2);
        const uint32_t y = lop3_xor3(x, t3, kRK[0][w]);
        return lop3_xor_and(y, m, kRK[0][w] ^ kRK[1][w]);
    }
#endif
    return t0 ^ t1 ^ t2 ^ t3 ^ rk<KEY, SEL>(w, m);
}

// Rounds 0..9 of AES-128 on (c0..c3) (little-endian column words), in place.
template <int KEY, bool SEL>
__device__ __forceinline__ void aes128_rounds(const Tab& tb, uint32_t& c0, uint32_t& c1, uint32_t& c2,
                                              uint32_t& c3, uint32_t m) {
    c0 ^= rk<KEY, SEL>(0, m);
    c1 ^= rk<KEY, SEL>(1, m);
    c2 ^= rk<KEY, SEL>(2, m);
    c3 ^= rk<KEY, SEL>(3, m);
#pragma unroll
    for (int r = 1; r < 10; r++) {
        const uint32_t n0 = mixcol<KEY, SEL>(T<0, 0>(tb, c0), T<1, 1>(tb, c1), T<2, 2>(tb, c2),
                                             T<3, 3>(tb, c3), 4 * r + 0, m);
        const uint32_t n1 = mixcol<KEY, SEL>(T<0, 0>(tb, c1), T<1, 1>(tb, c2), T<2, 2>(tb, c3),
                                             T<3, 3>(tb, c0), 4 * r + 1, m);
        const uint32_t n2 = mixcol<KEY, SEL>(T<0, 0>(tb, c2), T<1, 1>(tb, c3), T<2, 2>(tb, c0),
                                             T<3, 3>(tb, c1), 4 * r + 2, m);
        const uint32_t n3 = mixcol<KEY, SEL>(T<0, 0>(tb, c3), T<1, 1>(tb, c0), T<2, 2>(tb, c1),
                                             T<3, 3>(tb, c2), 4 * r + 3, m);
        c0 = n0;
        c1 = n1;
        c2 = n2;
        c3 = n3;
    }
}

// Last round (SubBytes + ShiftRows, no MixColumns) of output column c, whose
// bytes come from columns (a, b, c, d) = (c, c+1, c+2, c+3): S(x) sits in
// byte r of Te_{(r+2)&3}[x], so four lookups and three PRMTs build the word.
__device__ __forceinline__ uint32_t last_col(const Tab& tb, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
    return __byte_perm(__byte_perm(T<2, 0>(tb, a), T<3, 1>(tb, b), 0x3250),
                       __byte_perm(T<0, 2>(tb, c), T<1, 3>(tb, d), 0x7210), 0x7610);
}

// One full AES-128 encryption of (c0..c3) (little-endian column words).
template <int KEY, bool SEL>
__device__ __forceinline__ U4 aes128(const Tab& tb, U4 s, uint32_t m) {
    uint32_t c0 = s.x, c1 = s.y, c2 = s.z, c3 = s.w;
    aes128_rounds<KEY, SEL>(tb, c0, c1, c2, c3, m);
    U4 o;
    o.x = last_col(tb, c0, c1, c2, c3) ^ rk<KEY, SEL>(40, m);
    o.y = last_col(tb, c1, c2, c3, c0) ^ rk<KEY, SEL>(41, m);
    o.z = last_col(tb, c2, c3, c0, c1) ^ rk<KEY, SEL>(42, m);
    o.w = last_col(tb, c3, c0, c1, c2) ^ rk<KEY, SEL>(43, m);
    return o;
}

// MMO block AES_KEY(s) ^ s, but only its 8-byte half `h` (0: bytes 0..7,
// 1: bytes 8..15; hm = 0 - h). The last round then needs 8 of the 16 lookups:
// DCF evaluation reads only the sigma/tau lane x_i of the third block
// (slice_cmp, prg.py:99-119), so this is exact. Returns (lo, hi) words.
// TOP_HI: the caller uses only bit 31 of `hi` (the tau bit; sigma mod 2^w with
// w <= 32 lives in `lo`), so the high word's last round is the one lookup that
// yields its top byte: 5 last-round lookups instead of 8. The other bits of
// `hi` are then not the block's.
template <int KEY, bool TOP_HI = false>
__device__ __forceinline__ void mmo_half(const Tab& tb, U4 s, uint32_t hm, uint32_t& lo,
                                         uint32_t& hi) {
    uint32_t c0 = s.x, c1 = s.y, c2 = s.z, c3 = s.w;
    aes128_rounds<KEY, false>(tb, c0, c1, c2, c3, 0);
    // rotate the columns by 2*h: output columns (2h, 2h+1) = last_col of (a0..a3), (a1..a0)
    const uint32_t a0 = hm ? c2 : c0, a1 = hm ? c3 : c1, a2 = hm ? c0 : c2, a3 = hm ? c1 : c3;
    const uint32_t k_lo = kRK[KEY][40] ^ (hm & (kRK[KEY][40] ^ kRK[KEY][42]));
    const uint32_t k_hi = kRK[KEY][41] ^ (hm & (kRK[KEY][41] ^ kRK[KEY][43]));
    const uint32_t s_lo = hm ? s.z : s.x, s_hi = hm ? s.w : s.y;
    lo = lop3_xor3(last_col(tb, a0, a1, a2, a3), k_lo, s_lo);
    // byte 3 of last_col(a1, a2, a3, a0) is byte 3 of T<1,3>(a0): S(a0.b3)
    hi = TOP_HI ? lop3_xor3(T<1, 3>(tb, a0), k_hi, s_hi)
                : lop3_xor3(last_col(tb, a1, a2, a3, a0), k_hi, s_hi);
}

// MMO block AES_KEY(s) ^ s for DCF keygen's sigma/tau block at out_bits <= 32:
// the correction words read sigma_L / sigma_R mod 2^w (words x and z) and the
// tau bits (bit 31 of words y and w), so words y and w get only the last-round
// lookup of their top byte -- 10 of the 16 last-round lookups. Bits 0..30 of
// y and w are then not the block's.
template <int KEY>
__device__ __forceinline__ U4 mmo_sigma_tau32(const Tab& tb, U4 s) {
    uint32_t c0 = s.x, c1 = s.y, c2 = s.z, c3 = s.w;
    aes128_rounds<KEY, false>(tb, c0, c1, c2, c3, 0);
    U4 o;
    o.x = lop3_xor3(last_col(tb, c0, c1, c2, c3), kRK[KEY][40], s.x);
    o.y = lop3_xor3(T<1, 3>(tb, c0), kRK[KEY][41], s.y);   // byte 3 of last_col(c1, c2, c3, c0)
    o.z = lop3_xor3(last_col(tb, c2, c3, c0, c1), kRK[KEY][42], s.z);
    o.w = lop3_xor3(T<1, 3>(tb, c2), kRK[KEY][43], s.w);   // byte 3 of last_col(c3, c0, c1, c2)
    return o;
}

// Matyas-Meyer-Oseas block: AES_k(s) XOR s  (reference prg.expand, prg.py:43-60).
template <int KEY, bool SEL>
__device__ __forceinline__ U4 mmo(const Tab& tb, U4 s, uint32_t m) {
    U4 o = aes128<KEY, SEL>(tb, s, m);
    o.x ^= s.x;
    o.y ^= s.y;
    o.z ^= s.z;
    o.w ^= s.w;
    return o;
}

}  // namespace fssb
