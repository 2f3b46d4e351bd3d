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
    if (K == 0) {         // addr = ((c << 24) * 2^16) >> 32 + lo = byte0 << 8 | lo
        uint32_t t;
        asm("mul.lo.u32 %0, %1, %2;" : "=r"(t) : "r"(c), "r"(kAddrMul[0]));
        asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(addr) : "r"(t), "r"(kAddrMul[1]), "r"(lo));
    } else if (K == 3) {  // addr = (c * 2^8) >> 32 = byte3, then * 2^8 + lo
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
template <int KEY>
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
    hi = lop3_xor3(last_col(tb, a1, a2, a3, a0), k_hi, s_hi);
}

// ---- per-lane key among all three fixed keys (lane-pair evaluation) ----
// rk = RK1 ^ (ma & (RK1 ^ RK2)) ^ (mb & (RK1 ^ RK3)): ma selects k2, mb selects
// k3 (never both). Lanes of one warp then run ONE instruction stream while
// encrypting under different keys -- one more LOP3 per column than SEL.
__device__ __forceinline__ uint32_t rk3(int w, uint32_t ma, uint32_t mb) {
    return lop3_xor_and(lop3_xor_and(kRK[0][w], ma, kRK[0][w] ^ kRK[1][w]), mb, kRK[0][w] ^ kRK[2][w]);
}

__device__ __forceinline__ U4 mmo3(const Tab& tb, U4 s, uint32_t ma, uint32_t mb) {
    uint32_t c0 = s.x ^ rk3(0, ma, mb), c1 = s.y ^ rk3(1, ma, mb);
    uint32_t c2 = s.z ^ rk3(2, ma, mb), c3 = s.w ^ rk3(3, ma, mb);
#pragma unroll
    for (int r = 1; r < 10; r++) {
#define FSSB_MIX3(A, B, C, D, W)                                                                   \
    lop3_xor_and(lop3_xor_and(lop3_xor3(lop3_xor3(T<0, 0>(tb, A), T<1, 1>(tb, B), T<2, 2>(tb, C)),  \
                                        T<3, 3>(tb, D), kRK[0][W]),                                 \
                              ma, kRK[0][W] ^ kRK[1][W]),                                           \
                 mb, kRK[0][W] ^ kRK[2][W])
        const uint32_t n0 = FSSB_MIX3(c0, c1, c2, c3, 4 * r + 0);
        const uint32_t n1 = FSSB_MIX3(c1, c2, c3, c0, 4 * r + 1);
        const uint32_t n2 = FSSB_MIX3(c2, c3, c0, c1, 4 * r + 2);
        const uint32_t n3 = FSSB_MIX3(c3, c0, c1, c2, 4 * r + 3);
#undef FSSB_MIX3
        c0 = n0;
        c1 = n1;
        c2 = n2;
        c3 = n3;
    }
    U4 o;
    o.x = lop3_xor3(last_col(tb, c0, c1, c2, c3), rk3(40, ma, mb), s.x);
    o.y = lop3_xor3(last_col(tb, c1, c2, c3, c0), rk3(41, ma, mb), s.y);
    o.z = lop3_xor3(last_col(tb, c2, c3, c0, c1), rk3(42, ma, mb), s.z);
    o.w = lop3_xor3(last_col(tb, c3, c0, c1, c2), rk3(43, ma, mb), s.w);
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
