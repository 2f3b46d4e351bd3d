// B200 (sm_100a) kernels for AriaNN's FSS hot path and the C-ABI that exposes
// them (declared in include/ariann_fss.h).
//
// One thread walks the n tree levels of one element; seed / control bits stay
// in registers. Correction words are stored level-major (struct of arrays,
// exactly the reference's in-memory layout, fss.py:71-154), so at every level
// a warp reads 32 consecutive 16-byte scw words (512 B, one coalesced LDG.128
// per lane) plus 8-byte sigma/leaf words. Grids are persistent: one CTA per SM
// (the 128 KiB T-tables limit residency to one CTA; 1024 threads for eval, 512
// for keygen), each CTA striding through its own contiguous run of elements
// (cta_span).
//
// Evaluation computes only the AES blocks the output depends on: the block of
// the child selected by the public input bit (key k1 or k2 chosen per element)
// and, for comparison, the sigma/tau block (k3). The reference expands 2 (eq)
// or 3 (cmp) blocks per level (fss.py:365, 395); the outputs are identical.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <omp.h>

#include <initializer_list>
#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/ariann_fss.h"
#include "aes_ttable.cuh"
#include "common.cuh"

using fssb::U4;

namespace {

// Software-pipelined correction-word loads (level i+1 loads during level i's
// AES): +0.7 % for DCF eval at 1024 threads, -1.4 % for DPF eval
// (profiles/r01_aes_variants_c.json), so on for DCF only.
#ifndef FSSB_PREFETCH_DCF
#define FSSB_PREFETCH_DCF 1   // levels ahead (0: no prefetch)
#endif
#ifndef FSSB_PREFETCH_DPF
#define FSSB_PREFETCH_DPF 0   // levels ahead (0: no prefetch)
#endif
#ifdef FSSB_PREFETCH
#undef FSSB_PREFETCH_DCF
#undef FSSB_PREFETCH_DPF
#define FSSB_PREFETCH_DCF FSSB_PREFETCH
#define FSSB_PREFETCH_DPF FSSB_PREFETCH
#endif
#ifndef FSSB_W32
#define FSSB_W32 1
#endif
#ifndef FSSB_THREADS
#define FSSB_THREADS 1024
#endif
// Keygen through the lane-pair kernel (keygen_pair_kernel): DCF at every
// size (1024 threads x 64 registers beat 512 x 128 even at 2^22: -0.7 %, and
// -12 % at 2^16), DPF not (+2.4 % at 2^22; scripts/small_batch_probe.py,
// profiles/r02_small_batch.json).
#ifndef FSSB_KEYGEN_PAIR_DCF
#define FSSB_KEYGEN_PAIR_DCF 1
#endif
#ifndef FSSB_KEYGEN_PAIR_DPF
#define FSSB_KEYGEN_PAIR_DPF 0
#endif
// Eval kernels: 32 warps per SM (64 registers) hide the LDS / LDG latency best
// (profiles/r01_aes_variants_b.json: 512 -> 1024 threads = +5 % DCF, +17 % DPF).
constexpr int kThreads = FSSB_THREADS;
constexpr int kPfDcf = FSSB_PREFETCH_DCF;
constexpr int kPfDpf = FSSB_PREFETCH_DPF;
struct DpfCw {
    U4 s;
    uint32_t f;
};
// One level's DCF correction words as one thread reads them.
template <typename W>
struct DcfCw {
    U4 s;          // seed correction
    uint32_t f;    // tL, tR, tauL, tauR bits
    W sig, leaf;
};
// Keygen kernels need ~100-127 registers: 16 warps per SM.
constexpr int kKeygenThreads = 512;

__device__ __forceinline__ uint64_t ring_mask(int w) { return w >= 64 ? ~0ULL : ((1ULL << w) - 1); }

__device__ __forceinline__ U4 ld16(const uint8_t* p) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    return U4{v.x, v.y, v.z, v.w};
}

__device__ __forceinline__ void st16(uint8_t* p, U4 v) {
    *reinterpret_cast<uint4*>(p) = make_uint4(v.x, v.y, v.z, v.w);
}

__device__ __forceinline__ uint64_t lo64(U4 v) { return (uint64_t)v.x | ((uint64_t)v.y << 32); }
__device__ __forceinline__ uint64_t hi64(U4 v) { return (uint64_t)v.z | ((uint64_t)v.w << 32); }

__device__ __forceinline__ U4 xor4(U4 a, U4 b) { return U4{a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w}; }
__device__ __forceinline__ U4 and4(U4 a, uint32_t m) { return U4{a.x & m, a.y & m, a.z & m, a.w & m}; }
__device__ __forceinline__ U4 sel4(bool c, U4 a, U4 b) {
    return U4{c ? a.x : b.x, c ? a.y : b.y, c ? a.z : b.z, c ? a.w : b.w};
}

// Persistent grids: CTA b owns a contiguous run of whole 32-element warp tiles
// (runs balanced to within one tile) and its threads stride through the run.
// Unlike a grid-wide stride, the final partial pass is then spread evenly over
// all SMs instead of landing on the first CTAs while the last ones idle.
struct Span {
    uint64_t lo, hi;
};

__device__ __forceinline__ Span cta_span(uint64_t count) {
    const uint64_t tiles = (count + 31) / 32;
    const uint64_t t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
    Span sp;
    sp.lo = 32 * t0;
    sp.hi = 32 * t1 < count ? 32 * t1 : count;
    return sp;
}

// ------------------------------------------------------------------ expand
// prg.expand (prg.py:43-60): out block b = AES_{k_b}(seed) ^ seed.
__global__ void __launch_bounds__(kKeygenThreads, 1)
expand_kernel(const uint8_t* __restrict__ seeds, uint64_t count, int blocks, uint8_t* __restrict__ out) {
    extern __shared__ __align__(128) uint32_t tab[];
    fssb::load_tables(tab);
    const fssb::Tab tb = fssb::make_tab(tab);
    const Span sp = cta_span(count);
    for (uint64_t e = sp.lo + threadIdx.x; e < sp.hi; e += blockDim.x) {
        const U4 s = ld16(seeds + 16 * e);
        uint8_t* o = out + e * 16 * blocks;
        st16(o, fssb::mmo<0, false>(tb, s, 0));
        st16(o + 16, fssb::mmo<1, false>(tb, s, 0));
        if (blocks == 3) st16(o + 32, fssb::mmo<2, false>(tb, s, 0));
    }
}

// Public input of element e: x[e], or -- fused with the one online round of
// sign/eq_protocol (sharing.mask_and_reveal, sharing.py:214-230) -- the opening
// m_own[e] + m_peer[e] of the two parties' wire-packed masked messages.
__device__ __forceinline__ uint64_t load_x(const uint64_t* __restrict__ x, const void* __restrict__ m_own,
                                           const void* __restrict__ m_peer, int n, uint64_t e) {
    if (x) return x[e];
    const int wb = fssb::wire_bytes(n);
    return fssb::wire_get(wb, m_own, e) + fssb::wire_get(wb, m_peer, e);
}

// ------------------------------------------------------------- mask stream
// prg.mask_stream (prg.py:128-147): counter-mode use of G. Block i is the seed
// XOR (round_idx LE in bytes 0..7, i LE in bytes 8..15) with the top bit of
// byte 15 re-cleared; G(block) = AES_k1 ^ . || AES_k2 ^ . gives 4 u64 lanes =
// ring elements 4i .. 4i+3.
__global__ void __launch_bounds__(kKeygenThreads, 1)
mask_stream_kernel(U4 seed, uint64_t round_idx, uint64_t blocks, uint64_t count, uint64_t mask,
                   uint64_t* __restrict__ out) {
    extern __shared__ __align__(128) uint32_t tab[];
    fssb::load_tables(tab);
    const fssb::Tab tb = fssb::make_tab(tab);
    const Span sp = cta_span(blocks);
    for (uint64_t i = sp.lo + threadIdx.x; i < sp.hi; i += blockDim.x) {
        U4 b = U4{seed.x ^ (uint32_t)round_idx, seed.y ^ (uint32_t)(round_idx >> 32),
                  seed.z ^ (uint32_t)i, seed.w ^ (uint32_t)(i >> 32)};
        b.w &= 0x7FFFFFFFu;
        const U4 l = fssb::mmo<0, false>(tb, b, 0), r = fssb::mmo<1, false>(tb, b, 0);
        const uint64_t lanes[4] = {lo64(l), hi64(l), lo64(r), hi64(r)};
#pragma unroll
        for (int j = 0; j < 4; j++)
            if (4 * i + j < count) out[4 * i + j] = lanes[j] & mask;
    }
}

// ---------------------------------------------------------------- DPF eval
// fss.eval_eq (fss.py:357-377): t0 = party, per level expand, correct with
// scw/tcw when t, descend to child x_i (MSB first); out = t*cw_final + s2r(s).
//
__global__ void __launch_bounds__(kThreads, 1)
dpf_eval_kernel(int party, int n, uint64_t count, uint64_t ld, const uint8_t* __restrict__ seed0,
                const uint8_t* __restrict__ scw, const uint8_t* __restrict__ tcw,
                const uint64_t* __restrict__ cw_final, const uint64_t* __restrict__ x,
                const void* __restrict__ m_own, const void* __restrict__ m_peer,
                uint64_t* __restrict__ out) {
    extern __shared__ __align__(128) uint32_t tab[];
    fssb::load_tables(tab);
    const fssb::Tab tb = fssb::make_tab(tab);
    const uint64_t mask = ring_mask(n);
    const Span sp = cta_span(count);
    for (uint64_t e = sp.lo + threadIdx.x; e < sp.hi; e += blockDim.x) {
        U4 s = ld16(seed0 + 16 * e);
        uint32_t t = party;
        const uint64_t xe = load_x(x, m_own, m_peer, n, e) & mask;
        auto cw_at = [&](int i) {
            const uint64_t off = (uint64_t)(i < n ? i : n - 1) * ld + e;
            return DpfCw{ld16(scw + 16 * off), __ldg(tcw + off)};
        };
        // kPfDpf levels of correction words in flight (see dcf_eval_kernel)
        DpfCw ring[kPfDpf > 0 ? kPfDpf : 1];
#pragma unroll
        for (int j = 0; j < kPfDpf; j++) ring[j] = cw_at(j);
        for (int i = 0; i < n; i++) {
            DpfCw c;
            if (kPfDpf > 0) {
                c = ring[0];
#pragma unroll
                for (int j = 0; j + 1 < kPfDpf; j++) ring[j] = ring[j + 1];
                ring[kPfDpf > 0 ? kPfDpf - 1 : 0] = cw_at(i + kPfDpf);
            } else {
                c = cw_at(i);
            }
            const uint32_t xb = (uint32_t)(xe >> (n - 1 - i)) & 1u;
            const U4 a = fssb::mmo<0, true>(tb, s, 0u - xb);
            const uint32_t tm = 0u - t;
            s = xor4(a, and4(c.s, tm));
            const uint32_t tn = ((a.w >> 31) ^ (t & (c.f >> xb))) & 1u;
            s.w &= 0x7FFFFFFFu;
            t = tn;
        }
        uint64_t o = (((uint64_t)t * cw_final[e]) + lo64(s)) & mask;
        if (party) o = (0 - o) & mask;
        out[e] = o;
    }
}

// ---------------------------------------------------------------- DCF eval
// fss.eval_cmp (fss.py:380-426). Per level: child block (key k1/k2 by x_i) and
// the sigma/tau block (k3, lane x_i). out_i = tau*leaf[i] + sigma (mod 2^w).
//
// Ring arithmetic is mod 2^w, so the running sum is reduced once at the end
// (per level only when the per-level outputs are requested). W32: for
// out_bits <= 32 (hence n <= 32) sigma, leaf and the sum live in 32-bit
// registers and only the low words of sigma_cw / leaf_cw are read (values
// < 2^w, little-endian), which removes the 64-bit glue from the ALU pipe.
#ifndef FSSB_DCF_UNROLL
#define FSSB_DCF_UNROLL 1
#endif
constexpr int kDcfUnroll = FSSB_DCF_UNROLL;   // level-loop unroll (variant sweep)
template <bool W32, bool LEVELS>
__global__ void __launch_bounds__(kThreads, 1)
dcf_eval_kernel(int party, int n, int out_bits, uint64_t count, uint64_t ld,
                const uint8_t* __restrict__ seed0, const uint8_t* __restrict__ scw,
                const uint8_t* __restrict__ tcw, const uint64_t* __restrict__ sigma_cw,
                const uint64_t* __restrict__ leaf_cw, const uint64_t* __restrict__ x,
                const void* __restrict__ m_own, const void* __restrict__ m_peer,
                uint64_t* __restrict__ out, uint64_t* __restrict__ levels) {
    using W = typename std::conditional<W32, uint32_t, uint64_t>::type;
    extern __shared__ __align__(128) uint32_t tab[];
    fssb::load_tables(tab);
    const fssb::Tab tb = fssb::make_tab(tab);
    const uint64_t nmask = ring_mask(n);
    const uint64_t mask = ring_mask(out_bits);
    const W* __restrict__ sig_w = reinterpret_cast<const W*>(sigma_cw);
    const W* __restrict__ leaf_w = reinterpret_cast<const W*>(leaf_cw);
    constexpr int kStride = W32 ? 2 : 1;   // W-words per u64 element
    const Span sp = cta_span(count);
    for (uint64_t e = sp.lo + threadIdx.x; e < sp.hi; e += blockDim.x) {
        U4 s = ld16(seed0 + 16 * e);
        uint32_t t = party;
        W acc = 0;
        const uint64_t xe = load_x(x, m_own, m_peer, n, e) & nmask;
        // correction words of level i (clamped to the last level, so the
        // prefetch ring never reads past the arrays)
        auto cw_at = [&](int i) {
            const uint64_t off = (uint64_t)(i < n ? i : n - 1) * ld + e;
            return DcfCw<W>{ld16(scw + 16 * off), __ldg(tcw + off), __ldg(sig_w + kStride * off),
                            __ldg(leaf_w + kStride * off)};
        };
        // software pipeline, kPfDcf levels deep: ptxas schedules a load late in
        // the iteration that issues it, so distance 1 covers only the tail of one
        // level's AES; distance 0 loads each level's words where they are used
        DcfCw<W> ring[kPfDcf > 0 ? kPfDcf : 1];
#pragma unroll
        for (int j = 0; j < kPfDcf; j++) ring[j] = cw_at(j);
#pragma unroll kDcfUnroll
        for (int i = 0; i < n; i++) {
            DcfCw<W> c;
            if (kPfDcf > 0) {
                c = ring[0];
#pragma unroll
                for (int j = 0; j + 1 < kPfDcf; j++) ring[j] = ring[j + 1];
                ring[kPfDcf > 0 ? kPfDcf - 1 : 0] = cw_at(i + kPfDcf);
            } else {
                c = cw_at(i);
            }
            const U4 cw = c.s;
            const uint32_t f = c.f;
            const W sig = c.sig, leaf = c.leaf;
            const uint32_t xb = (uint32_t)(xe >> (n - 1 - i)) & 1u;
            const uint32_t tm = 0u - t;
            // sigma/tau lane x_i of the third block (slice_cmp, prg.py:99-119):
            // only that 8-byte half of AES_k3(s) ^ s is computed
            uint32_t lane_lo, lane_hi;
            const U4 a = fssb::mmo<0, true>(tb, s, 0u - xb);
            // W32: sigma is lane_lo mod 2^w, and only the tau bit of lane_hi is read
            fssb::mmo_half<2, W32>(tb, s, 0u - xb, lane_lo, lane_hi);
            W lane;
            if (W32) lane = (W)lane_lo;
            else lane = (W)(((uint64_t)lane_hi << 32) | lane_lo);
            const uint32_t tau = ((lane_hi >> 31) ^ (t & (f >> (2 + xb)))) & 1u;
            const W sigma = lane ^ (sig & (W)(0 - (W)t));
            const W oi = (leaf & (W)(0 - (W)tau)) + sigma;
            acc += oi;
            if (LEVELS) levels[(uint64_t)i * count + e] = (party ? (0 - (uint64_t)oi) : (uint64_t)oi) & mask;
            s = xor4(a, and4(cw, tm));
            const uint32_t tn = ((a.w >> 31) ^ (t & (f >> xb))) & 1u;
            s.w &= 0x7FFFFFFFu;
            t = tn;
        }
        const uint64_t off = (uint64_t)n * ld + e;
        const W lo = W32 ? (W)s.x : (W)lo64(s);
        const W last = (__ldg(leaf_w + kStride * off) & (W)(0 - (W)t)) + lo;
        acc += last;
        if (LEVELS) levels[(uint64_t)n * count + e] = (party ? (0 - (uint64_t)last) : (uint64_t)last) & mask;
        out[e] = (party ? (0 - (uint64_t)acc) : (uint64_t)acc) & mask;
    }
}

// ------------------------------------------------ eval from ARNK payloads
// A party that receives its keys as an ARNK container (reference cli.py:150-160:
// read the file, unpack, evaluate once -- the keys are single-use) can
// evaluate straight from the element-major payload rows, skipping the unpack
// pass (fss_arnk_unpack) and the level-major copy entirely. Element e's record
// (LAYOUT.md:48-71) is read front to back by its own thread, one level record
// (scw 16 | flags 1 | sigma w) per level: lanes hit different lines, but each
// thread streams its own 824-byte record sequentially, so the L1 (what the
// T-tables leave of it) serves the rest of each sector and DRAM traffic stays
// at the payload bytes. Records sit at odd byte offsets: they are read as
// aligned 32-bit words and realigned with funnel shifts.

// The NB bytes at p (any alignment) as little-endian words o[0..(NB+3)/4),
// read with 16-byte loads: the lanes of a warp read 32 different records, so
// each load instruction costs ~32 L1 wavefronts whatever its width -- and the
// L1 data path is shared with the T-table lookups. Only the aligned 16-byte
// chunks that hold wanted bytes are loaded; for the last element of the
// payload (lim = payload end, else NULL) a chunk that would extend past the end
// is read byte by byte up to it, so no byte outside the payload is read
// (compute-sanitizer initcheck: the allocation's slack is never initialised).
// The realignment by the record's offset (uniform across a warp when the
// record stride is a multiple of 16) is a switch over the 4 word offsets with
// funnel shifts for the byte offset.
__device__ __noinline__ uint4 ld_chunk_tail(const uint4* a, const uint8_t* lim) {
    const uint8_t* b = reinterpret_cast<const uint8_t*>(a);
    uint32_t w[4] = {0, 0, 0, 0};
    for (int i = 0; i < 16 && b + i < lim; i++) w[i >> 2] |= (uint32_t)__ldg(b + i) << (8 * (i & 3));
    return make_uint4(w[0], w[1], w[2], w[3]);
}

template <int NB>
__device__ __forceinline__ void ld_stream(const uint8_t* p, uint32_t (&o)[(NB + 3) / 4],
                                          const uint8_t* lim = nullptr) {
    constexpr int NO = (NB + 3) / 4, NC = (NB + 30) / 16;   // output words, chunks touched at worst
    const uint4* a = reinterpret_cast<const uint4*>((uintptr_t)p & ~(uintptr_t)15);
    const uint32_t off = (uint32_t)(uintptr_t)p & 15u;
    const uint32_t last = (off + NB - 1) >> 4;             // last chunk holding a wanted byte
    const uint32_t sh = 8u * (off & 3u);
    uint32_t w[4 * NC + 4];
#pragma unroll
    for (int c = 0; c < NC; c++) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if ((uint32_t)c <= last)
            v = (lim && reinterpret_cast<const uint8_t*>(a + c + 1) > lim) ? ld_chunk_tail(a + c, lim)
                                                                           : __ldg(a + c);
        w[4 * c] = v.x;
        w[4 * c + 1] = v.y;
        w[4 * c + 2] = v.z;
        w[4 * c + 3] = v.w;
    }
#pragma unroll
    for (int j = 4 * NC; j < 4 * NC + 4; j++) w[j] = 0u;
#define FSSB_REALIGN(Q)                                                          \
    _Pragma("unroll") for (int j = 0; j < NO; j++) o[j] = __funnelshift_r(w[j + Q], w[j + Q + 1], sh)
    switch (off >> 2) {
        case 0: FSSB_REALIGN(0); break;
        case 1: FSSB_REALIGN(1); break;
        case 2: FSSB_REALIGN(2); break;
        default: FSSB_REALIGN(3); break;
    }
#undef FSSB_REALIGN
}

// A W-byte little-endian ring value at p.
template <int W>
__device__ __forceinline__ uint64_t ld_ring(const uint8_t* p, const uint8_t* lim = nullptr) {
    uint32_t o[(W + 3) / 4];
    ld_stream<W>(p, o, lim);
    uint64_t v = o[0];
    if (W > 4) v |= (uint64_t)o[(W + 3) / 4 - 1] << 32;
    return W >= 8 ? v : v & ((1ULL << (8 * W)) - 1);
}

template <int W>
__global__ void __launch_bounds__(kThreads, 1)
dcf_eval_packed_kernel(int party, int n, uint64_t count, const uint8_t* __restrict__ payload,
                       const uint64_t* __restrict__ x, const void* __restrict__ m_own,
                       const void* __restrict__ m_peer, uint64_t* __restrict__ out) {
    extern __shared__ __align__(128) uint32_t tab[];
    fssb::load_tables(tab);
    const fssb::Tab tb = fssb::make_tab(tab);
    constexpr uint32_t rec = 17 + W;
    constexpr int NW = (17 + W + 3) / 4;          // words of one level record
    const uint64_t EB = W + 16 + (uint64_t)n * rec + (uint64_t)(n + 1) * W;
    const uint32_t tail = W + 16 + n * rec;       // the leaf block
    const uint64_t mask = ring_mask(n);           // packed keys: out_bits == n
    const Span sp = cta_span(count);
    for (uint64_t e = sp.lo + threadIdx.x; e < sp.hi; e += blockDim.x) {
        const uint8_t* kp = payload + e * EB;
        const uint8_t* lim = e + 1 == count ? kp + EB : nullptr;   // payload end
        uint32_t sw[4];
        ld_stream<16>(kp + W, sw, lim);
        U4 s = U4{sw[0], sw[1], sw[2], sw[3]};
        uint32_t t = party;
        uint64_t acc = 0;
        const uint64_t xe = load_x(x, m_own, m_peer, n, e) & mask;
        for (int i = 0; i < n; i++) {
            uint32_t o[NW];
            ld_stream<rec>(kp + W + 16 + (uint32_t)i * rec, o, lim);
            const U4 cw = U4{o[0], o[1], o[2], o[3]};
            const uint32_t f = o[4] & 0xFFu;
            uint64_t sig = (uint64_t)__funnelshift_r(o[4], NW > 5 ? o[5] : 0u, 8);
            if (W > 3) sig |= (uint64_t)__funnelshift_r(NW > 5 ? o[5] : 0u, NW > 6 ? o[6] : 0u, 8) << 32;
            if (W < 8) sig &= (1ULL << (8 * W)) - 1;
            const uint64_t leaf = ld_ring<W>(kp + tail + (uint32_t)i * W, lim);
            const uint32_t xb = (uint32_t)(xe >> (n - 1 - i)) & 1u;
            const U4 a = fssb::mmo<0, true>(tb, s, 0u - xb);
            const uint32_t tm = 0u - t;
            uint32_t lane_lo, lane_hi;
            // n <= 32: the ring sum mod 2^n never sees lane_hi beyond its tau bit
            fssb::mmo_half<2, (W <= 4)>(tb, s, 0u - xb, lane_lo, lane_hi);
            const uint64_t lane = ((uint64_t)lane_hi << 32) | lane_lo;
            const uint32_t tau = ((lane_hi >> 31) ^ (t & (f >> (2 + xb)))) & 1u;
            const uint64_t sigma = lane ^ (sig & (0 - (uint64_t)t));
            acc += (leaf & (0 - (uint64_t)tau)) + sigma;
            s = xor4(a, and4(cw, tm));
            const uint32_t tn = ((a.w >> 31) ^ (t & (f >> xb))) & 1u;
            s.w &= 0x7FFFFFFFu;
            t = tn;
        }
        acc += (ld_ring<W>(kp + tail + (uint32_t)n * W, lim) & (0 - (uint64_t)t)) + lo64(s);
        out[e] = (party ? (0 - acc) : acc) & mask;
    }
}

template <int W>
__global__ void __launch_bounds__(kThreads, 1)
dpf_eval_packed_kernel(int party, int n, uint64_t count, const uint8_t* __restrict__ payload,
                       const uint64_t* __restrict__ x, const void* __restrict__ m_own,
                       const void* __restrict__ m_peer, uint64_t* __restrict__ out) {
    extern __shared__ __align__(128) uint32_t tab[];
    fssb::load_tables(tab);
    const fssb::Tab tb = fssb::make_tab(tab);
    const uint64_t EB = W + 16 + 17 * (uint64_t)n + W;
    const uint64_t mask = ring_mask(n);
    const Span sp = cta_span(count);
    for (uint64_t e = sp.lo + threadIdx.x; e < sp.hi; e += blockDim.x) {
        const uint8_t* kp = payload + e * EB;
        const uint8_t* lim = e + 1 == count ? kp + EB : nullptr;   // payload end
        uint32_t sw[4];
        ld_stream<16>(kp + W, sw, lim);
        U4 s = U4{sw[0], sw[1], sw[2], sw[3]};
        uint32_t t = party;
        const uint64_t xe = load_x(x, m_own, m_peer, n, e) & mask;
        for (int i = 0; i < n; i++) {
            uint32_t o[5];
            ld_stream<17>(kp + W + 16 + 17u * i, o, lim);
            const U4 cw = U4{o[0], o[1], o[2], o[3]};
            const uint32_t f = o[4] & 0xFFu;
            const uint32_t xb = (uint32_t)(xe >> (n - 1 - i)) & 1u;
            const U4 a = fssb::mmo<0, true>(tb, s, 0u - xb);
            s = xor4(a, and4(cw, 0u - t));
            const uint32_t tn = ((a.w >> 31) ^ (t & (f >> xb))) & 1u;
            s.w &= 0x7FFFFFFFu;
            t = tn;
        }
        const uint64_t cwf = ld_ring<W>(kp + W + 16 + 17u * n, lim);
        uint64_t o = (((uint64_t)t * cwf) + lo64(s)) & mask;
        if (party) o = (0 - o) & mask;
        out[e] = o;
    }
}

// -------------------------------------------------------------- DPF keygen
// fss._keygen_eq_core (fss.py:173-216): both parties' walks, 4 AES blocks/level.
__global__ void __launch_bounds__(kKeygenThreads, 1)
dpf_keygen_kernel(int n, uint64_t count, const uint64_t* __restrict__ alpha,
                  const uint64_t* __restrict__ alpha0, const uint8_t* __restrict__ s0_init,
                  const uint8_t* __restrict__ s1_init, uint8_t* __restrict__ scw,
                  uint8_t* __restrict__ tcw, uint64_t* __restrict__ cw_final,
                  uint64_t* __restrict__ alpha1) {
    extern __shared__ __align__(128) uint32_t tab[];
    fssb::load_tables(tab);
    const fssb::Tab tb = fssb::make_tab(tab);
    const uint64_t mask = ring_mask(n);
    const Span sp = cta_span(count);
    for (uint64_t e = sp.lo + threadIdx.x; e < sp.hi; e += blockDim.x) {
        U4 s0 = ld16(s0_init + 16 * e), s1 = ld16(s1_init + 16 * e);
        uint32_t t0 = 0, t1 = 1;
        const uint64_t al = alpha[e] & mask;
        for (int i = 0; i < n; i++) {
            const uint32_t a = (uint32_t)(al >> (n - 1 - i)) & 1u;
            U4 l0 = fssb::mmo<0, false>(tb, s0, 0), r0 = fssb::mmo<1, false>(tb, s0, 0);
            U4 l1 = fssb::mmo<0, false>(tb, s1, 0), r1 = fssb::mmo<1, false>(tb, s1, 0);
            const uint32_t tl0 = l0.w >> 31, tr0 = r0.w >> 31, tl1 = l1.w >> 31, tr1 = r1.w >> 31;
            l0.w &= 0x7FFFFFFFu; r0.w &= 0x7FFFFFFFu; l1.w &= 0x7FFFFFFFu; r1.w &= 0x7FFFFFFFu;
            // seed correction reuses the off-path child's string
            const U4 cws = a ? xor4(l0, l1) : xor4(r0, r1);
            const uint32_t cw_tl = tl0 ^ tl1 ^ 1u ^ a;
            const uint32_t cw_tr = tr0 ^ tr1 ^ a;
            const uint64_t off = (uint64_t)i * count + e;
            st16(scw + 16 * off, cws);
            tcw[off] = (uint8_t)(cw_tl | (cw_tr << 1));
            // advance both parties along alpha
            s0 = xor4(sel4(a, r0, l0), and4(cws, 0u - t0));
            s1 = xor4(sel4(a, r1, l1), and4(cws, 0u - t1));
            const uint32_t n0 = (a ? tr0 : tl0) ^ (t0 & (a ? cw_tr : cw_tl));
            const uint32_t n1 = (a ? tr1 : tl1) ^ (t1 & (a ? cw_tr : cw_tl));
            t0 = n0;
            t1 = n1;
        }
        const uint64_t v = (1 - lo64(s0) + lo64(s1)) & mask;
        cw_final[e] = t1 ? ((0 - v) & mask) : v;
        alpha1[e] = (al - alpha0[e]) & mask;
    }
}

// -------------------------------------------------------------- DCF keygen
// fss._keygen_cmp_core (fss.py:219-289): 6 AES blocks/level (3 per party).
__global__ void __launch_bounds__(kKeygenThreads, 1)
dcf_keygen_kernel(int n, int out_bits, uint64_t count, const uint64_t* __restrict__ alpha,
                  const uint64_t* __restrict__ alpha0, const uint8_t* __restrict__ s0_init,
                  const uint8_t* __restrict__ s1_init, uint8_t* __restrict__ scw,
                  uint8_t* __restrict__ tcw, uint64_t* __restrict__ sigma_cw,
                  uint64_t* __restrict__ leaf_cw, uint64_t* __restrict__ alpha1) {
    extern __shared__ __align__(128) uint32_t tab[];
    fssb::load_tables(tab);
    const fssb::Tab tb = fssb::make_tab(tab);
    const uint64_t nmask = ring_mask(n);
    const uint64_t mask = ring_mask(out_bits);
    const Span sp = cta_span(count);
    for (uint64_t e = sp.lo + threadIdx.x; e < sp.hi; e += blockDim.x) {
        U4 s0 = ld16(s0_init + 16 * e), s1 = ld16(s1_init + 16 * e);
        uint32_t t0 = 0, t1 = 1;
        const uint64_t al = alpha[e] & nmask;
        for (int i = 0; i < n; i++) {
            const uint32_t a = (uint32_t)(al >> (n - 1 - i)) & 1u;
            U4 l0 = fssb::mmo<0, false>(tb, s0, 0), r0 = fssb::mmo<1, false>(tb, s0, 0);
            const U4 g0 = fssb::mmo<2, false>(tb, s0, 0);
            U4 l1 = fssb::mmo<0, false>(tb, s1, 0), r1 = fssb::mmo<1, false>(tb, s1, 0);
            const U4 g1 = fssb::mmo<2, false>(tb, s1, 0);
            const uint32_t tl0 = l0.w >> 31, tr0 = r0.w >> 31, tl1 = l1.w >> 31, tr1 = r1.w >> 31;
            l0.w &= 0x7FFFFFFFu; r0.w &= 0x7FFFFFFFu; l1.w &= 0x7FFFFFFFu; r1.w &= 0x7FFFFFFFu;
            const uint64_t gl0 = lo64(g0) & mask, gr0 = hi64(g0) & mask;
            const uint64_t gl1 = lo64(g1) & mask, gr1 = hi64(g1) & mask;
            const uint32_t ul0 = g0.y >> 31, ur0 = g0.w >> 31, ul1 = g1.y >> 31, ur1 = g1.w >> 31;

            const U4 cws = a ? xor4(l0, l1) : xor4(r0, r1);
            const uint32_t cw_tl = tl0 ^ tl1 ^ 1u ^ a;
            const uint32_t cw_tr = tr0 ^ tr1 ^ a;
            // sigma collapses on the stay side (alpha bit), fss.py:245-249
            const uint64_t cw_sig = a ? (gr0 ^ gr1) : (gl0 ^ gl1);
            const uint32_t cw_ul = ul0 ^ ul1 ^ a;
            const uint32_t cw_ur = ur0 ^ ur1 ^ 1u ^ a;
            const uint64_t off = (uint64_t)i * count + e;
            st16(scw + 16 * off, cws);
            tcw[off] = (uint8_t)(cw_tl | (cw_tr << 1) | (cw_ul << 2) | (cw_ur << 3));
            sigma_cw[off] = cw_sig;
            // leaf word from the exit side (not alpha bit) after correction, fss.py:268-273
            const uint64_t g0x = (a ? gl0 : gr0) ^ (t0 ? cw_sig : 0);
            const uint64_t g1x = (a ? gl1 : gr1) ^ (t1 ? cw_sig : 0);
            const uint32_t u1x = (a ? ul1 : ur1) ^ (t1 & (a ? cw_ul : cw_ur));
            const uint64_t leaf = ((uint64_t)a - g0x + g1x) & mask;
            leaf_cw[off] = u1x ? ((0 - leaf) & mask) : leaf;
            // advance along alpha
            s0 = xor4(sel4(a, r0, l0), and4(cws, 0u - t0));
            s1 = xor4(sel4(a, r1, l1), and4(cws, 0u - t1));
            const uint32_t n0 = (a ? tr0 : tl0) ^ (t0 & (a ? cw_tr : cw_tl));
            const uint32_t n1 = (a ? tr1 : tl1) ^ (t1 & (a ? cw_tr : cw_tl));
            t0 = n0;
            t1 = n1;
        }
        const uint64_t v = (1 - (lo64(s0) & mask) + (lo64(s1) & mask)) & mask;
        leaf_cw[(uint64_t)n * count + e] = t1 ? ((0 - v) & mask) : v;
        alpha1[e] = (al - alpha0[e]) & nmask;
    }
}

// ---------------------------------------------------- keygen, lane pairs
// Small batches: a PAIR of lanes deals one key pair -- the even lane walks
// party 0's seed, the odd lane party 1's (same three fixed keys: one
// instruction stream), so each lane encrypts 3 (DCF) or 2 (DPF) blocks per
// level instead of 6 / 4. Per level the partners swap what the correction
// words need (the off-path child seed, the sigma/tau block, the t bits) by
// shuffles and compute identical correction words; the even lane stores the
// seed / t corrections, the odd lane sigma and the leaf word.
constexpr int kPairKeygenThreads = 1024;

// W32 (DCF, out_bits <= 32): the sigma/tau block through mmo_sigma_tau32.
template <bool CMP, bool W32 = false>
__global__ void __launch_bounds__(kPairKeygenThreads, 1)
keygen_pair_kernel(int n, int out_bits, uint64_t count, const uint64_t* __restrict__ alpha,
                   const uint64_t* __restrict__ alpha0, const uint8_t* __restrict__ s0_init,
                   const uint8_t* __restrict__ s1_init, uint8_t* __restrict__ scw,
                   uint8_t* __restrict__ tcw, uint64_t* __restrict__ sigma_cw,
                   uint64_t* __restrict__ leaf_cw, uint64_t* __restrict__ cw_final,
                   uint64_t* __restrict__ alpha1) {
    extern __shared__ __align__(128) uint32_t tab[];
    fssb::load_tables(tab);
    const fssb::Tab tb = fssb::make_tab(tab);
    const uint64_t nmask = ring_mask(n);
    const uint64_t mask = ring_mask(out_bits);
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t p = lane & 1;                 // the party this lane walks
    const uint32_t pm = 3u << (lane & ~1u);
    const uint32_t q = lane ^ 1u;                // partner lane
    const Span sp = cta_span(count);
    for (uint64_t e = sp.lo + (threadIdx.x >> 1); e < sp.hi; e += blockDim.x >> 1) {
        U4 s = ld16((p ? s1_init : s0_init) + 16 * e);
        uint32_t t = p;
        const uint64_t al = alpha[e] & nmask;
        for (int i = 0; i < n; i++) {
            const uint32_t a = (uint32_t)(al >> (n - 1 - i)) & 1u;
            U4 l = fssb::mmo<0, false>(tb, s, 0), r = fssb::mmo<1, false>(tb, s, 0);
            const uint32_t tl = l.w >> 31, tr = r.w >> 31;
            l.w &= 0x7FFFFFFFu;
            r.w &= 0x7FFFFFFFu;
            // the off-path child of both parties gives the seed correction
            const U4 side = a ? l : r;
            U4 cws;
            cws.x = side.x ^ __shfl_sync(pm, side.x, q);
            cws.y = side.y ^ __shfl_sync(pm, side.y, q);
            cws.z = side.z ^ __shfl_sync(pm, side.z, q);
            cws.w = side.w ^ __shfl_sync(pm, side.w, q);
            uint32_t g_x = 0, g_y = 0, g_z = 0, g_w = 0, h_x = 0, h_y = 0, h_z = 0, h_w = 0;
            if (CMP) {
                const U4 g = W32 ? fssb::mmo_sigma_tau32<2>(tb, s) : fssb::mmo<2, false>(tb, s, 0);
                g_x = g.x; g_y = g.y; g_z = g.z; g_w = g.w;
                h_x = __shfl_sync(pm, g.x, q);
                h_y = __shfl_sync(pm, g.y, q);
                h_z = __shfl_sync(pm, g.z, q);
                h_w = __shfl_sync(pm, g.w, q);
            }
            const uint32_t bits = tl | (tr << 1) | (t << 2);
            const uint32_t pb = __shfl_sync(pm, bits, q);
            // (party 0, party 1) views of the exchanged values
            const uint32_t b0 = p ? pb : bits, b1 = p ? bits : pb;
            const uint32_t tl0 = b0 & 1u, tr0 = (b0 >> 1) & 1u, t0 = (b0 >> 2) & 1u;
            const uint32_t tl1 = b1 & 1u, tr1 = (b1 >> 1) & 1u, t1 = (b1 >> 2) & 1u;
            const uint32_t cw_tl = tl0 ^ tl1 ^ 1u ^ a;
            const uint32_t cw_tr = tr0 ^ tr1 ^ a;
            const uint64_t off = (uint64_t)i * count + e;
            if (!p) {
                st16(scw + 16 * off, cws);
            }
            uint32_t tbyte = cw_tl | (cw_tr << 1);
            if (CMP) {
                const uint32_t G0x = p ? h_x : g_x, G0y = p ? h_y : g_y, G0z = p ? h_z : g_z, G0w = p ? h_w : g_w;
                const uint32_t G1x = p ? g_x : h_x, G1y = p ? g_y : h_y, G1z = p ? g_z : h_z, G1w = p ? g_w : h_w;
                const uint64_t gl0 = (((uint64_t)G0y << 32) | G0x) & mask, gr0 = (((uint64_t)G0w << 32) | G0z) & mask;
                const uint64_t gl1 = (((uint64_t)G1y << 32) | G1x) & mask, gr1 = (((uint64_t)G1w << 32) | G1z) & mask;
                const uint32_t ul0 = G0y >> 31, ur0 = G0w >> 31, ul1 = G1y >> 31, ur1 = G1w >> 31;
                // sigma collapses on the stay side (alpha bit), fss.py:245-249
                const uint64_t cw_sig = a ? (gr0 ^ gr1) : (gl0 ^ gl1);
                const uint32_t cw_ul = ul0 ^ ul1 ^ a;
                const uint32_t cw_ur = ur0 ^ ur1 ^ 1u ^ a;
                tbyte |= (cw_ul << 2) | (cw_ur << 3);
                if (p) {
                    // leaf word from the exit side after correction, fss.py:268-273
                    sigma_cw[off] = cw_sig;
                    const uint64_t g0x = (a ? gl0 : gr0) ^ (t0 ? cw_sig : 0);
                    const uint64_t g1x = (a ? gl1 : gr1) ^ (t1 ? cw_sig : 0);
                    const uint32_t u1x = (a ? ul1 : ur1) ^ (t1 & (a ? cw_ul : cw_ur));
                    const uint64_t leaf = ((uint64_t)a - g0x + g1x) & mask;
                    leaf_cw[off] = u1x ? ((0 - leaf) & mask) : leaf;
                }
            }
            if (!p) tcw[off] = (uint8_t)tbyte;
            // advance this lane's party along alpha
            s = xor4(sel4(a, r, l), and4(cws, 0u - t));
            t = (a ? tr : tl) ^ (t & (a ? cw_tr : cw_tl));
        }
        const uint32_t o_lo = __shfl_sync(pm, s.x, q), o_hi = __shfl_sync(pm, s.y, q);
        const uint32_t o_t = __shfl_sync(pm, t, q);
        if (p) {   // this lane holds (s1, t1), its partner (s0, t0)
            const uint64_t s0r = ((uint64_t)o_hi << 32) | o_lo;
            if (CMP) {
                const uint64_t v = (1 - (s0r & mask) + (lo64(s) & mask)) & mask;
                leaf_cw[(uint64_t)n * count + e] = t ? ((0 - v) & mask) : v;
            } else {
                const uint64_t v = (1 - s0r + lo64(s)) & mask;
                cw_final[e] = t ? ((0 - v) & mask) : v;
            }
        } else {
            (void)o_t;
            alpha1[e] = (al - alpha0[e]) & nmask;
        }
    }
}

// ------------------------------------------------------------ PCG64 tapes
// Device restatement of numpy's Generator(PCG64) draws behind fss._sample_tape
// (fss.py:292-303): PCG64 XSL-RR 128/64, step-then-output. The 32-bit stream
// splits each 64-bit output low half first (numpy next_uint32), bounded draws
// with power-of-two ranges are word >> (32-n) (Lemire, no rejection), uint8
// draws take the 4 bytes of each word in little-endian order.
struct Pcg {
    unsigned __int128 state, inc;
};

__device__ __forceinline__ unsigned __int128 pcg_mult() {
    return ((unsigned __int128)0x2360ed051fc65da4ULL << 64) | 0x4385df649fccf645ULL;
}

__device__ __forceinline__ Pcg pcg_advance(Pcg p, uint64_t delta) {
    unsigned __int128 cur_mult = pcg_mult(), cur_plus = p.inc, acc_mult = 1, acc_plus = 0;
    while (delta) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    p.state = acc_mult * p.state + acc_plus;
    return p;
}

__device__ __forceinline__ uint64_t pcg_next(Pcg& p) {
    p.state = p.state * pcg_mult() + p.inc;
    const uint64_t hi = (uint64_t)(p.state >> 64), lo = (uint64_t)p.state;
    const uint64_t xr = hi ^ lo;
    const unsigned rot = (unsigned)(hi >> 58);
    return (xr >> rot) | (xr << ((64 - rot) & 63));
}

struct TapePlan {
    uint64_t state_lo, state_hi, inc_lo, inc_hi;
    int n;
    uint64_t count;    // elements of the whole tape (numpy's `count`)
    int draw_alpha;    // alpha drawn (1) or given (0)
    int draw_alpha0;   // alpha0 drawn (1) or not (0: seeds-only tape)
    int has_uint32;    // numpy's buffered half-word present at start
    uint32_t uinteger;
    uint64_t raw64;    // number of 64-bit draws before the 32-bit stream (n > 32)
    uint64_t words;    // number of 32-bit words in the stream
    // element slice [lo, hi) of the tape that is written (outputs indexed from
    // lo), and the raw-output range [r_begin, r_end) one launch covers; the
    // whole tape is lo = 0, hi = count, r = [0, total)
    uint64_t lo, hi;
    uint64_t r_begin, r_end;
    int emit_buffered; // this launch writes word 0 (numpy's buffered half-word)
};

// Thread j handles raw outputs [r_begin + j*kChunk, r_begin + (j+1)*kChunk).
constexpr int kChunk = 16;

// 32-bit word w of the stream -> its tape slot, written when its element lies
// in the slice.
__device__ __forceinline__ void emit_word(const TapePlan& P, uint64_t w, uint32_t v, uint64_t* alpha,
                                          uint64_t* alpha0, uint8_t* s0, uint8_t* s1) {
    const uint64_t N = P.count;
    uint64_t k = w;
    if (P.n <= 32) {
        const int sh = 32 - P.n;
        if (P.draw_alpha) {
            if (k < N) { if (k >= P.lo && k < P.hi) alpha[k - P.lo] = (uint64_t)(v >> sh); return; }
            k -= N;
        }
        if (P.draw_alpha0) {
            if (k < N) { if (k >= P.lo && k < P.hi) alpha0[k - P.lo] = (uint64_t)(v >> sh); return; }
            k -= N;
        }
    }
    // seeds: 4 words per seed, byte 15 top bit cleared (prg.random_seeds, prg.py:36-40)
    uint8_t* dst = k < 4 * N ? s0 : s1;
    if (k >= 4 * N) k -= 4 * N;
    const uint64_t e = k >> 2;
    if (e < P.lo || e >= P.hi) return;
    if ((k & 3) == 3) v &= 0x7FFFFFFFu;
    reinterpret_cast<uint32_t*>(dst)[k - 4 * P.lo] = v;
}

__global__ void pcg64_tape_kernel(TapePlan P, uint64_t* __restrict__ alpha, uint64_t* __restrict__ alpha0,
                                  uint8_t* __restrict__ s0, uint8_t* __restrict__ s1) {
    const uint64_t h = (uint64_t)P.has_uint32;
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j == 0 && P.emit_buffered) emit_word(P, 0, P.uinteger, alpha, alpha0, s0, s1);
    const uint64_t begin = P.r_begin + j * kChunk;
    if (begin >= P.r_end) return;
    const uint64_t end = begin + kChunk < P.r_end ? begin + kChunk : P.r_end;
    Pcg p;
    p.state = ((unsigned __int128)P.state_hi << 64) | P.state_lo;
    p.inc = ((unsigned __int128)P.inc_hi << 64) | P.inc_lo;
    p = pcg_advance(p, begin);
    const uint64_t N = P.count;
    const int sh64 = 64 - P.n;
    for (uint64_t r = begin; r < end; r++) {
        const uint64_t v = pcg_next(p);
        if (r < P.raw64) {  // n > 32: 64-bit Lemire draws, v >> (64-n)
            uint64_t k = r;
            if (P.draw_alpha) {
                if (k < N) { if (k >= P.lo && k < P.hi) alpha[k - P.lo] = v >> sh64; continue; }
                k -= N;
            }
            if (k >= P.lo && k < P.hi) alpha0[k - P.lo] = v >> sh64;
            continue;
        }
        const uint64_t q = r - P.raw64;
        const uint64_t w_lo = h + 2 * q, w_hi = w_lo + 1;
        if (w_lo < P.words) emit_word(P, w_lo, (uint32_t)v, alpha, alpha0, s0, s1);
        if (w_hi < P.words) emit_word(P, w_hi, (uint32_t)(v >> 32), alpha, alpha0, s0, s1);
    }
}

// RingTensor.random (ring.py:61-65) through numpy's Generator(PCG64):
//   raw = integers(0, 2^63, uint64)   -> one 64-bit output per element, v >> 1
//   raw = raw << 1 | integers(0, 2)   -> one 32-bit word per element, w >> 31
//   raw &= mask(n)
// (both bounded draws are Lemire with a power-of-two range: no rejection.)
// The 64-bit part takes outputs [0, count); the 32-bit words follow, with
// numpy's buffered half-word (has_uint32) served first.
__global__ void pcg64_ring_kernel(TapePlan P, uint64_t* __restrict__ out) {
    const uint64_t N = P.count;
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t begin = j * kChunk;
    if (begin >= N) return;
    const uint64_t mask = P.n >= 64 ? ~0ULL : ((1ULL << P.n) - 1);
    const uint64_t h = (uint64_t)P.has_uint32;
    Pcg base;
    base.state = ((unsigned __int128)P.state_hi << 64) | P.state_lo;
    base.inc = ((unsigned __int128)P.inc_hi << 64) | P.inc_lo;
    Pcg p = pcg_advance(base, begin);    // 64-bit draws: outputs [0, N)
    Pcg w;                                // 32-bit words: outputs N, N+1, ...
    uint64_t q = ~0ULL, cur = 0;
#pragma unroll
    for (int i = 0; i < kChunk; i++) {
        const uint64_t k = begin + i;
        if (k >= N) break;
        const uint64_t hi = pcg_next(p) & ~1ULL;   // (v >> 1) << 1
        uint32_t word;
        if (k < h) {
            word = P.uinteger;                      // numpy's buffered half-word
        } else {
            const uint64_t r = k - h;
            if (q == ~0ULL) {
                q = r >> 1;
                w = pcg_advance(base, N + q);
                cur = pcg_next(w);
            } else if ((r >> 1) != q) {
                q = r >> 1;
                cur = pcg_next(w);
            }
            word = (r & 1) ? (uint32_t)(cur >> 32) : (uint32_t)cur;   // low half first
        }
        out[k] = (hi | (uint64_t)(word >> 31)) & mask;
    }
}

// ------------------------------------------------------------ runtime glue

constexpr int kOk = FSS_OK, kEinval = FSS_EINVAL, kEcuda = FSS_ECUDA;

int set_err(int code, const char* fmt, const char* a = "") {
    char buf[512];
    snprintf(buf, sizeof(buf), fmt, a);
    return fssb::set_error(code, buf);
}

// A NULL device pointer would fault inside the kernel and poison the CUDA
// context; reject it up front (before any CUDA call) with FSS_EINVAL.
bool any_null(std::initializer_list<const void*> ptrs) {
    for (const void* p : ptrs)
        if (!p) return true;
    return false;
}
#define FSS_REQUIRE(...) \
    if (any_null({__VA_ARGS__})) return set_err(kEinval, "null device pointer%s")

// Per-device launch facts, set once: the SM count and, per kernel, the 128 KiB
// dynamic shared-memory opt-in (cudaFuncSetAttribute is per device, and costs
// a driver call; the online protocols launch small kernels back to back, so it
// is done on a kernel's first launch on a device only). Two party threads may
// launch concurrently: the table is guarded by a mutex (the fast path is a
// short scan of a few entries).
struct DevInfo {
    int sms = 0;
    std::vector<const void*> attr_done;   // kernels whose smem opt-in is set
};
std::mutex g_dev_mu;
DevInfo g_dev[64];

template <typename K>
int prep_launch(K kernel, int* grid, int smem = fssb::kTableBytes) {
    int dev = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return set_err(kEcuda, "cudaGetDevice: %s", cudaGetErrorString(err));
    const void* key = reinterpret_cast<const void*>(kernel);
    std::lock_guard<std::mutex> lock(g_dev_mu);
    DevInfo& d = g_dev[dev & 63];
    if (!d.sms) {
        err = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
        if (err != cudaSuccess) return set_err(kEcuda, "cudaDeviceGetAttribute: %s", cudaGetErrorString(err));
        err = fssb::table_image_upload();   // the T-table image the kernels' TMA copies read
        if (err != cudaSuccess) {
            d.sms = 0;
            return set_err(kEcuda, "T-table image upload: %s", cudaGetErrorString(err));
        }
    }
    bool done = false;
    for (const void* k : d.attr_done) done |= (k == key);
    if (!done) {
        err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (err != cudaSuccess) return set_err(kEcuda, "cudaFuncSetAttribute: %s", cudaGetErrorString(err));
        d.attr_done.push_back(key);
    }
    *grid = d.sms;
    return kOk;
}

uint64_t ring_mask_host(int w) { return w >= 64 ? ~0ULL : ((1ULL << w) - 1); }


// Launch shape of the AES kernels: one CTA per SM (the tables fill 128 KiB of
// shared memory) with max_threads threads; each CTA strides through its own
// contiguous run of elements (cta_span). Batches too small to give every SM
// max_threads elements are spread over all SMs with fewer threads each.
// (Trimming the thread count so the last pass over a run is full measured
// slower than 1024 threads with a partial last pass -- profiles/r01_wave_bench.json.)
int balanced_grid(uint64_t count, int sms, int max_threads, int* threads) {
    const uint64_t per_sm = (count + sms - 1) / sms;
    if (per_sm >= (uint64_t)max_threads) {
        *threads = max_threads;
        return sms;
    }
    if (per_sm >= 32) {
        *threads = (int)((per_sm + 31) / 32 * 32);
        return sms;
    }
    *threads = 32;
    const uint64_t grid = (count + 31) / 32;
    return (int)(grid < (uint64_t)sms ? (grid ? grid : 1) : sms);
}

int eval_grid(uint64_t count, int sms, int* threads) { return balanced_grid(count, sms, kThreads, threads); }

int check_launch() {
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return set_err(kEcuda, "kernel launch: %s", cudaGetErrorString(err));
    return kOk;
}

}  // namespace

extern "C" {

const char* fss_last_error(void) { return fssb::last_error(); }

int fss_abi_version(void) { return FSS_ABI_VERSION; }

int fss_aes_mmo_expand(const uint8_t* seeds, uint64_t count, int out_blocks, uint8_t* out,
                       void* stream) {
    if (out_blocks < 2 || out_blocks > 3) return set_err(kEinval, "out_blocks must be 2 or 3%s");
    if (count == 0) return kOk;
    FSS_REQUIRE(seeds, out);
    int sms;
    if (int rc = prep_launch(expand_kernel, &sms)) return rc;
    int threads;
    const int grid = balanced_grid(count, sms, kKeygenThreads, &threads);
    expand_kernel<<<grid, threads, fssb::kTableBytes, (cudaStream_t)stream>>>(
        seeds, count, out_blocks, out);
    return check_launch();
}

}  // extern "C"

namespace {

int launch_dpf_eval(int party, int n, uint64_t count, uint64_t ld, const uint8_t* seed0,
                    const uint8_t* scw, const uint8_t* tcw, const uint64_t* cw_final,
                    const uint64_t* x, const void* m_own, const void* m_peer, uint64_t* out,
                    void* stream) {
    if (party != 0 && party != 1) return set_err(kEinval, "party must be 0 or 1%s");
    if (n < 1 || n > 64) return set_err(kEinval, "n out of range%s");
    if (count == 0) return kOk;
    if (ld < count) return set_err(kEinval, "level stride ld must be >= count%s");
    if (!x && (!m_own || !m_peer)) return set_err(kEinval, "need x or both masked messages%s");
    FSS_REQUIRE(seed0, scw, tcw, cw_final, out);
    int sms;
    if (int rc = prep_launch(dpf_eval_kernel, &sms)) return rc;
    int threads;
    const int grid = eval_grid(count, sms, &threads);
    dpf_eval_kernel<<<grid, threads, fssb::kTableBytes, (cudaStream_t)stream>>>(
        party, n, count, ld, seed0, scw, tcw, cw_final, x, m_own, m_peer, out);
    return check_launch();
}

int launch_dcf_eval(int party, int n, int out_bits, uint64_t count, uint64_t ld, const uint8_t* seed0,
                    const uint8_t* scw, const uint8_t* tcw, const uint64_t* sigma_cw,
                    const uint64_t* leaf_cw, const uint64_t* x, const void* m_own, const void* m_peer,
                    uint64_t* out, uint64_t* levels, void* stream) {
    if (party != 0 && party != 1) return set_err(kEinval, "party must be 0 or 1%s");
    if (n < 1 || n > 63 || out_bits < n || out_bits > 63)
        return set_err(kEinval, "need 1 <= n <= out_bits <= 63%s");
    if (count == 0) return kOk;
    if (ld < count) return set_err(kEinval, "level stride ld must be >= count%s");
    if (!x && (!m_own || !m_peer)) return set_err(kEinval, "need x or both masked messages%s");
    FSS_REQUIRE(seed0, scw, tcw, sigma_cw, leaf_cw, out);
    int sms;
    const bool w32 = FSSB_W32 && out_bits <= 32;
    auto kern = levels ? (w32 ? dcf_eval_kernel<true, true> : dcf_eval_kernel<false, true>)
                       : (w32 ? dcf_eval_kernel<true, false> : dcf_eval_kernel<false, false>);
    if (int rc = prep_launch(kern, &sms)) return rc;
    int threads;
    const int grid = eval_grid(count, sms, &threads);
    kern<<<grid, threads, fssb::kTableBytes, (cudaStream_t)stream>>>(
        party, n, out_bits, count, ld, seed0, scw, tcw, sigma_cw, leaf_cw, x, m_own, m_peer, out, levels);
    return check_launch();
}

// Host-buffer evaluation as one native call: the element range is streamed in
// chunks over two CUDA streams -- H2D of x (pinned host), the eval kernel, D2H
// of the shares (pinned host) -- so the copies of one chunk overlap the kernel
// of the other. Chunks alternate streams and each stream reuses its own slot of
// the caller's device scratch (2 * chunk words each for x and out), which stream
// order makes safe. Returns after enqueueing; the caller synchronises.
struct HostPipe {
    const uint64_t* x_host;
    uint64_t* out_host;
    uint64_t* x_dev;
    uint64_t* out_dev;
    uint64_t chunk;
    cudaStream_t st[2];
    uint64_t* stage;  // NULL: host buffers are pinned; else 4 * chunk pinned words
};

template <typename Launch>
int run_host_pipe_pinned(const HostPipe& hp, uint64_t count, Launch launch) {
    for (uint64_t i = 0, lo = 0; lo < count; i++, lo += hp.chunk) {
        const uint64_t m = count - lo < hp.chunk ? count - lo : hp.chunk;
        const int slot = (int)(i & 1);
        cudaStream_t s = hp.st[slot];
        uint64_t* xd = hp.x_dev + slot * hp.chunk;
        uint64_t* od = hp.out_dev + slot * hp.chunk;
        cudaError_t err = cudaMemcpyAsync(xd, hp.x_host + lo, m * 8, cudaMemcpyHostToDevice, s);
        if (err != cudaSuccess) return set_err(kEcuda, "H2D: %s", cudaGetErrorString(err));
        if (int rc = launch(lo, m, xd, od, s)) return rc;
        err = cudaMemcpyAsync(hp.out_host + lo, od, m * 8, cudaMemcpyDeviceToHost, s);
        if (err != cudaSuccess) return set_err(kEcuda, "D2H: %s", cudaGetErrorString(err));
    }
    return kOk;
}

// Host memcpy between pageable and pinned memory, split over up to 8 OpenMP
// threads: one core copies ~4 GB/s on the B200 boxes, so a single-threaded
// staging copy (2 x 8 B per element) would be slower than the kernel.
void par_memcpy(void* dst, const void* src, size_t bytes) {
    constexpr size_t kMin = 1 << 20;
    // processors, not omp_get_max_threads(): torchrun exports OMP_NUM_THREADS=1
    int nt = omp_get_num_procs();
    nt = nt > 8 ? 8 : nt;
    if (bytes < kMin || nt <= 1) {
        memcpy(dst, src, bytes);
        return;
    }
    const size_t piece = (bytes / nt + 63) & ~(size_t)63;
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int i = 0; i < nt; i++) {
        const size_t lo = (size_t)i * piece;
        if (lo < bytes)
            memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo,
                   lo + piece <= bytes ? piece : bytes - lo);
    }
}

// Size of staged chunk i starting at element lo. Long ranges ramp up and down
// (chunk/4, chunk/2, chunk, ..., chunk, chunk/2, chunk/4): the first kernel
// waits only for a quarter chunk's host copy + H2D, and after the last kernel
// only a quarter chunk's D2H + host copy remains.
#ifndef FSSB_STAGED_RAMP
#define FSSB_STAGED_RAMP 1
#endif
uint64_t staged_chunk(uint64_t i, uint64_t lo, uint64_t count, uint64_t chunk) {
    const uint64_t r = count - lo, q = chunk / 4;
    if (!FSSB_STAGED_RAMP || count < 8 * chunk || q == 0) return r < chunk ? r : chunk;
    uint64_t m = i == 0 ? q : (i == 1 ? 2 * q : chunk);
    if (r <= q) return r;
    if (r <= 3 * q) m = r - q < m ? r - q : m;                  // then the last quarter
    else if (r <= chunk + 3 * q) m = r - 3 * q < m ? r - 3 * q : m;   // then a half, a quarter
    return m < r ? m : r;
}

// Pageable host buffers (e.g. numpy arrays): chunks are staged through pinned
// slots by host memcpy, which overlaps the other slot's copies and kernel.
// Returns when every share is in out_host.
// Three staging slots, drained two chunks behind: after enqueueing chunk i the
// host copies out chunk i-2's shares, so a slow host copy (first-touch page
// faults of a fresh numpy result) is absorbed while chunks i-1 and i are still
// queued; with two slots the host waited on chunk i-1 and the GPU idled
// whenever that copy outran one kernel (0.3-0.4 ms gaps in the trace).
// Chunk i runs on stream i & 1 and uses slot i % 3; a slot is refilled only
// after the drain of its previous chunk returned (kernel and D2H complete).
#ifndef FSSB_STAGE_SLOTS
#define FSSB_STAGE_SLOTS 3   // 2..3 (the buffers are sized for 3); drain lag = slots - 1
#endif
constexpr int kStageSlots = FSSB_STAGE_SLOTS;

template <typename Launch>
int run_host_pipe_staged(const HostPipe& hp, uint64_t count, Launch launch) {
    constexpr int K = kStageSlots;
    cudaEvent_t h2d[K], d2h[K];
    uint64_t* sin[K];
    uint64_t* sout[K];
    bool in_busy[K], out_busy[K];
    uint64_t out_lo[K], out_m[K];
    for (int k = 0; k < K; k++) {
        cudaEventCreateWithFlags(&h2d[k], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&d2h[k], cudaEventDisableTiming);
        sin[k] = hp.stage + k * hp.chunk;
        sout[k] = hp.stage + (K + k) * hp.chunk;
        in_busy[k] = out_busy[k] = false;
        out_lo[k] = out_m[k] = 0;
    }
    // A page-locked out_host (the drop-in hands out pinned numpy results) takes
    // the shares straight from the D2H copies: no staging slot, no copy-out.
#ifndef FSSB_DIRECT_D2H
#define FSSB_DIRECT_D2H 1
#endif
    cudaPointerAttributes pa;
    const bool out_pinned = FSSB_DIRECT_D2H && cudaPointerGetAttributes(&pa, hp.out_host) == cudaSuccess &&
                            pa.type == cudaMemoryTypeHost;
    cudaGetLastError();   // a pageable pointer may leave an error code behind
    int rc = kOk;
    auto drain = [&](int k) {
        if (!out_busy[k]) return;
        cudaEventSynchronize(d2h[k]);
        if (!out_pinned) par_memcpy(hp.out_host + out_lo[k], sout[k], out_m[k] * 8);
        out_busy[k] = false;
    };
    uint64_t i = 0;
    for (uint64_t lo = 0, m = 0; lo < count && rc == kOk; i++, lo += m) {
        m = staged_chunk(i, lo, count, hp.chunk);
        const int slot = (int)(i % K);
        cudaStream_t s = hp.st[i & 1];
        uint64_t* xd = hp.x_dev + slot * hp.chunk;
        uint64_t* od = hp.out_dev + slot * hp.chunk;
        drain(slot);                                          // chunk i-3 (normally done already)
        if (in_busy[slot]) cudaEventSynchronize(h2d[slot]);   // staging slot free again
        par_memcpy(sin[slot], hp.x_host + lo, m * 8);
        cudaError_t err = cudaMemcpyAsync(xd, sin[slot], m * 8, cudaMemcpyHostToDevice, s);
        if (err != cudaSuccess) { rc = set_err(kEcuda, "H2D: %s", cudaGetErrorString(err)); break; }
        cudaEventRecord(h2d[slot], s);
        in_busy[slot] = true;
        if ((rc = launch(lo, m, xd, od, s)) != kOk) break;
        err = cudaMemcpyAsync(out_pinned ? hp.out_host + lo : sout[slot], od, m * 8, cudaMemcpyDeviceToHost, s);
        if (err != cudaSuccess) { rc = set_err(kEcuda, "D2H: %s", cudaGetErrorString(err)); break; }
        cudaEventRecord(d2h[slot], s);
        out_busy[slot] = true;
        out_lo[slot] = lo;
        out_m[slot] = m;
        if (i >= K - 1) drain((int)((i - (K - 1)) % K));      // K - 1 chunks behind
    }
    if (rc == kOk) {
        for (uint64_t j = i >= K - 1 ? i - (K - 1) : 0; j < i; j++) drain((int)(j % K));   // in element order
    } else {
        cudaStreamSynchronize(hp.st[0]);
        cudaStreamSynchronize(hp.st[1]);
    }
    for (int k = 0; k < K; k++) {
        cudaEventDestroy(h2d[k]);
        cudaEventDestroy(d2h[k]);
    }
    return rc;
}

template <typename Launch>
int run_host_pipe(const HostPipe& hp, uint64_t count, Launch launch) {
    if (!hp.x_host || !hp.out_host || !hp.x_dev || !hp.out_dev || hp.chunk == 0)
        return set_err(kEinval, "pipelined eval needs host/device buffers and a chunk size%s");
    return hp.stage ? run_host_pipe_staged(hp, count, launch) : run_host_pipe_pinned(hp, count, launch);
}

}  // namespace

extern "C" {

int fss_dpf_eval(int party, int n, uint64_t count, uint64_t ld, const uint8_t* seed0,
                 const uint8_t* scw, const uint8_t* tcw, const uint64_t* cw_final, const uint64_t* x,
                 uint64_t* out, void* stream) {
    return launch_dpf_eval(party, n, count, ld, seed0, scw, tcw, cw_final, x, nullptr, nullptr, out,
                           stream);
}

int fss_dpf_eval_masked(int party, int n, uint64_t count, uint64_t ld, const uint8_t* seed0,
                        const uint8_t* scw, const uint8_t* tcw, const uint64_t* cw_final,
                        const void* m_own, const void* m_peer, uint64_t* out, void* stream) {
    return launch_dpf_eval(party, n, count, ld, seed0, scw, tcw, cw_final, nullptr, m_own, m_peer, out,
                           stream);
}

int fss_dcf_eval(int party, int n, int out_bits, uint64_t count, uint64_t ld, const uint8_t* seed0,
                 const uint8_t* scw, const uint8_t* tcw, const uint64_t* sigma_cw,
                 const uint64_t* leaf_cw, const uint64_t* x, uint64_t* out, uint64_t* levels,
                 void* stream) {
    return launch_dcf_eval(party, n, out_bits, count, ld, seed0, scw, tcw, sigma_cw, leaf_cw, x, nullptr,
                           nullptr, out, levels, stream);
}

int fss_dcf_eval_host(int party, int n, int out_bits, uint64_t count, uint64_t ld,
                      const uint8_t* seed0, const uint8_t* scw, const uint8_t* tcw,
                      const uint64_t* sigma_cw, const uint64_t* leaf_cw, const uint64_t* x_host,
                      uint64_t* out_host, uint64_t* x_dev, uint64_t* out_dev, uint64_t chunk,
                      uint64_t* stage, void* stream_a, void* stream_b) {
    if (ld < count) return set_err(kEinval, "level stride ld must be >= count%s");
    const HostPipe hp{x_host, out_host, x_dev, out_dev, chunk,
                      {(cudaStream_t)stream_a, (cudaStream_t)stream_b}, stage};
    return run_host_pipe(hp, count, [&](uint64_t lo, uint64_t m, const uint64_t* xd, uint64_t* od,
                                        cudaStream_t s) {
        return launch_dcf_eval(party, n, out_bits, m, ld, seed0 + 16 * lo, scw + 16 * lo, tcw + lo,
                               sigma_cw + lo, leaf_cw + lo, xd, nullptr, nullptr, od, nullptr, s);
    });
}

int fss_dpf_eval_host(int party, int n, uint64_t count, uint64_t ld, const uint8_t* seed0,
                      const uint8_t* scw, const uint8_t* tcw, const uint64_t* cw_final,
                      const uint64_t* x_host, uint64_t* out_host, uint64_t* x_dev, uint64_t* out_dev,
                      uint64_t chunk, uint64_t* stage, void* stream_a, void* stream_b) {
    if (ld < count) return set_err(kEinval, "level stride ld must be >= count%s");
    const HostPipe hp{x_host, out_host, x_dev, out_dev, chunk,
                      {(cudaStream_t)stream_a, (cudaStream_t)stream_b}, stage};
    return run_host_pipe(hp, count, [&](uint64_t lo, uint64_t m, const uint64_t* xd, uint64_t* od,
                                        cudaStream_t s) {
        return launch_dpf_eval(party, n, m, ld, seed0 + 16 * lo, scw + 16 * lo, tcw + lo,
                               cw_final + lo, xd, nullptr, nullptr, od, s);
    });
}

int fss_dcf_eval_masked(int party, int n, int out_bits, uint64_t count, uint64_t ld,
                        const uint8_t* seed0, const uint8_t* scw, const uint8_t* tcw,
                        const uint64_t* sigma_cw, const uint64_t* leaf_cw, const void* m_own,
                        const void* m_peer, uint64_t* out, void* stream) {
    return launch_dcf_eval(party, n, out_bits, count, ld, seed0, scw, tcw, sigma_cw, leaf_cw, nullptr,
                           m_own, m_peer, out, nullptr, stream);
}

int fss_dcf_eval_packed(int party, int n, uint64_t count, const uint8_t* payload, const uint64_t* x,
                        const void* m_own, const void* m_peer, uint64_t* out, void* stream) {
    if (party != 0 && party != 1) return set_err(kEinval, "party must be 0 or 1%s");
    if (n < 1 || n > 63) return set_err(kEinval, "n out of range%s");
    if (count == 0) return kOk;
    if (!x && (!m_own || !m_peer)) return set_err(kEinval, "need x or both masked messages%s");
    FSS_REQUIRE(payload, out);
    void (*kern)(int, int, uint64_t, const uint8_t*, const uint64_t*, const void*, const void*, uint64_t*);
    switch ((n + 7) / 8) {
        case 1: kern = dcf_eval_packed_kernel<1>; break;
        case 2: kern = dcf_eval_packed_kernel<2>; break;
        case 3: kern = dcf_eval_packed_kernel<3>; break;
        case 4: kern = dcf_eval_packed_kernel<4>; break;
        case 5: kern = dcf_eval_packed_kernel<5>; break;
        case 6: kern = dcf_eval_packed_kernel<6>; break;
        case 7: kern = dcf_eval_packed_kernel<7>; break;
        default: kern = dcf_eval_packed_kernel<8>; break;
    }
    int sms;
    if (int rc = prep_launch(kern, &sms)) return rc;
    int threads;
    const int grid = eval_grid(count, sms, &threads);
    kern<<<grid, threads, fssb::kTableBytes, (cudaStream_t)stream>>>(party, n, count, payload, x, m_own, m_peer,
                                                                      out);
    return check_launch();
}

int fss_dpf_eval_packed(int party, int n, uint64_t count, const uint8_t* payload, const uint64_t* x,
                        const void* m_own, const void* m_peer, uint64_t* out, void* stream) {
    if (party != 0 && party != 1) return set_err(kEinval, "party must be 0 or 1%s");
    if (n < 1 || n > 64) return set_err(kEinval, "n out of range%s");
    if (count == 0) return kOk;
    if (!x && (!m_own || !m_peer)) return set_err(kEinval, "need x or both masked messages%s");
    FSS_REQUIRE(payload, out);
    void (*kern)(int, int, uint64_t, const uint8_t*, const uint64_t*, const void*, const void*, uint64_t*);
    switch ((n + 7) / 8) {
        case 1: kern = dpf_eval_packed_kernel<1>; break;
        case 2: kern = dpf_eval_packed_kernel<2>; break;
        case 3: kern = dpf_eval_packed_kernel<3>; break;
        case 4: kern = dpf_eval_packed_kernel<4>; break;
        case 5: kern = dpf_eval_packed_kernel<5>; break;
        case 6: kern = dpf_eval_packed_kernel<6>; break;
        case 7: kern = dpf_eval_packed_kernel<7>; break;
        default: kern = dpf_eval_packed_kernel<8>; break;
    }
    int sms;
    if (int rc = prep_launch(kern, &sms)) return rc;
    int threads;
    const int grid = eval_grid(count, sms, &threads);
    kern<<<grid, threads, fssb::kTableBytes, (cudaStream_t)stream>>>(party, n, count, payload, x, m_own, m_peer,
                                                                      out);
    return check_launch();
}

int fss_dpf_keygen(int n, uint64_t count, const uint64_t* alpha, const uint64_t* alpha0,
                   const uint8_t* s0, const uint8_t* s1, uint8_t* scw, uint8_t* tcw,
                   uint64_t* cw_final, uint64_t* alpha1, void* stream) {
    if (n < 1 || n > 64) return set_err(kEinval, "n out of range%s");
    if (count == 0) return kOk;
    FSS_REQUIRE(alpha, alpha0, s0, s1, scw, tcw, cw_final, alpha1);
    int sms;
    if (FSSB_KEYGEN_PAIR_DPF) {
        if (int rc = prep_launch(keygen_pair_kernel<false>, &sms)) return rc;
        {
            int threads;
            const int grid = balanced_grid(2 * count, sms, kPairKeygenThreads, &threads);
            keygen_pair_kernel<false><<<grid, threads, fssb::kTableBytes, (cudaStream_t)stream>>>(
                n, n, count, alpha, alpha0, s0, s1, scw, tcw, nullptr, nullptr, cw_final, alpha1);
            return check_launch();
        }
    }
    if (int rc = prep_launch(dpf_keygen_kernel, &sms)) return rc;
    int threads;
    const int grid = balanced_grid(count, sms, kKeygenThreads, &threads);
    dpf_keygen_kernel<<<grid, threads, fssb::kTableBytes, (cudaStream_t)stream>>>(
        n, count, alpha, alpha0, s0, s1, scw, tcw, cw_final, alpha1);
    return check_launch();
}

int fss_dcf_keygen(int n, int out_bits, uint64_t count, const uint64_t* alpha,
                   const uint64_t* alpha0, const uint8_t* s0, const uint8_t* s1, uint8_t* scw,
                   uint8_t* tcw, uint64_t* sigma_cw, uint64_t* leaf_cw, uint64_t* alpha1,
                   void* stream) {
    if (n < 1 || n > 63 || out_bits < n || out_bits > 63)
        return set_err(kEinval, "need 1 <= n <= out_bits <= 63%s");
    if (count == 0) return kOk;
    FSS_REQUIRE(alpha, alpha0, s0, s1, scw, tcw, sigma_cw, leaf_cw, alpha1);
    int sms;
    if (FSSB_KEYGEN_PAIR_DCF) {
        auto kern = FSSB_W32 && out_bits <= 32 ? keygen_pair_kernel<true, true> : keygen_pair_kernel<true, false>;
        if (int rc = prep_launch(kern, &sms)) return rc;
        int threads;
        const int grid = balanced_grid(2 * count, sms, kPairKeygenThreads, &threads);
        kern<<<grid, threads, fssb::kTableBytes, (cudaStream_t)stream>>>(
            n, out_bits, count, alpha, alpha0, s0, s1, scw, tcw, sigma_cw, leaf_cw, nullptr, alpha1);
        return check_launch();
    }
    if (int rc = prep_launch(dcf_keygen_kernel, &sms)) return rc;
    int threads;
    const int grid = balanced_grid(count, sms, kKeygenThreads, &threads);
    dcf_keygen_kernel<<<grid, threads, fssb::kTableBytes, (cudaStream_t)stream>>>(
        n, out_bits, count, alpha, alpha0, s0, s1, scw, tcw, sigma_cw, leaf_cw, alpha1);
    return check_launch();
}

}  // extern "C"

namespace {

// One launch over the raw outputs [r_begin, r_end) of plan P.
int launch_tape_range(TapePlan P, uint64_t r_begin, uint64_t r_end, int emit_buffered, uint64_t* alpha,
                      uint64_t* alpha0, uint8_t* s0, uint8_t* s1, void* stream) {
    if (r_end <= r_begin && !emit_buffered) return kOk;
    P.r_begin = r_begin;
    P.r_end = r_end > r_begin ? r_end : r_begin;
    P.emit_buffered = emit_buffered;
    const uint64_t threads = (P.r_end - P.r_begin + kChunk - 1) / kChunk;
    const int bs = 256;
    const uint64_t grid = threads ? (threads + bs - 1) / bs : 1;
    pcg64_tape_kernel<<<(unsigned)grid, bs, 0, (cudaStream_t)stream>>>(P, alpha, alpha0, s0, s1);
    return check_launch();
}

// The tape of `count` elements (fss._sample_tape, fss.py:292-303), of which
// only the element slice [lo, lo + m) is materialised (outputs indexed from 0).
// A rank of a sharded dealer draws its slice of the global tape this way: the
// raw PCG64 outputs feeding that slice are reached by LCG jump-ahead, so every
// rank's keys equal the corresponding slice of a single-device keygen(count).
// st_out always describes the state after the WHOLE tape.
int launch_tape(const fss_pcg64_state* st, int n, uint64_t count, int draw_alpha, int draw_alpha0,
                uint64_t* alpha, uint64_t* alpha0, uint8_t* s0, uint8_t* s1, fss_pcg64_state* st_out,
                void* stream, uint64_t lo = 0, uint64_t m = ~0ULL) {
    if (m == ~0ULL) m = count - lo;
    if (lo > count || m > count - lo) return set_err(kEinval, "tape slice out of range%s");
    if (!st || (m && (!s0 || !s1 || (draw_alpha && !alpha) || (draw_alpha0 && !alpha0))))
        return set_err(kEinval, "null pointer%s");
    TapePlan P;
    P.state_lo = st->state_lo; P.state_hi = st->state_hi;
    P.inc_lo = st->inc_lo; P.inc_hi = st->inc_hi;
    P.n = n; P.count = count; P.draw_alpha = draw_alpha ? 1 : 0;
    P.draw_alpha0 = draw_alpha0 ? 1 : 0;
    P.has_uint32 = st->has_uint32 ? 1 : 0;
    P.uinteger = st->uinteger;
    P.lo = lo; P.hi = lo + m;
    const uint64_t na = (P.draw_alpha ? count : 0) + (P.draw_alpha0 ? count : 0);
    if (n <= 32) {
        P.raw64 = 0;
        P.words = na + 8 * count;
    } else {
        P.raw64 = na;
        P.words = 8 * count;
    }
    const uint64_t h = (uint64_t)P.has_uint32;
    const uint64_t raw_words = P.words >= h ? (P.words - h + 1) / 2 : 0;
    const uint64_t total = P.raw64 + raw_words;
    // host-side bookkeeping for the caller's generator: raws consumed and the
    // buffered half-word left behind (numpy's has_uint32 / uinteger)
    if (st_out) {
        *st_out = *st;
        st_out->advance = total;
        const int used_buffer = (P.words > 0 && h);
        const uint64_t fresh = P.words - (used_buffer ? 1 : 0);
        st_out->has_uint32 = (P.words == 0) ? st->has_uint32 : (int)(fresh & 1);
        st_out->uinteger = 0;  // caller fills from the last raw output when has_uint32
    }
    if (m == 0) return kOk;
    if (lo == 0 && m == count)  // the whole tape: one launch over every raw output
        return launch_tape_range(P, 0, total, (int)(h && P.words > 0), alpha, alpha0, s0, s1, stream);
    // a slice: one launch per tape segment, over the raws feeding [lo, lo + m)
    auto words = [&](uint64_t a, uint64_t b) -> int {  // 32-bit words [a, b) of the stream
        const uint64_t a1 = a > h ? a : h;
        const int buffered = (int)(h && a == 0 && b > 0);
        if (b <= a1) return launch_tape_range(P, 0, 0, buffered, alpha, alpha0, s0, s1, stream);
        return launch_tape_range(P, P.raw64 + (a1 - h) / 2, P.raw64 + (b - 1 - h) / 2 + 1, buffered,
                                 alpha, alpha0, s0, s1, stream);
    };
    uint64_t seg = 0;  // start of the current segment in its stream
    if (n <= 32) {
        if (P.draw_alpha) { if (int rc = words(seg + lo, seg + lo + m)) return rc; seg += count; }
        if (P.draw_alpha0) { if (int rc = words(seg + lo, seg + lo + m)) return rc; seg += count; }
    } else {
        if (P.draw_alpha) {
            if (int rc = launch_tape_range(P, lo, lo + m, 0, alpha, alpha0, s0, s1, stream)) return rc;
            seg += count;
        }
        if (P.draw_alpha0)
            if (int rc = launch_tape_range(P, seg + lo, seg + lo + m, 0, alpha, alpha0, s0, s1, stream))
                return rc;
        seg = 0;
    }
    if (int rc = words(seg + 4 * lo, seg + 4 * (lo + m))) return rc;
    return words(seg + 4 * count + 4 * lo, seg + 4 * count + 4 * (lo + m));
}

}  // namespace

extern "C" {

int fss_pcg64_tape(const fss_pcg64_state* st, int n, uint64_t count, int draw_alpha,
                   uint64_t* alpha, uint64_t* alpha0, uint8_t* s0, uint8_t* s1,
                   fss_pcg64_state* st_out, void* stream) {
    if (n < 1 || n > 63) return set_err(kEinval, "device tape supports n <= 63%s");
    return launch_tape(st, n, count, draw_alpha, 1, alpha, alpha0, s0, s1, st_out, stream);
}

int fss_pcg64_tape_slice(const fss_pcg64_state* st, int n, uint64_t count, uint64_t lo, uint64_t m,
                         int draw_alpha, uint64_t* alpha, uint64_t* alpha0, uint8_t* s0, uint8_t* s1,
                         fss_pcg64_state* st_out, void* stream) {
    if (n < 1 || n > 63) return set_err(kEinval, "device tape supports n <= 63%s");
    return launch_tape(st, n, count, draw_alpha, 1, alpha, alpha0, s0, s1, st_out, stream, lo, m);
}

int fss_pcg64_seeds(const fss_pcg64_state* st, uint64_t count, uint8_t* s0, uint8_t* s1,
                    fss_pcg64_state* st_out, void* stream) {
    return launch_tape(st, 32, count, 0, 0, nullptr, nullptr, s0, s1, st_out, stream);
}

int fss_mask_stream(uint64_t seed_lo, uint64_t seed_hi, uint64_t round_idx, uint64_t count,
                    int n_bits, uint64_t* out, void* stream) {
    if (n_bits < 1 || n_bits > 64) return set_err(kEinval, "ring width out of range%s");
    if (count == 0) return kOk;
    int sms;
    if (int rc = prep_launch(mask_stream_kernel, &sms)) return rc;
    const uint64_t blocks = (count + 3) / 4;
    const U4 seed = U4{(uint32_t)seed_lo, (uint32_t)(seed_lo >> 32), (uint32_t)seed_hi,
                       (uint32_t)(seed_hi >> 32)};
    int threads;
    const int grid = balanced_grid(blocks, sms, kKeygenThreads, &threads);
    mask_stream_kernel<<<grid, threads, fssb::kTableBytes,
                         (cudaStream_t)stream>>>(seed, round_idx, blocks, count, ring_mask_host(n_bits),
                                                 out);
    return check_launch();
}

int fss_pcg64_ring_random(const fss_pcg64_state* st, int n_bits, uint64_t count, uint64_t* out,
                          fss_pcg64_state* st_out, void* stream) {
    if (n_bits < 1 || n_bits > 64) return set_err(kEinval, "ring width out of range%s");
    if (!st || (count && !out)) return set_err(kEinval, "null pointer%s");
    TapePlan P;
    P.state_lo = st->state_lo; P.state_hi = st->state_hi;
    P.inc_lo = st->inc_lo; P.inc_hi = st->inc_hi;
    P.n = n_bits; P.count = count; P.draw_alpha = 0; P.draw_alpha0 = 0;
    P.has_uint32 = st->has_uint32 ? 1 : 0;
    P.uinteger = st->uinteger;
    P.raw64 = count;
    P.words = count;
    P.lo = 0; P.hi = count; P.r_begin = 0; P.r_end = 0; P.emit_buffered = 0;  // unused here
    const uint64_t h = (uint64_t)P.has_uint32;
    const uint64_t fresh = count > h ? count - h : 0;        // words drawn from new outputs
    if (st_out) {
        *st_out = *st;
        st_out->advance = count + (fresh + 1) / 2;
        st_out->has_uint32 = count == 0 ? st->has_uint32 : (int)(fresh & 1);
        st_out->uinteger = 0;  // caller fills from the last raw output when has_uint32
    }
    if (count == 0) return kOk;
    const uint64_t threads = (count + kChunk - 1) / kChunk;
    const int bs = 256;
    pcg64_ring_kernel<<<(unsigned)((threads + bs - 1) / bs), bs, 0, (cudaStream_t)stream>>>(P, out);
    return check_launch();
}

}  // extern "C"

namespace fssb {
namespace {
thread_local char g_err[512] = {0};
}
int set_error(int code, const char* msg) {
    strncpy(g_err, msg, sizeof(g_err) - 1);
    g_err[sizeof(g_err) - 1] = 0;
    return code;
}
const char* last_error() { return g_err; }
}  // namespace fssb
