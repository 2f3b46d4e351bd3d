// Bitsliced fixed-key AES-128 (the design SURVEY.md §8d proposed), kept as a
// measured alternative to the T-table kernels (aes_ttable.cuh).
//
// One thread encrypts 32 blocks at once: state word x[8*b + k] holds bit k
// (LSB = 0) of state byte b for all 32 blocks (bit j of the word = block j).
//  * AddRoundKey with a compile-time key is a conditional NOT per slice, which
//    folds into the neighbouring LOP3s (free).
//  * SubBytes is the Boyar-Peralta S-box circuit (32 AND + XOR/XNOR; verified
//    exhaustively against the S-box by tests/test_bitsliced_host.py).
//  * ShiftRows is register renaming; MixColumns is XOR networks on slices.
//  * In/out transposition: four 32x32 bit-matrix transposes per 32 blocks.
// Everything is __host__ __device__ so the same code is unit-tested on the
// CPU (tests/test_bitsliced_host.py builds it with g++).
#pragma once
#include <stdint.h>

#include "aes_consts.h"

#ifndef __CUDACC__
#define FSSB_HD inline
#else
#define FSSB_HD __host__ __device__ __forceinline__
#endif

namespace fssb {
namespace bs {

// 32x32 bit-matrix transpose in place: afterwards bit j of A[i] = bit i of the
// original A[j] (Hacker's Delight 7-3, indices mirrored for LSB-first bits).
FSSB_HD void transpose32(uint32_t* A) {
    uint32_t m = 0x0000FFFFu;
#pragma unroll
    for (int j = 16; j != 0; j >>= 1, m ^= (m << j)) {
#pragma unroll
        for (int k = 0; k < 32; k = ((k | j) + 1) & ~j) {
            const uint32_t t = ((A[k] >> j) ^ A[k | j]) & m;
            A[k] ^= t << j;
            A[k | j] ^= t;
        }
    }
}

// Boyar-Peralta S-box on the 8 slices of one byte (in/out: s[k] = bit k, LSB 0).
FSSB_HD void sbox(uint32_t* s) {
    const uint32_t U0 = s[7], U1 = s[6], U2 = s[5], U3 = s[4], U4 = s[3], U5 = s[2], U6 = s[1],
                   U7 = s[0];
    const uint32_t T1 = U0 ^ U3, T2 = U0 ^ U5, T3 = U0 ^ U6, T4 = U3 ^ U5, T5 = U4 ^ U6;
    const uint32_t T6 = T1 ^ T5, T7 = U1 ^ U2, T8 = U7 ^ T6, T9 = U7 ^ T7, T10 = T6 ^ T7;
    const uint32_t T11 = U1 ^ U5, T12 = U2 ^ U5, T13 = T3 ^ T4, T14 = T6 ^ T11, T15 = T5 ^ T11;
    const uint32_t T16 = T5 ^ T12, T17 = T9 ^ T16, T18 = U3 ^ U7, T19 = T7 ^ T18, T20 = T1 ^ T19;
    const uint32_t T21 = U6 ^ U7, T22 = T7 ^ T21, T23 = T2 ^ T22, T24 = T2 ^ T10, T25 = T20 ^ T17;
    const uint32_t T26 = T3 ^ T16, T27 = T1 ^ T12;
    const uint32_t M1 = T13 & T6, M2 = T23 & T8, M3 = T14 ^ M1, M4 = T19 & U7, M5 = M4 ^ M1;
    const uint32_t M6 = T3 & T16, M7 = T22 & T9, M8 = T26 ^ M6, M9 = T20 & T17, M10 = M9 ^ M6;
    const uint32_t M11 = T1 & T15, M12 = T4 & T27, M13 = M12 ^ M11, M14 = T2 & T10, M15 = M14 ^ M11;
    const uint32_t M16 = M3 ^ M2, M17 = M5 ^ T24, M18 = M8 ^ M7, M19 = M10 ^ M15, M20 = M16 ^ M13;
    const uint32_t M21 = M17 ^ M15, M22 = M18 ^ M13, M23 = M19 ^ T25, M24 = M22 ^ M23;
    const uint32_t M25 = M22 & M20, M26 = M21 ^ M25, M27 = M20 ^ M21, M28 = M23 ^ M25;
    const uint32_t M29 = M28 & M27, M30 = M26 & M24, M31 = M20 & M23, M32 = M27 & M31;
    const uint32_t M33 = M27 ^ M25, M34 = M21 & M22, M35 = M24 & M34, M36 = M24 ^ M25;
    const uint32_t M37 = M21 ^ M29, M38 = M32 ^ M33, M39 = M23 ^ M30, M40 = M35 ^ M36;
    const uint32_t M41 = M38 ^ M40, M42 = M37 ^ M39, M43 = M37 ^ M38, M44 = M39 ^ M40;
    const uint32_t M45 = M42 ^ M41;
    const uint32_t M46 = M44 & T6, M47 = M40 & T8, M48 = M39 & U7, M49 = M43 & T16;
    const uint32_t M50 = M38 & T9, M51 = M37 & T17, M52 = M42 & T15, M53 = M45 & T27;
    const uint32_t M54 = M41 & T10, M55 = M44 & T13, M56 = M40 & T23, M57 = M39 & T19;
    const uint32_t M58 = M43 & T3, M59 = M38 & T22, M60 = M37 & T20, M61 = M42 & T1;
    const uint32_t M62 = M45 & T4, M63 = M41 & T2;
    const uint32_t L0 = M61 ^ M62, L1 = M50 ^ M56, L2 = M46 ^ M48, L3 = M47 ^ M55;
    const uint32_t L4 = M54 ^ M58, L5 = M49 ^ M61, L6 = M62 ^ L5, L7 = M46 ^ L3;
    const uint32_t L8 = M51 ^ M59, L9 = M52 ^ M53, L10 = M53 ^ L4, L11 = M60 ^ L2;
    const uint32_t L12 = M48 ^ M51, L13 = M50 ^ L0, L14 = M52 ^ M61, L15 = M55 ^ L1;
    const uint32_t L16 = M56 ^ L0, L17 = M57 ^ L1, L18 = M58 ^ L8, L19 = M63 ^ L4;
    const uint32_t L20 = L0 ^ L1, L21 = L1 ^ L7, L22 = L3 ^ L12, L23 = L18 ^ L2;
    const uint32_t L24 = L15 ^ L9, L25 = L6 ^ L10, L26 = L7 ^ L9, L27 = L8 ^ L10;
    const uint32_t L28 = L11 ^ L14, L29 = L11 ^ L17;
    s[7] = L6 ^ L24;
    s[6] = ~(L16 ^ L26);
    s[5] = ~(L19 ^ L28);
    s[4] = L6 ^ L21;
    s[3] = L20 ^ L22;
    s[2] = L25 ^ L29;
    s[1] = ~(L13 ^ L27);
    s[0] = ~(L6 ^ L23);
}

template <int KEY, int ROUND>
FSSB_HD void add_round_key(uint32_t* x) {
#pragma unroll
    for (int b = 0; b < 16; b++) {
        const uint32_t kb = (kRK[KEY][4 * ROUND + b / 4] >> (8 * (b % 4))) & 0xFFu;
#pragma unroll
        for (int k = 0; k < 8; k++)
            if ((kb >> k) & 1u) x[8 * b + k] = ~x[8 * b + k];
    }
}

// ShiftRows: new byte (row r, col c) = old byte (row r, col c + r); byte b = 4c + r.
FSSB_HD void shift_rows(const uint32_t* x, uint32_t* y) {
#pragma unroll
    for (int c = 0; c < 4; c++)
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int k = 0; k < 8; k++) y[8 * (4 * c + r) + k] = x[8 * (4 * ((c + r) & 3) + r) + k];
}

// MixColumns on one column (a: 4 bytes x 8 slices, in place):
// out_i = xtime(a_i ^ a_{i+1}) ^ a_{i+1} ^ a_{i+2} ^ a_{i+3}
FSSB_HD void mix_column(uint32_t* a) {
    uint32_t o[32];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const uint32_t* a0 = a + 8 * i;
        const uint32_t* a1 = a + 8 * ((i + 1) & 3);
        const uint32_t* a2 = a + 8 * ((i + 2) & 3);
        const uint32_t* a3 = a + 8 * ((i + 3) & 3);
        uint32_t t[8], r[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            t[k] = a0[k] ^ a1[k];
            r[k] = a1[k] ^ a2[k] ^ a3[k];
        }
        o[8 * i + 0] = t[7] ^ r[0];
        o[8 * i + 1] = t[0] ^ t[7] ^ r[1];
        o[8 * i + 2] = t[1] ^ r[2];
        o[8 * i + 3] = t[2] ^ t[7] ^ r[3];
        o[8 * i + 4] = t[3] ^ t[7] ^ r[4];
        o[8 * i + 5] = t[4] ^ r[5];
        o[8 * i + 6] = t[5] ^ r[6];
        o[8 * i + 7] = t[6] ^ r[7];
    }
#pragma unroll
    for (int k = 0; k < 32; k++) a[k] = o[k];
}

template <int KEY, int ROUND>
FSSB_HD void round_(uint32_t* x) {
#pragma unroll
    for (int b = 0; b < 16; b++) sbox(x + 8 * b);
    uint32_t y[128];
    shift_rows(x, y);
    if (ROUND < 10) {
#pragma unroll
        for (int c = 0; c < 4; c++) mix_column(y + 32 * c);
    }
#pragma unroll
    for (int k = 0; k < 128; k++) x[k] = y[k];
    add_round_key<KEY, ROUND>(x);
}

// AES-128 under fixed key KEY (0..2 = prg.CIPHER_KEYS) on 32 bitsliced blocks.
template <int KEY>
FSSB_HD void encrypt(uint32_t* x) {
    add_round_key<KEY, 0>(x);
    round_<KEY, 1>(x);
    round_<KEY, 2>(x);
    round_<KEY, 3>(x);
    round_<KEY, 4>(x);
    round_<KEY, 5>(x);
    round_<KEY, 6>(x);
    round_<KEY, 7>(x);
    round_<KEY, 8>(x);
    round_<KEY, 9>(x);
    round_<KEY, 10>(x);
}

// 32 blocks (w[j*4 + c] = little-endian word c of block j) -> slices x[128].
FSSB_HD void to_slices(const uint32_t* w, uint32_t* x) {
#pragma unroll
    for (int c = 0; c < 4; c++) {
        uint32_t* A = x + 32 * c;
#pragma unroll
        for (int j = 0; j < 32; j++) A[j] = w[4 * j + c];
        transpose32(A);
    }
}

FSSB_HD void from_slices(uint32_t* x, uint32_t* w) {
#pragma unroll
    for (int c = 0; c < 4; c++) {
        uint32_t* A = x + 32 * c;
        transpose32(A);
#pragma unroll
        for (int j = 0; j < 32; j++) w[4 * j + c] = A[j];
    }
}

}  // namespace bs
}  // namespace fssb
