/*
 * fss_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the AriaNN reference's FSS hot path
 * (/root/reference/pkg/src/ariann/{prg,fss}.py) in plain C. It exists to
 * CHECK the CUDA product path (tests/, __graft_entry__.smoke()) and to serve as
 * the timed CPU baseline in bench.py (`cpu_baseline`, `--impl reference`).
 * Nothing in paper_2006_04593_b200/ links, imports or calls it.
 *
 * Parity of this restatement is pinned (tests/test_oracle.py) against
 *   - the reference's 15 committed PRG vectors (pkg/prg_vectors.txt:3-17), and
 *   - golden fixtures produced by running the Python reference itself in the
 *     build container (tests/golden/make_golden.py, fixtures in tests/golden),
 *   - sha256 digests of the reference's keys / shares at the BASELINE sizes
 *     (DCF 2^16, DPF 2^20: tests/golden/make_large_golden.py,
 *     tests/test_large_golden.py).
 *
 * Algorithms follow the reference line by line, including its over-computation
 * (eval expands 2 / 3 blocks per level exactly as fss.py:365 / fss.py:395 do), so
 * the baseline does the reference's work, just in C:
 *   AES-128 (FIPS-197)       -- the third-party `cryptography`/OpenSSL AES used
 *                               by prg.py:15,30,57 (declared cryptography>=41,
 *                               48.0.0 in the build container). Textbook byte
 *                               implementation plus an AES-NI path for speed.
 *   oracle_expand            -- prg.expand            prg.py:43-60
 *   slice_eq / slice_cmp     -- prg.slice_eq/_cmp     prg.py:71-86, 99-119
 *   seed_to_ring             -- prg.seed_to_ring      prg.py:122-125
 *   oracle_keygen_eq         -- fss._keygen_eq_core   fss.py:173-216
 *   oracle_keygen_cmp        -- fss._keygen_cmp_core  fss.py:219-289
 *   oracle_eval_eq           -- fss.eval_eq           fss.py:357-377
 *   oracle_eval_cmp          -- fss.eval_cmp          fss.py:380-426
 *   oracle_pack_* / unpack_* -- fss._pack_/_unpack_*  fss.py:540-602
 * Element loops are parallelised with OpenMP (elements are independent; the
 * reference's "levels outer, elements vectorised" order gives identical bytes).
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#if defined(__x86_64__)
#include <immintrin.h>
#include <cpuid.h>
#endif

/* ------------------------------------------------------------------ AES */

static uint8_t SBOX[256];
static uint8_t RK[3][11][16];            /* expanded round keys for k1,k2,k3 */
static int g_init = 0;
static int g_use_ni = 0;

static uint8_t gmul(uint8_t a, uint8_t b) {
    uint8_t p = 0;
    while (b) {
        if (b & 1) p ^= a;
        a = (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0));
        b >>= 1;
    }
    return p;
}

static void build_sbox(void) {
    /* S(x) = affine(x^-1) over GF(2^8) mod x^8+x^4+x^3+x+1 (FIPS-197 5.1.1) */
    for (int x = 0; x < 256; x++) {
        uint8_t inv = 0;
        if (x) {
            for (int y = 1; y < 256; y++)
                if (gmul((uint8_t)x, (uint8_t)y) == 1) { inv = (uint8_t)y; break; }
        }
        uint8_t s = inv, r = inv;
        for (int k = 0; k < 4; k++) {
            r = (uint8_t)((r << 1) | (r >> 7));
            s ^= r;
        }
        SBOX[x] = (uint8_t)(s ^ 0x63);
    }
}

static void key_expand(const uint8_t key[16], uint8_t rk[11][16]) {
    /* FIPS-197 5.2 for Nk=4 */
    uint8_t w[44][4];
    uint8_t rcon = 1;
    for (int i = 0; i < 4; i++) memcpy(w[i], key + 4 * i, 4);
    for (int i = 4; i < 44; i++) {
        uint8_t t[4];
        memcpy(t, w[i - 1], 4);
        if (i % 4 == 0) {
            uint8_t t0 = t[0];
            t[0] = (uint8_t)(SBOX[t[1]] ^ rcon);
            t[1] = SBOX[t[2]];
            t[2] = SBOX[t[3]];
            t[3] = SBOX[t0];
            rcon = gmul(rcon, 2);
        }
        for (int k = 0; k < 4; k++) w[i][k] = (uint8_t)(w[i - 4][k] ^ t[k]);
    }
    for (int r = 0; r < 11; r++)
        for (int c = 0; c < 4; c++) memcpy(&rk[r][4 * c], w[4 * r + c], 4);
}

static int cpu_has_aesni(void) {
#if defined(__x86_64__)
    unsigned a, b, c, d;
    if (!__get_cpuid(1, &a, &b, &c, &d)) return 0;
    return (c & bit_AES) ? 1 : 0;
#else
    return 0;
#endif
}

static void oracle_init(void) {
    if (g_init) return;
    build_sbox();
    /* prg.CIPHER_KEYS: 00..0f, 10..1f, 20..2f  (prg.py:24-28, LAYOUT.md:14-21) */
    for (int k = 0; k < 3; k++) {
        uint8_t key[16];
        for (int i = 0; i < 16; i++) key[i] = (uint8_t)(16 * k + i);
        key_expand(key, RK[k]);
    }
    g_use_ni = cpu_has_aesni();
    g_init = 1;
}

/* Textbook AES-128 encryption (FIPS-197 5.1). State byte order = memory order. */
static void aes_enc_ref(int k, const uint8_t in[16], uint8_t out[16]) {
    uint8_t s[16], t[16];
    for (int i = 0; i < 16; i++) s[i] = (uint8_t)(in[i] ^ RK[k][0][i]);
    for (int r = 1; r <= 10; r++) {
        /* SubBytes + ShiftRows: row j of column c comes from column c+j */
        for (int c = 0; c < 4; c++)
            for (int j = 0; j < 4; j++) t[4 * c + j] = SBOX[s[4 * ((c + j) & 3) + j]];
        if (r != 10) {
            for (int c = 0; c < 4; c++) {
                uint8_t a0 = t[4 * c], a1 = t[4 * c + 1], a2 = t[4 * c + 2], a3 = t[4 * c + 3];
                s[4 * c + 0] = (uint8_t)(gmul(a0, 2) ^ gmul(a1, 3) ^ a2 ^ a3);
                s[4 * c + 1] = (uint8_t)(a0 ^ gmul(a1, 2) ^ gmul(a2, 3) ^ a3);
                s[4 * c + 2] = (uint8_t)(a0 ^ a1 ^ gmul(a2, 2) ^ gmul(a3, 3));
                s[4 * c + 3] = (uint8_t)(gmul(a0, 3) ^ a1 ^ a2 ^ gmul(a3, 2));
            }
        } else {
            memcpy(s, t, 16);
        }
        for (int i = 0; i < 16; i++) s[i] ^= RK[k][r][i];
    }
    memcpy(out, s, 16);
}

#if defined(__x86_64__)
__attribute__((target("aes,sse4.1")))
static void aes_enc_ni(int k, const uint8_t in[16], uint8_t out[16]) {
    __m128i x = _mm_loadu_si128((const __m128i*)in);
    x = _mm_xor_si128(x, _mm_loadu_si128((const __m128i*)RK[k][0]));
    for (int r = 1; r < 10; r++) x = _mm_aesenc_si128(x, _mm_loadu_si128((const __m128i*)RK[k][r]));
    x = _mm_aesenclast_si128(x, _mm_loadu_si128((const __m128i*)RK[k][10]));
    _mm_storeu_si128((__m128i*)out, x);
}
#endif

static inline void aes_enc(int k, const uint8_t in[16], uint8_t out[16]) {
#if defined(__x86_64__)
    if (g_use_ni) { aes_enc_ni(k, in, out); return; }
#endif
    aes_enc_ref(k, in, out);
}

/* ------------------------------------------------------------------ PRG */

/* G(s) block b = AES_{k_b}(s) XOR s   (prg.py:43-60; inputs NOT top-bit cleared) */
static inline void mmo(const uint8_t seed[16], int blocks, uint8_t* out) {
    for (int b = 0; b < blocks; b++) {
        aes_enc(b, seed, out + 16 * b);
        for (int i = 0; i < 16; i++) out[16 * b + i] ^= seed[i];
    }
}

static inline uint64_t ring_mask(int w) { return w >= 64 ? ~0ULL : ((1ULL << w) - 1); }

static inline uint64_t le64(const uint8_t* p) {
    uint64_t v;
    memcpy(&v, p, 8);
    return v;
}

/* prg.seed_to_ring prg.py:122-125 */
static inline uint64_t seed_to_ring(const uint8_t s[16], int w) { return le64(s) & ring_mask(w); }

typedef struct {
    uint8_t sl[16], sr[16];
    uint8_t tl, tr;
    uint64_t gl, gr;   /* sigma lanes (cmp only) */
    uint8_t ul, ur;    /* tau bits (cmp only) */
} slice_t;

/* prg.slice_eq prg.py:71-86 and prg.slice_cmp prg.py:99-119 */
static inline void do_slice(const uint8_t* raw, int cmp, int w, slice_t* o) {
    memcpy(o->sl, raw, 16);
    memcpy(o->sr, raw + 16, 16);
    o->tl = (uint8_t)((o->sl[15] >> 7) & 1);
    o->tr = (uint8_t)((o->sr[15] >> 7) & 1);
    o->sl[15] &= 0x7F;
    o->sr[15] &= 0x7F;
    if (cmp) {
        uint64_t l0 = le64(raw + 32), l1 = le64(raw + 40);
        o->gl = l0 & ring_mask(w);
        o->gr = l1 & ring_mask(w);
        o->ul = (uint8_t)(l0 >> 63);
        o->ur = (uint8_t)(l1 >> 63);
    }
}

static inline void xor16(uint8_t* d, const uint8_t* s) {
    for (int i = 0; i < 16; i++) d[i] ^= s[i];
}

/* ------------------------------------------------------------ public API */

int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

int oracle_aesni(void) { oracle_init(); return g_use_ni; }
void oracle_use_aesni(int on) { oracle_init(); g_use_ni = on ? cpu_has_aesni() : 0; }

void oracle_aes128(int key_idx, const uint8_t* in, uint8_t* out) {
    oracle_init();
    aes_enc_ref(key_idx, in, out);
}

void oracle_round_keys(int key_idx, uint8_t* out176) {
    oracle_init();
    memcpy(out176, RK[key_idx], 176);
}

/* prg.expand prg.py:43-60 */
void oracle_expand(const uint8_t* seeds, uint64_t N, int blocks, uint8_t* out) {
    oracle_init();
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)N; e++) mmo(seeds + 16 * e, blocks, out + (uint64_t)e * 16 * blocks);
}

/* fss._keygen_eq_core fss.py:173-216 */
void oracle_keygen_eq(int n, uint64_t N, const uint64_t* alpha, const uint64_t* alpha0,
                      const uint8_t* s0_init, const uint8_t* s1_init,
                      uint8_t* scw, uint8_t* tcw, uint64_t* cw_final, uint64_t* alpha1) {
    oracle_init();
    const uint64_t mask = ring_mask(n);
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)N; e++) {
        uint8_t s[2][16], raw[2][32];
        uint8_t t[2] = {0, 1};
        memcpy(s[0], s0_init + 16 * e, 16);
        memcpy(s[1], s1_init + 16 * e, 16);
        for (int i = 0; i < n; i++) {
            uint8_t a = (uint8_t)((alpha[e] >> (n - 1 - i)) & 1);
            slice_t sl[2];
            for (int j = 0; j < 2; j++) {
                mmo(s[j], 2, raw[j]);
                do_slice(raw[j], 0, 0, &sl[j]);
            }
            uint8_t cw_seed[16];
            for (int b = 0; b < 16; b++)
                cw_seed[b] = a ? (uint8_t)(sl[0].sl[b] ^ sl[1].sl[b]) : (uint8_t)(sl[0].sr[b] ^ sl[1].sr[b]);
            uint8_t cw_tl = (uint8_t)(sl[0].tl ^ sl[1].tl ^ 1 ^ a);
            uint8_t cw_tr = (uint8_t)(sl[0].tr ^ sl[1].tr ^ a);
            memcpy(scw + ((uint64_t)i * N + e) * 16, cw_seed, 16);
            tcw[(uint64_t)i * N + e] = (uint8_t)(cw_tl | (cw_tr << 1));
            for (int j = 0; j < 2; j++) {
                if (t[j]) {
                    xor16(sl[j].sl, cw_seed);
                    xor16(sl[j].sr, cw_seed);
                }
                sl[j].tl ^= (uint8_t)(t[j] & cw_tl);
                sl[j].tr ^= (uint8_t)(t[j] & cw_tr);
                memcpy(s[j], a ? sl[j].sr : sl[j].sl, 16);
                t[j] = a ? sl[j].tr : sl[j].tl;
            }
        }
        uint64_t v = (1 - seed_to_ring(s[0], n) + seed_to_ring(s[1], n)) & mask;
        cw_final[e] = t[1] ? ((0 - v) & mask) : v;
        alpha1[e] = (alpha[e] - alpha0[e]) & mask;
    }
}

/* fss._keygen_cmp_core fss.py:219-289 */
void oracle_keygen_cmp(int n, int out_bits, uint64_t N, const uint64_t* alpha, const uint64_t* alpha0,
                       const uint8_t* s0_init, const uint8_t* s1_init,
                       uint8_t* scw, uint8_t* tcw, uint64_t* sigma_cw, uint64_t* leaf_cw,
                       uint64_t* alpha1) {
    oracle_init();
    const uint64_t omask = ring_mask(out_bits);
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)N; e++) {
        uint8_t s[2][16], raw[2][48];
        uint8_t t[2] = {0, 1};
        memcpy(s[0], s0_init + 16 * e, 16);
        memcpy(s[1], s1_init + 16 * e, 16);
        for (int i = 0; i < n; i++) {
            uint8_t a = (uint8_t)((alpha[e] >> (n - 1 - i)) & 1);
            slice_t sl[2];
            for (int j = 0; j < 2; j++) {
                mmo(s[j], 3, raw[j]);
                do_slice(raw[j], 1, out_bits, &sl[j]);
            }
            uint8_t cw_seed[16];
            for (int b = 0; b < 16; b++)
                cw_seed[b] = a ? (uint8_t)(sl[0].sl[b] ^ sl[1].sl[b]) : (uint8_t)(sl[0].sr[b] ^ sl[1].sr[b]);
            uint8_t cw_tl = (uint8_t)(sl[0].tl ^ sl[1].tl ^ 1 ^ a);
            uint8_t cw_tr = (uint8_t)(sl[0].tr ^ sl[1].tr ^ a);
            uint64_t cw_sig = a ? (sl[0].gr ^ sl[1].gr) : (sl[0].gl ^ sl[1].gl);
            uint8_t cw_ul = (uint8_t)(sl[0].ul ^ sl[1].ul ^ a);
            uint8_t cw_ur = (uint8_t)(sl[0].ur ^ sl[1].ur ^ 1 ^ a);
            memcpy(scw + ((uint64_t)i * N + e) * 16, cw_seed, 16);
            tcw[(uint64_t)i * N + e] = (uint8_t)(cw_tl | (cw_tr << 1) | (cw_ul << 2) | (cw_ur << 3));
            sigma_cw[(uint64_t)i * N + e] = cw_sig;
            for (int j = 0; j < 2; j++) {
                if (t[j]) {
                    xor16(sl[j].sl, cw_seed);
                    xor16(sl[j].sr, cw_seed);
                    sl[j].gl ^= cw_sig;
                    sl[j].gr ^= cw_sig;
                }
                sl[j].tl ^= (uint8_t)(t[j] & cw_tl);
                sl[j].tr ^= (uint8_t)(t[j] & cw_tr);
                sl[j].ul ^= (uint8_t)(t[j] & cw_ul);
                sl[j].ur ^= (uint8_t)(t[j] & cw_ur);
            }
            /* leaf from the exit side (not a), after correction (fss.py:268-273) */
            uint64_t g0x = a ? sl[0].gl : sl[0].gr;
            uint64_t g1x = a ? sl[1].gl : sl[1].gr;
            uint8_t u1x = a ? sl[1].ul : sl[1].ur;
            uint64_t leaf = ((uint64_t)a - g0x + g1x) & omask;
            leaf_cw[(uint64_t)i * N + e] = u1x ? ((0 - leaf) & omask) : leaf;
            for (int j = 0; j < 2; j++) {
                memcpy(s[j], a ? sl[j].sr : sl[j].sl, 16);
                t[j] = a ? sl[j].tr : sl[j].tl;
            }
        }
        uint64_t v = (1 - seed_to_ring(s[0], out_bits) + seed_to_ring(s[1], out_bits)) & omask;
        leaf_cw[(uint64_t)n * N + e] = t[1] ? ((0 - v) & omask) : v;
        alpha1[e] = (alpha[e] - alpha0[e]) & ring_mask(n);
    }
}

/* fss.eval_eq fss.py:357-377 (x already reduced mod 2^n by the caller, fss.py:347-354) */
void oracle_eval_eq(int party, int n, uint64_t N, const uint8_t* seed0, const uint8_t* scw,
                    const uint8_t* tcw, const uint64_t* cw_final, const uint64_t* x, uint64_t* out) {
    oracle_init();
    const uint64_t mask = ring_mask(n);
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)N; e++) {
        uint8_t s[16], raw[32];
        uint8_t t = (uint8_t)party;
        memcpy(s, seed0 + 16 * e, 16);
        uint64_t xe = x[e] & mask;
        for (int i = 0; i < n; i++) {
            slice_t sl;
            mmo(s, 2, raw);
            do_slice(raw, 0, 0, &sl);
            uint8_t f = tcw[(uint64_t)i * N + e];
            if (t) {
                xor16(sl.sl, scw + ((uint64_t)i * N + e) * 16);
                xor16(sl.sr, scw + ((uint64_t)i * N + e) * 16);
            }
            sl.tl ^= (uint8_t)(t & (f & 1));
            sl.tr ^= (uint8_t)(t & ((f >> 1) & 1));
            int xb = (int)((xe >> (n - 1 - i)) & 1);
            memcpy(s, xb ? sl.sr : sl.sl, 16);
            t = xb ? sl.tr : sl.tl;
        }
        uint64_t o = ((uint64_t)t * cw_final[e] + seed_to_ring(s, n)) & mask;
        out[e] = party == 1 ? ((0 - o) & mask) : o;
    }
}

/* fss.eval_cmp fss.py:380-426; levels (n+1, N) may be NULL */
void oracle_eval_cmp(int party, int n, int out_bits, uint64_t N, const uint8_t* seed0,
                     const uint8_t* scw, const uint8_t* tcw, const uint64_t* sigma_cw,
                     const uint64_t* leaf_cw, const uint64_t* x, uint64_t* out, uint64_t* levels) {
    oracle_init();
    const uint64_t nmask = ring_mask(n);
    const uint64_t mask = ring_mask(out_bits);
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)N; e++) {
        uint8_t s[16], raw[48];
        uint8_t t = (uint8_t)party;
        uint64_t acc = 0;
        memcpy(s, seed0 + 16 * e, 16);
        uint64_t xe = x[e] & nmask;
        for (int i = 0; i < n; i++) {
            slice_t sl;
            mmo(s, 3, raw);
            do_slice(raw, 1, out_bits, &sl);
            uint64_t idx = (uint64_t)i * N + e;
            uint8_t f = tcw[idx];
            if (t) {
                xor16(sl.sl, scw + idx * 16);
                xor16(sl.sr, scw + idx * 16);
            }
            sl.tl ^= (uint8_t)(t & (f & 1));
            sl.tr ^= (uint8_t)(t & ((f >> 1) & 1));
            uint64_t sig_sel = t ? sigma_cw[idx] : 0;
            sl.gl ^= sig_sel;
            sl.gr ^= sig_sel;
            sl.ul ^= (uint8_t)(t & ((f >> 2) & 1));
            sl.ur ^= (uint8_t)(t & ((f >> 3) & 1));
            int xb = (int)((xe >> (n - 1 - i)) & 1);
            uint64_t g = xb ? sl.gr : sl.gl;
            uint8_t u = xb ? sl.ur : sl.ul;
            uint64_t oi = ((uint64_t)u * leaf_cw[idx] + g) & mask;
            acc = (acc + oi) & mask;
            if (levels) levels[idx] = party == 1 ? ((0 - oi) & mask) : oi;
            memcpy(s, xb ? sl.sr : sl.sl, 16);
            t = xb ? sl.tr : sl.tl;
        }
        uint64_t idx = (uint64_t)n * N + e;
        uint64_t last = ((uint64_t)t * leaf_cw[idx] + seed_to_ring(s, out_bits)) & mask;
        acc = (acc + last) & mask;
        if (levels) levels[idx] = party == 1 ? ((0 - last) & mask) : last;
        out[e] = party == 1 ? ((0 - acc) & mask) : acc;
    }
}

/* ------------------------------------------------- ARNK element payloads */
/* LAYOUT.md:48-71; fss.py:509-602. w = ceil(n/8) LE bytes per ring value. */

static inline void put_le(uint8_t* p, uint64_t v, int w) {
    for (int b = 0; b < w; b++) p[b] = (uint8_t)(v >> (8 * b));
}

static inline uint64_t get_le(const uint8_t* p, int w) {
    uint64_t v = 0;
    for (int b = 0; b < w; b++) v |= (uint64_t)p[b] << (8 * b);
    return v;
}

uint64_t oracle_eq_elem_bytes(int n) { int w = (n + 7) / 8; return (uint64_t)(w + 16 + 17 * n + w); }
uint64_t oracle_cmp_elem_bytes(int n) { int w = (n + 7) / 8; return (uint64_t)(w + 16 + n * (17 + w) + (n + 1) * w); }

/* fss._pack_eq fss.py:540-550 */
void oracle_pack_eq(int n, uint64_t N, const uint64_t* alpha_share, const uint8_t* seed0,
                    const uint8_t* scw, const uint8_t* tcw, const uint64_t* cw_final, uint8_t* buf) {
    const int w = (n + 7) / 8;
    const uint64_t E = oracle_eq_elem_bytes(n);
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)N; e++) {
        uint8_t* p = buf + (uint64_t)e * E;
        put_le(p, alpha_share[e], w); p += w;
        memcpy(p, seed0 + 16 * e, 16); p += 16;
        for (int i = 0; i < n; i++) {
            memcpy(p, scw + ((uint64_t)i * N + e) * 16, 16); p += 16;
            *p++ = tcw[(uint64_t)i * N + e];
        }
        put_le(p, cw_final[e], w);
    }
}

/* fss._unpack_eq fss.py:553-565 */
void oracle_unpack_eq(int n, uint64_t N, const uint8_t* buf, uint64_t* alpha_share, uint8_t* seed0,
                      uint8_t* scw, uint8_t* tcw, uint64_t* cw_final) {
    const int w = (n + 7) / 8;
    const uint64_t E = oracle_eq_elem_bytes(n);
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)N; e++) {
        const uint8_t* p = buf + (uint64_t)e * E;
        alpha_share[e] = get_le(p, w); p += w;
        memcpy(seed0 + 16 * e, p, 16); p += 16;
        for (int i = 0; i < n; i++) {
            memcpy(scw + ((uint64_t)i * N + e) * 16, p, 16); p += 16;
            tcw[(uint64_t)i * N + e] = *p++;
        }
        cw_final[e] = get_le(p, w);
    }
}

/* fss._pack_cmp fss.py:568-583 */
void oracle_pack_cmp(int n, uint64_t N, const uint64_t* alpha_share, const uint8_t* seed0,
                     const uint8_t* scw, const uint8_t* tcw, const uint64_t* sigma_cw,
                     const uint64_t* leaf_cw, uint8_t* buf) {
    const int w = (n + 7) / 8;
    const uint64_t E = oracle_cmp_elem_bytes(n);
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)N; e++) {
        uint8_t* p = buf + (uint64_t)e * E;
        put_le(p, alpha_share[e], w); p += w;
        memcpy(p, seed0 + 16 * e, 16); p += 16;
        for (int i = 0; i < n; i++) {
            memcpy(p, scw + ((uint64_t)i * N + e) * 16, 16); p += 16;
            *p++ = tcw[(uint64_t)i * N + e];
            put_le(p, sigma_cw[(uint64_t)i * N + e], w); p += w;
        }
        for (int i = 0; i <= n; i++) {
            put_le(p, leaf_cw[(uint64_t)i * N + e], w); p += w;
        }
    }
}

/* fss._unpack_cmp fss.py:586-602 */
void oracle_unpack_cmp(int n, uint64_t N, const uint8_t* buf, uint64_t* alpha_share, uint8_t* seed0,
                       uint8_t* scw, uint8_t* tcw, uint64_t* sigma_cw, uint64_t* leaf_cw) {
    const int w = (n + 7) / 8;
    const uint64_t E = oracle_cmp_elem_bytes(n);
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)N; e++) {
        const uint8_t* p = buf + (uint64_t)e * E;
        alpha_share[e] = get_le(p, w); p += w;
        memcpy(seed0 + 16 * e, p, 16); p += 16;
        for (int i = 0; i < n; i++) {
            memcpy(scw + ((uint64_t)i * N + e) * 16, p, 16); p += 16;
            tcw[(uint64_t)i * N + e] = *p++;
            sigma_cw[(uint64_t)i * N + e] = get_le(p, w); p += w;
        }
        for (int i = 0; i <= n; i++) {
            leaf_cw[(uint64_t)i * N + e] = get_le(p, w); p += w;
        }
    }
}
