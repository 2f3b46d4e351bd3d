/*
 * ariann_fss.h -- C ABI of the B200 (sm_100a) FSS hot path.
 *
 * Drop-in boundary for AriaNN's function-secret-sharing path
 * (reference: /root/reference/pkg/src/ariann/{prg,fss}.py). The reference is
 * pure Python + numpy, so its "FFI" is the Python module surface; each entry
 * point below replaces the body of one reference function and is bound from
 * Python with ctypes (paper_2006_04593_b200/_lib.py).
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer (caller-owned; the library never keeps
 *     it after return). Layouts are the reference's in-memory struct-of-arrays
 *     layout (fss.py:71-154): seeds (count,16) u8; scw (n,ld,16) u8; tcw (n,ld)
 *     u8; sigma_cw (n,ld) u64; leaf_cw (n+1,ld) u64; ring values u64 masked to
 *     their ring width. `ld` is the element stride between levels (== count for
 *     a freshly generated batch, larger for a column slice of a bigger batch).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream). Calls are
 *     asynchronous and reentrant; there is no global mutable state except the
 *     thread-local error string.
 *   - Return 0 on success; FSS_EINVAL (-> Python ValueError) or FSS_ECUDA
 *     (-> RuntimeError); fss_last_error() gives the calling thread's message.
 *     Arguments -- ranges, party, and NULL for any required buffer when
 *     count > 0 -- are validated before any CUDA call, so a bad call never
 *     faults inside a kernel (which would poison the process's CUDA context).
 */
#ifndef ARIANN_FSS_H
#define ARIANN_FSS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSS_ABI_VERSION 6
#define FSS_OK 0
#define FSS_EINVAL 1
#define FSS_ECUDA 2

/* numpy PCG64 bit-generator state (Generator.bit_generator.state) */
typedef struct {
    uint64_t state_lo, state_hi; /* 128-bit LCG state */
    uint64_t inc_lo, inc_hi;     /* 128-bit increment */
    int32_t has_uint32;          /* buffered 32-bit half-word present */
    uint32_t uinteger;           /* the buffered half-word */
    uint64_t advance;            /* out: 64-bit outputs consumed */
} fss_pcg64_state;

const char* fss_last_error(void);
int fss_abi_version(void);

/* prg.expand (prg.py:43-60): out[e, 16b:16b+16] = AES_{k_b}(seeds[e]) ^ seeds[e],
 * b < out_blocks in {2,3}; seeds are used as given (top bit not cleared). */
int fss_aes_mmo_expand(const uint8_t* seeds, uint64_t count, int out_blocks, uint8_t* out,
                       void* stream);

/* prg.mask_stream (prg.py:128-147): count ring elements mod 2^n_bits of the
 * aggregation-mask stream for a 16-byte seed (seed_lo = LE bytes 0..7,
 * seed_hi = bytes 8..15) and a round counter; block i = seed ^ (round || i),
 * top bit cleared, 2-block MMO expansion -> 4 u64 lanes. */
int fss_mask_stream(uint64_t seed_lo, uint64_t seed_hi, uint64_t round_idx, uint64_t count,
                    int n_bits, uint64_t* out, void* stream);

/* fss._sample_tape (fss.py:292-303) through numpy's PCG64 Generator
 * (_uniform_ring fss.py:47-51, random_seeds prg.py:36-40) for 1 <= n <= 63:
 * draws alpha (if draw_alpha), alpha0, s0, s1 exactly as numpy would from `st`.
 * st_out receives the number of 64-bit outputs consumed (`advance`) and the
 * resulting has_uint32 flag; the caller advances its generator accordingly. */
int fss_pcg64_tape(const fss_pcg64_state* st, int n, uint64_t count, int draw_alpha,
                   uint64_t* alpha, uint64_t* alpha0, uint8_t* s0, uint8_t* s1,
                   fss_pcg64_state* st_out, void* stream);

/* Element slice [lo, lo + m) of the tape fss_pcg64_tape would draw for
 * `count` elements, written from index 0 of each output (alpha, alpha0: m
 * words; s0, s1: m x 16 bytes). Only the PCG64 outputs feeding the slice are
 * generated (LCG jump-ahead), so one rank of a sharded dealer produces exactly
 * its slice of the single-device tape. st_out describes the
 * generator after the WHOLE count-element tape, so every rank advances its copy
 * of the generator identically. New (no reference counterpart): the
 * reference's dealer is single-process (dealer.py:96-103). */
int fss_pcg64_tape_slice(const fss_pcg64_state* st, int n, uint64_t count, uint64_t lo, uint64_t m,
                         int draw_alpha, uint64_t* alpha, uint64_t* alpha0, uint8_t* s0, uint8_t* s1,
                         fss_pcg64_state* st_out, void* stream);

/* The two random_seeds draws of _sample_tape alone (prg.py:36-40; s0 then s1)
 * -- the tail of the n = 64 tape, whose alpha / alpha0 are drawn by
 * fss_pcg64_ring_random (fss._uniform_ring's n == 64 branch, fss.py:48-50). */
int fss_pcg64_seeds(const fss_pcg64_state* st, uint64_t count, uint8_t* s0, uint8_t* s1,
                    fss_pcg64_state* st_out, void* stream);

/* RingTensor.random (ring.py:61-65) through numpy's PCG64 Generator:
 * out[i] = ((integers(0, 2^63)[i] << 1) | integers(0, 2)[i]) mod 2^n_bits,
 * bit-identical to the reference's draws (both the 64-bit and the buffered
 * 32-bit stream). st_out as for fss_pcg64_tape. Used for Beaver triples and
 * share() so the whole dealer runs on device. */
int fss_pcg64_ring_random(const fss_pcg64_state* st, int n_bits, uint64_t count, uint64_t* out,
                          fss_pcg64_state* st_out, void* stream);

/* fss._keygen_eq_core (fss.py:173-216). Outputs are level-major with ld=count. */
int fss_dpf_keygen(int n, uint64_t count, const uint64_t* alpha, const uint64_t* alpha0,
                   const uint8_t* s0, const uint8_t* s1, uint8_t* scw, uint8_t* tcw,
                   uint64_t* cw_final, uint64_t* alpha1, void* stream);

/* fss._keygen_cmp_core (fss.py:219-289); n <= out_bits <= 63. */
int fss_dcf_keygen(int n, int out_bits, uint64_t count, const uint64_t* alpha,
                   const uint64_t* alpha0, const uint8_t* s0, const uint8_t* s1, uint8_t* scw,
                   uint8_t* tcw, uint64_t* sigma_cw, uint64_t* leaf_cw, uint64_t* alpha1,
                   void* stream);

/* fss.eval_eq (fss.py:357-377); x reduced mod 2^n inside. */
int fss_dpf_eval(int party, int n, uint64_t count, uint64_t ld, const uint8_t* seed0,
                 const uint8_t* scw, const uint8_t* tcw, const uint64_t* cw_final, const uint64_t* x,
                 uint64_t* out, void* stream);

/* fss.eval_cmp (fss.py:380-426); levels (n+1,count) may be NULL (return_levels). */
int fss_dcf_eval(int party, int n, int out_bits, uint64_t count, uint64_t ld, const uint8_t* seed0,
                 const uint8_t* scw, const uint8_t* tcw, const uint64_t* sigma_cw,
                 const uint64_t* leaf_cw, const uint64_t* x, uint64_t* out, uint64_t* levels,
                 void* stream);

/* The two evaluations fused with the opening of the single online message of
 * sign_protocol / eq_protocol (fss.py:444-491 -> sharing.mask_and_reveal,
 * sharing.py:214-230): x[e] = (m_own[e] + m_peer[e]) mod 2^n, where m_own /
 * m_peer are the two parties' wire-packed masked inputs (width
 * fss_wire_bytes(n)). Saves the separate open kernel and the x round trip. */
int fss_dpf_eval_masked(int party, int n, uint64_t count, uint64_t ld, const uint8_t* seed0,
                        const uint8_t* scw, const uint8_t* tcw, const uint64_t* cw_final,
                        const void* m_own, const void* m_peer, uint64_t* out, void* stream);
int fss_dcf_eval_masked(int party, int n, int out_bits, uint64_t count, uint64_t ld,
                        const uint8_t* seed0, const uint8_t* scw, const uint8_t* tcw,
                        const uint64_t* sigma_cw, const uint64_t* leaf_cw, const void* m_own,
                        const void* m_peer, uint64_t* out, void* stream);

/* eval_cmp / eval_eq on HOST buffers as one native call (the pinned-host path
 * of the drop-in): [0, count) is streamed in `chunk`-element pieces over two
 * streams -- cudaMemcpyAsync of x_host (pinned) into x_dev, the eval kernel,
 * cudaMemcpyAsync of the shares into out_host (pinned) -- so copies overlap
 * kernels. stage == NULL: x_host / out_host are pinned; x_dev / out_dev are
 * caller scratch of 2 * chunk words each; returns once enqueued and the
 * caller synchronises stream_a and stream_b. stage != NULL (6 * chunk pinned
 * words; x_dev / out_dev then 3 * chunk words each): x_host / out_host may be
 * pageable (numpy arrays); chunks are staged through three slots by host
 * memcpy overlapping the GPU work, and the call returns when out_host is
 * complete (ABI 6: three staging slots, ABI 5 had two). A page-locked
 * out_host receives the shares by D2H directly (no copy-out). */
int fss_dcf_eval_host(int party, int n, int out_bits, uint64_t count, uint64_t ld,
                      const uint8_t* seed0, const uint8_t* scw, const uint8_t* tcw,
                      const uint64_t* sigma_cw, const uint64_t* leaf_cw, const uint64_t* x_host,
                      uint64_t* out_host, uint64_t* x_dev, uint64_t* out_dev, uint64_t chunk,
                      uint64_t* stage, void* stream_a, void* stream_b);
int fss_dpf_eval_host(int party, int n, uint64_t count, uint64_t ld, const uint8_t* seed0,
                      const uint8_t* scw, const uint8_t* tcw, const uint64_t* cw_final,
                      const uint64_t* x_host, uint64_t* out_host, uint64_t* x_dev, uint64_t* out_dev,
                      uint64_t chunk, uint64_t* stage, void* stream_a, void* stream_b);

/* eval_cmp / eval_eq straight from one party's ARNK payload rows (the
 * element-major container layout, LAYOUT.md:48-71; payload = count *
 * fss_arnk_elem_bytes(kind, n) bytes, as fss_arnk_pack writes them) instead of
 * unpacked level-major keys: a party that loads a key file evaluates without
 * the unpack pass. out_bits == n (packed keys carry one width). Public input:
 * x, or (x == NULL) the opening of the two wire-packed masked messages as in
 * fss_*_eval_masked. New (no reference counterpart). */
int fss_dcf_eval_packed(int party, int n, uint64_t count, const uint8_t* payload, const uint64_t* x,
                        const void* m_own, const void* m_peer, uint64_t* out, void* stream);
int fss_dpf_eval_packed(int party, int n, uint64_t count, const uint8_t* payload, const uint64_t* x,
                        const void* m_own, const void* m_peer, uint64_t* out, void* stream);

/* ARNK per-party payloads (LAYOUT.md:48-71; fss._pack_eq/_pack_cmp fss.py:540-583,
 * _unpack_eq/_unpack_cmp fss.py:553-602). kind 0 = equality, 1 = comparison.
 * payload is count * fss_arnk_elem_bytes(kind, n) bytes, element-major.
 * Level rows have stride ld >= count on both sides (ld > count addresses a
 * column range of larger arrays, e.g. one chunk of a streamed key file).
 * Unused pointers (cw_final for cmp, sigma/leaf for eq) may be NULL. */
uint64_t fss_arnk_elem_bytes(int kind, int n);
int fss_arnk_pack(int kind, int n, uint64_t count, uint64_t ld, const uint64_t* alpha_share,
                  const uint8_t* seed0, const uint8_t* scw, const uint8_t* tcw,
                  const uint64_t* cw_final, const uint64_t* sigma_cw, const uint64_t* leaf_cw,
                  uint8_t* payload, void* stream);
int fss_arnk_unpack(int kind, int n, uint64_t count, uint64_t ld, const uint8_t* payload,
                    uint64_t* alpha_share, uint8_t* seed0, uint8_t* scw, uint8_t* tcw,
                    uint64_t* cw_final, uint64_t* sigma_cw, uint64_t* leaf_cw, void* stream);

/* Elementwise ring arithmetic mod 2^n_bits (ring.py:99-129): out = op(a, b) & mask,
 * b == NULL uses b_scalar. NEG / MASK ignore b. out may alias a or b. */
#define FSS_RING_ADD 0
#define FSS_RING_SUB 1
#define FSS_RING_MUL 2
#define FSS_RING_NEG 3
#define FSS_RING_MASK 4
int fss_ring_op(int op, int n_bits, uint64_t count, const uint64_t* a, const uint64_t* b,
                uint64_t b_scalar, uint64_t* out, void* stream);

/* Wire format (sharing.py:191-207): ring values travel at the smallest
 * power-of-two width covering n_bits -- 1, 2, 4 or 8 bytes, little-endian. */
int fss_wire_bytes(int n_bits);

/* wire[i] = (a[i] op b[i]) mod 2^n_bits at wire width; op FSS_RING_ADD or
 * FSS_RING_SUB; b == NULL packs a alone. mask_and_reveal's m_j = y_j + alpha_j
 * (sharing.py:224-226), reveal's own share (sharing.py:233-242), Beaver's
 * delta_j = x_j - a_j / eps_j = y_j - b_j (beaver.py:279-281). */
int fss_wire_pack(int op, int n_bits, uint64_t count, const uint64_t* a, const uint64_t* b,
                  void* wire, void* stream);

/* out[i] = (own[i] + peer[i]) mod 2^n_bits from two wire buffers (peer may be
 * NULL): the public x = m_0 + m_1 both parties reconstruct (sharing.py:228-230). */
int fss_wire_open(int n_bits, uint64_t count, const void* own, const void* peer, uint64_t* out,
                  void* stream);

/* Elementwise Beaver product share (beaver.py:257-294 with OP_MUL), fused with
 * the opening: delta = d_own + d_peer, eps = e_own + e_peer (wire width),
 * z = delta*b + a*eps + c (+ delta*eps, party 0). */
int fss_beaver_mul(int party, int n_bits, uint64_t count, const void* delta_own,
                   const void* delta_peer, const void* eps_own, const void* eps_peer,
                   const uint64_t* a, const uint64_t* b, const uint64_t* c, uint64_t* z,
                   void* stream);

/* argmax's pairwise differences (nn_ops.py:111-114): v is (rows, m) u64;
 * out is (rows, m*(m-1)) with out[r][j*(m-1)+k] = v[r][i] - v[r][j] mod 2^n,
 * i running over the indices != j in ascending order. */
int fss_ring_pairwise(int n_bits, uint64_t rows, int m, const uint64_t* v, uint64_t* out, void* stream);

/* out[q] = (in[q*g] + ... + in[q*g+g-1] + add) mod 2^n for q < groups: argmax's
 * per-row counts (nn_ops.py:115-116) and maxpool's window sums (:174). */
int fss_ring_group_sum(int n_bits, uint64_t groups, int g, const uint64_t* in, uint64_t add, uint64_t* out,
                       void* stream);

/* CUDA IPC for the peer-memory exchange (runtime.PeerTransport): export a
 * device allocation as an opaque handle (fss_ipc_handle_bytes() bytes), map a
 * peer process's allocation (peer access enabled lazily), unmap it. Replaces
 * the byte transport under Session.exchange (runtime.py:228-257) when both
 * parties run on one node: the eval kernel then loads the peer's masked message
 * directly (fss_*_eval_masked with m_peer = the mapped pointer). */
int fss_ipc_handle_bytes(void);
int fss_ipc_alloc(uint64_t nbytes, void** dev_ptr);   /* whole allocation: exportable */
int fss_ipc_free(void* dev_ptr);
int fss_memcpy_d2d(void* dst, const void* src, uint64_t nbytes, void* stream);
int fss_ipc_get_handle(const void* dev_ptr, uint8_t* handle);
int fss_ipc_open_handle(const uint8_t* handle, void** dev_ptr);
int fss_ipc_close_handle(void* dev_ptr);

/* Host scheduling words of the in-process two-party runtime
 * (runtime.run_local_pair; the reference runs its two parties as two threads
 * over blocking queues, runtime.py:285-311). Not a reference entry point.
 * fss_host_wait first adds 1 to *bump (if not NULL) and stores pass_to into
 * *turn (if turn != NULL and pass_to >= 0), then waits -- callers drop the GIL
 * for the call -- until *word >= target and, for at most grace_s after that,
 * until *turn == me (turn NULL or me < 0: no turn condition). It spins for
 * spin_s, then yields for spin_s, then naps (<= 50 us); once *word >= target
 * it spins. Returns 0, 1 after timeout_s, FSS_EINVAL for a NULL word.
 * load / store / add are acquire / release / acq_rel atomics on one word. */
int64_t fss_host_load(const int64_t* word);
void fss_host_store(int64_t* word, int64_t value);
int64_t fss_host_add(int64_t* word, int64_t delta);
int fss_host_wait(const int64_t* word, int64_t target, int64_t* turn, int64_t me, int64_t pass_to,
                  int64_t* bump, double spin_s, double grace_s, double timeout_s);

/* Stream ordering for the in-process pair (not a reference entry point):
 * timing-free events, and fss_streams_link -- the first n_waiters of
 * (waiter0, waiter1) wait for the work queued so far on the first n_producers
 * of (producer0, producer1) (streams of the current device, 0 = the legacy
 * default stream); run_local_pair forks / joins the party streams with it. */
int fss_event_create(void** ev);
int fss_event_destroy(void* ev);
int fss_event_record(void* ev, void* stream);
int fss_stream_wait_event(void* stream, void* ev);
int fss_streams_link(void* waiter0, void* waiter1, int n_waiters, void* producer0, void* producer1,
                     int n_producers);

/* Diagnostics (not a reference entry point): on-box peak probes used as the
 * roofline denominators of the AES work. Synchronous; runs ~10 ms of probe
 * kernels on the current device. */
typedef struct {
    double lds_wavefronts_per_s;  /* conflict-free LDS.32 warp lookups, T-table access pattern */
    double lop3_lane_ops_per_s;   /* lop3.b32 lane-ops */
    double sm_clock_hz;           /* SM clock seen by the LDS probe (clock64 / globaltimer) */
    int32_t sms;
} fss_peaks;
int fss_probe_peaks(fss_peaks* out);

#ifdef __cplusplus
}
#endif

#endif /* ARIANN_FSS_H */
