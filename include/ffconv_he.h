/*
 * ffconv_he.h -- C ABI of the packed RNS-BFV evaluator (drop-in boundary).
 *
 * The reference (cipherpack, pure Python) has no FFI: its operator boundary is
 * the Python class `HeContext` (/root/reference/pkg/src/cipherpack/hesim.py:186-366),
 * constructed once per run at runner.py:297.  Every entry point below backs one
 * of its methods; the Python mirror (paper_2102_03494_b200/hesim.py) binds these
 * symbols through ctypes and keeps counters, depths and error behaviour in Python.
 *
 *   fhe_encode        <- HeContext.encode            hesim.py:203-215
 *   fhe_encrypt       <- HeContext.encrypt           hesim.py:217-219
 *   fhe_ct_zero       <- HeContext.encrypt_zero      hesim.py:221-225
 *   fhe_decrypt       <- HeContext.decrypt           hesim.py:231-238
 *   fhe_rotate(_many) <- HeContext.rotate            hesim.py:244-261
 *   fhe_mul_plain(_many) <- HeContext.mul_plain      hesim.py:263-302
 *   fhe_mul_scalar    <- mul_plain by a constant     engine.py:92-97,189-195 (conv_conv)
 *   fhe_add(_many)    <- HeContext.add_cc            hesim.py:304-316
 *   fhe_add_plain     <- HeContext.add_plain         hesim.py:318-326
 *   fhe_square        <- HeContext.square            hesim.py:328-345
 *   fhe_mod_switch    <- (no reference counterpart; BASELINE cfg1 "rescale")
 *   fhe_rotate_and_sum <- HeContext.rotate_and_sum   hesim.py:347-366
 *   fhe_combine       <- combine_to_dense            packing.py:350-368
 *   fhe_ct_gemm       <- conv_conv channel sums      engine.py:178-197
 *
 * Scheme: RNS-BFV over Z[X]/(X^n+1).  One ciphertext "slot row" of the reference
 * (n_slots = N) is one batching row of a ring of degree n = 2N; row 0 and row 1
 * carry two independent slot vectors (two images).  Plaintext moduli may be a
 * list t_0..t_{T-1} (plaintext CRT): a ciphertext object holds T x R physical
 * ciphertexts laid out [T][R][2][level][n] (uint64, NTT domain, limb-major).
 *
 * Conventions (shared bit-for-bit by the CUDA library and the golden C model in
 * oracle/golden_rlwe.c) are documented in DESIGN.md section "Golden spec".
 *
 * All functions return 0 on success and a negative code on failure; the message
 * is available from fhe_last_error().  No C++ exceptions cross this boundary.
 */
#ifndef FFCONV_HE_H
#define FFCONV_HE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FHE_MAX_Q 24   /* ciphertext primes q_0..q_{L-1}             */
#define FHE_MAX_P 2    /* special (key-switching) primes              */
#define FHE_MAX_B 26   /* auxiliary primes for ct x ct multiplication */
#define FHE_MAX_T 8    /* plaintext CRT moduli                        */

#define FHE_OK 0
#define FHE_EINVAL -1
#define FHE_ENOMEM -2
#define FHE_EDEVICE -3
#define FHE_ELEVEL -4

typedef struct fhe_params {
    uint32_t log_n;   /* ring degree n = 2^log_n (2 <= log_n <= 16; 2^15, 2^16 rows run on CTA clusters); N = n/2 slots per row */
    uint32_t L;       /* ciphertext primes at the top level                              */
    uint32_t K;       /* special primes (must be 1)                                      */
    uint32_t n_aux;   /* auxiliary base size for fhe_square (0 disables squaring)         */
    uint32_t T;       /* plaintext moduli                                                */
    uint32_t flags;   /* reserved, 0                                                     */
    uint64_t q[FHE_MAX_Q];
    uint64_t p[FHE_MAX_P];
    uint64_t b[FHE_MAX_B];
    uint64_t t[FHE_MAX_T];
    uint64_t seed;    /* all key material and encryption randomness derive from it       */
    int32_t device;   /* CUDA device ordinal (ignored by the golden model)               */
    int32_t reserved;
} fhe_params;

typedef struct fhe_ctx fhe_ctx;
typedef struct fhe_ct fhe_ct;
typedef struct fhe_pt fhe_pt;
typedef struct fhe_graph fhe_graph;

const char *fhe_last_error(void);
const char *fhe_backend_name(void);   /* "cuda-sm100a" or "golden-c" */

int fhe_ctx_create(const fhe_params *params, fhe_ctx **out);
void fhe_ctx_destroy(fhe_ctx *ctx);
int fhe_sync(fhe_ctx *ctx);
/* bytes of device (or host, golden) memory held by keys and tables */
int fhe_ctx_key_bytes(fhe_ctx *ctx, uint64_t *out);
/* the context's CUDA stream (cudaStream_t), for event timing by the caller */
int fhe_ctx_stream(fhe_ctx *ctx, void **stream);
/* measured integer-pipe roofline: chained 64-bit Shoup modular multiplications
 * per second over the whole GPU (register resident, all SMs) */
int fhe_peak_modmul(fhe_ctx *ctx, uint32_t iters, double *modmul_per_s);
/* kind 0: exact-quotient Shoup chains (= fhe_peak_modmul); kind 1: the
 * approximate-quotient Shoup form the NTT butterflies issue. */
int fhe_peak_modmul_kind(fhe_ctx *ctx, uint32_t iters, int kind, double *modmul_per_s);
/* per-kernel CUDA-event profiling: when enabled, every launch is bracketed by
 * events; fhe_prof_report syncs and writes "name calls total_ms\n" lines
 * (then clears).  fhe_launch_count: kernels launched since creation. */
int fhe_prof_enable(fhe_ctx *ctx, int on);
int fhe_prof_report(fhe_ctx *ctx, char *buf, uint32_t len);
int fhe_launch_count(fhe_ctx *ctx, uint64_t *out);
/* algorithmic modular multiplications issued since creation: (n/2) log2 n per
 * row (I)NTT, 2 l (l+1) n + 2 l n per key switch (inner product + ModDown
 * scaling), 2 l n per hoisted-dot term; elementwise ops are not counted. */
int fhe_work_modmuls(fhe_ctx *ctx, double *out);
/* generate Galois keys for the given rotation steps now (otherwise lazily) */
int fhe_keygen_rotations(fhe_ctx *ctx, const uint32_t *steps, uint32_t m);

/* ---- ciphertext objects ------------------------------------------------ */
/* R row-pairs (two slot vectors each) per plaintext modulus; level in [1, L]. */
int fhe_ct_create(fhe_ctx *ctx, uint32_t R, uint32_t level, fhe_ct **out);
void fhe_ct_destroy(fhe_ct *ct);
uint32_t fhe_ct_level(const fhe_ct *ct);
uint32_t fhe_ct_rows(const fhe_ct *ct);
/* raw NTT-domain words, [T*R][2][level][n] */
int fhe_ct_read(fhe_ctx *ctx, const fhe_ct *ct, uint64_t *words);
int fhe_ct_write(fhe_ctx *ctx, fhe_ct *ct, const uint64_t *words);
/* the same words to/from caller-owned DEVICE memory (e.g. a torch CUDA tensor used as
 * an NCCL send/recv buffer); the golden model treats the pointers as host memory */
int fhe_ct_to_device(fhe_ctx *ctx, const fhe_ct *ct, void *dst);
int fhe_ct_from_device(fhe_ctx *ctx, fhe_ct *ct, const void *src);
/* transparent encryption of zero: (0, 0) */
int fhe_ct_zero(fhe_ctx *ctx, fhe_ct *ct);

/* D2D copy of the words of src into dst (same R and level), asynchronous */
int fhe_ct_copy(fhe_ctx *ctx, const fhe_ct *src, fhe_ct *dst);

/* ---- plan capture (the op sequence of a walk is data-independent) --------------
 * fhe_capture_begin starts recording every launch of the context into a CUDA graph;
 * ciphertexts created until fhe_capture_end come from a device arena of arena_bytes
 * that the graph keeps (fixed addresses across replays).  Keys, plaintexts and
 * workspaces must already exist (run the walk once first): creating them inside a
 * capture fails.  fhe_graph_launch replays the recorded work on the context's stream;
 * ciphertexts created during the capture hold the replay's results.
 * fhe_ctx_peak_bytes: the largest ciphertext memory held at once (arena sizing). */
int fhe_capture_begin(fhe_ctx *ctx, uint64_t arena_bytes);
int fhe_capture_end(fhe_ctx *ctx, fhe_graph **out);
int fhe_graph_launch(fhe_ctx *ctx, fhe_graph *graph);
int fhe_graph_nodes(fhe_graph *graph, uint64_t *out);
void fhe_graph_destroy(fhe_graph *graph);
int fhe_ctx_peak_bytes(fhe_ctx *ctx, uint64_t *out, int reset);

/* ---- plaintexts --------------------------------------------------------- */
int fhe_pt_create(fhe_ctx *ctx, fhe_pt **out);
void fhe_pt_destroy(fhe_pt *pt);
/* slots: [T][n] residues mod t_k; position r*N + i is row r, slot i */
int fhe_encode(fhe_ctx *ctx, const uint64_t *slots, fhe_pt *out);
/* [T][L][n] NTT-domain words of the lifted plaintext */
int fhe_pt_read(fhe_ctx *ctx, const fhe_pt *pt, uint64_t *words);

/* ---- client side ---------------------------------------------------------- */
/* slots: [T][R][n] residues; secret-key encryption at the top level.  Each call
 * must use a fresh nonce (the randomness is a pure function of seed, nonce and
 * the physical ciphertext index).
 * Host buffers in page-locked memory (cudaMallocHost / cudaHostRegister) make
 * fhe_encrypt and fhe_decrypt asynchronous: the copies run on the context's copy
 * stream and overlap evaluation; the input must stay untouched and the output is
 * valid only after fhe_sync().  Pageable buffers are copied synchronously. */
int fhe_encrypt(fhe_ctx *ctx, const uint64_t *slots, uint32_t nonce, fhe_ct *out);
int fhe_decrypt(fhe_ctx *ctx, const fhe_ct *ct, uint64_t *slots);
/* slots [lo, lo + cnt) of both batching rows only: out [T*R][2][cnt] residues mod t_k
 * (the logits of a network sit in slot 0; the full decrypt moves T*R*n words) */
int fhe_decrypt_slots(fhe_ctx *ctx, const fhe_ct *ct, uint32_t lo, uint32_t cnt, uint64_t *out);
/* Deferred checks (no host synchronization on the evaluation path):
 * fhe_check_zero_tail enqueues the rotate_and_sum precondition of the reference
 * (hesim.py:360-361: every slot at index >= m is zero) for every physical
 * ciphertext of ct and both batching rows; a violation sets bit 0 of the sticky
 * flags.  Every decryption (fhe_decrypt, fhe_check_zero_tail) max-reduces the
 * distance of t x / Q to the nearest integer over all coefficients (the invariant
 * noise, top 32 bits of the fraction, units of 2^-32): a value near 2^31 means
 * the noise budget is exhausted and the decrypted slots are garbage.
 * fhe_status synchronizes the context's stream and reads (and with reset != 0
 * clears) both. */
int fhe_check_zero_tail(fhe_ctx *ctx, const fhe_ct *ct, uint32_t m);
int fhe_status(fhe_ctx *ctx, uint32_t *noise_dist, uint32_t *flags, int reset);
/* diagnostic: coefficient-form x = c0 + c1*s over Q_level, [T*R][level][n]
 * (the caller derives the exact invariant noise |[t x]_Q| / Q from it) */
int fhe_decrypt_raw(fhe_ctx *ctx, const fhe_ct *ct, uint64_t *coef);

/* test access to the stages of one key-switched rotation (parity after every kernel, not
 * only after every primitive).  For each physical ciphertext of a (at most 128):
 *   digits [count][l][n]        INTT_i(tau_g(c1)_i), the coefficient-form digits (rotation step 1)
 *   ext    [count][l][l+1][n]   NTT_i(centered lift of digit j), canonical; column l is the
 *                               special prime; the diagonal i == j (read from the input, never
 *                               materialized) is zero
 *   acc    [count][2][l+1][n]   sum_j ext_j,i * ksk_j,i per output polynomial, WITHOUT the
 *                               rotation's c0 addend; the special prime's row (index l) in
 *                               coefficient form, as ModDown consumes it
 * Host pointers; the golden model and the CUDA library fill them from their own pipelines. */
int fhe_debug_rotate_stages(fhe_ctx *ctx, const fhe_ct *a, uint32_t k, uint64_t *digits, uint64_t *ext, uint64_t *acc);

/* ---- evaluation (out may alias an input unless stated) --------------------- */
int fhe_add(fhe_ctx *ctx, const fhe_ct *a, const fhe_ct *b, fhe_ct *out);
int fhe_mul_plain(fhe_ctx *ctx, const fhe_ct *a, const fhe_pt *pt, fhe_ct *out);
/* fused HMA: acc += a * pt in place (= fhe_add(acc, fhe_mul_plain(a, pt)); acc must not alias a) */
int fhe_mul_plain_acc(fhe_ctx *ctx, const fhe_ct *a, const fhe_pt *pt, fhe_ct *acc);
int fhe_mul_scalar(fhe_ctx *ctx, const fhe_ct *a, int64_t w, fhe_ct *out);
int fhe_add_plain(fhe_ctx *ctx, const fhe_ct *a, const fhe_pt *pt, fhe_ct *out);
/* left rotation of both rows by k in [1, N): Galois element 5^k mod 2n, then
 * hybrid key switching; out must not alias a */
int fhe_rotate(fhe_ctx *ctx, const fhe_ct *a, uint32_t k, fhe_ct *out);
/* drop the last prime with rounding; out must have level = a.level - 1 */
int fhe_mod_switch(fhe_ctx *ctx, const fhe_ct *a, fhe_ct *out);
/* slot-wise square with relinearization; out must not alias a */
int fhe_square(fhe_ctx *ctx, const fhe_ct *a, fhe_ct *out);

/* hoisted dot products: out[s] = sum_k R[k] * tau_{g[k]}(pt[s]) for s < S, where
 * tau_g is the plaintext automorphism X -> X^g (a slot rotation, applied in the
 * NTT domain) and every R[k] has the shape of out[s].  With R[k] = rotate(x, k_i)
 * and g[k] = 5^k_i this equals sum_k rotate(x * pt[s], k_i) slot for slot: the top
 * levels of S rotate-and-sum trees over one input, as a modular GEMM. */
int fhe_hoisted_dot(fhe_ctx *ctx, fhe_ct *const *R, const uint32_t *g, uint32_t K, fhe_pt *const *pt,
                    uint32_t S, fhe_ct *const *out);
/* batched forms: m independent operations in one launch sequence */
int fhe_rotate_many(fhe_ctx *ctx, fhe_ct *const *a, fhe_ct *const *out, uint32_t m, uint32_t k);
/* out[i] = a[i] + rotate(a[i], k): one rotate-and-sum level, the addition fused
 * into the key-switching epilogue */
int fhe_rotate_add_many(fhe_ctx *ctx, fhe_ct *const *a, fhe_ct *const *out, uint32_t m, uint32_t k);
/* m rotations with their own steps k[i] in [1, N) (e.g. a combine chain) */
int fhe_rotate_multi(fhe_ctx *ctx, fhe_ct *const *a, fhe_ct *const *out, const uint32_t *k, uint32_t m);
/* out[j] = rotate(a, k[j]) for j < m, sharing one digit decomposition + ModUp of a
 * (hoisted rotations; SURVEY a14 "shared ModUp per source ct"); words equal m
 * separate fhe_rotate calls.  Replaces the per-destination rotations of one masked
 * source in the reference's H-Im2Col moves (packing.py:249-279). */
int fhe_rotate_hoisted(fhe_ctx *ctx, const fhe_ct *a, const uint32_t *k, uint32_t m, fhe_ct *const *out);
int fhe_mul_plain_many(fhe_ctx *ctx, fhe_ct *const *a, fhe_pt *const *pt, fhe_ct *const *out, uint32_t m);
int fhe_add_many(fhe_ctx *ctx, fhe_ct *const *a, fhe_ct *const *b, fhe_ct *const *out, uint32_t m);

/* ---- composite operators (one call per reference operator) ------------
 * rotate_and_sum (hesim.py:347-366) of m same-level objects: slot 0 of out[i] <- sum of
 * the first span slots of a[i]; ceil(log2 span) levels acc += rotate(acc, 2^h),
 * h = rounds-1 .. 0, each level ONE fused rotate-and-add launch sequence over all m
 * objects.  Words equal the fhe_rotate / fhe_add sequence.  out[i] must not alias a[i]. */
int fhe_rotate_and_sum(fhe_ctx *ctx, fhe_ct *const *a, fhe_ct *const *out, uint32_t m, uint32_t span);
/* combine_to_dense (packing.py:350-368) as a pairwise tree: m slot-0-anchored payloads of
 * lengths[i] slots are concatenated in order; every level merges adjacent blocks
 * (left, right) into left + rotate(right, N - len(left)) with the addition fused into
 * the key-switching epilogue, an odd last block moves up unchanged.  m - 1 rotations
 * and additions (the reference's counts), one Galois key per distinct left length.
 * sum(lengths) <= N; out must not alias an input. */
int fhe_combine(fhe_ctx *ctx, fhe_ct *const *cts, const uint32_t *lengths, uint32_t m, fhe_ct *out);
/* ct-GEMM, the ConvPack channel sums (engine.py:178-197): out[o] = sum_k w[k*O + o] * a[k]
 * for o < O over K same-shape inputs, integer weights reduced per prime; every input
 * word is read once per tile of 8 outputs.  Words equal the fhe_mul_scalar / fhe_add
 * sequence.  out must not alias an input. */
int fhe_ct_gemm(fhe_ctx *ctx, fhe_ct *const *a, uint32_t K, const int64_t *w, uint32_t O, fhe_ct *const *out);

#ifdef __cplusplus
}
#endif
#endif /* FFCONV_HE_H */
