/*
 * golden_rlwe.c -- TEST INFRASTRUCTURE ONLY (oracle).  Never linked into, or
 * called by, the product path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker.
 *
 * A plain-C, single-threaded, obviously-correct model of the packed RNS-BFV
 * scheme that the CUDA library implements.  It exports the same C ABI
 * (include/ffconv_he.h) so a parity test can drive both with identical inputs
 * and compare ciphertext words bit for bit after every operation.
 *
 * What pins it:
 *   - slot level: decrypt(op(encrypt(x))) must equal the reference slot engine
 *     (cipherpack.hesim.HeContext, /root/reference/pkg/src/cipherpack/hesim.py:186-366)
 *     on the reference's own known-answer vectors (test_hesim.py) and on fixtures
 *     generated from the reference (tests/golden/make_fixtures.py);
 *   - coefficient level: the reference has no ciphertexts, so the
 *     conventions below ARE the golden spec: NTT
 *     ordering, minimal primitive roots, ChaCha20-derived samplers, secret-key
 *     encryption with round(Q m / t) scaling, single-prime-digit hybrid key
 *     switching with one special prime, HPS-style fixed-point scale-and-round.
 *
 * All arithmetic is exact (unsigned __int128); nothing here is tuned for speed.
 */
#include "ffconv_he.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef uint64_t u64;
typedef uint32_t u32;
typedef int64_t i64;

static __thread char g_err[512];

static int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char *fhe_last_error(void) { return g_err; }
const char *fhe_backend_name(void) { return "golden-c"; }

/* ------------------------------------------------------------------ */
/* modular arithmetic                                                  */
/* ------------------------------------------------------------------ */

static inline u64 mulmod(u64 a, u64 b, u64 m) { return (u64)((u128)a * b % m); }
static inline u64 addmod(u64 a, u64 b, u64 m) { u64 s = a + b; return s >= m ? s - m : s; }
static inline u64 submod(u64 a, u64 b, u64 m) { return a >= b ? a - b : a + m - b; }
static inline u64 negmod(u64 a, u64 m) { return a ? m - a : 0; }
static inline u64 smod(i64 v, u64 m) {          /* signed -> [0, m) */
    if (v >= 0) return (u64)v % m;
    u64 r = (u64)(-(v + 1)) % m;                 /* avoids overflow at INT64_MIN */
    return m - 1 - r;
}

static u64 powmod(u64 a, u64 e, u64 m) {
    u64 r = 1 % m;
    a %= m;
    while (e) {
        if (e & 1) r = mulmod(r, a, m);
        a = mulmod(a, a, m);
        e >>= 1;
    }
    return r;
}
static u64 invmod(u64 a, u64 m) { return powmod(a, m - 2, m); } /* m prime */

static int is_prime(u64 n) {
    static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) {
        if (n == bases[i]) return 1;
        if (n % bases[i] == 0) return 0;
    }
    u64 d = n - 1;
    int s = 0;
    while (!(d & 1)) { d >>= 1; s++; }
    for (int i = 0; i < 12; i++) {
        u64 x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int r = 1; r < s; r++) {
            x = mulmod(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

static inline u32 brev(u32 x, u32 bits) {
    u32 r = 0;
    for (u32 i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* floor(r * 2^128 / m) for r < m: the 128-bit fraction r/m */
static u128 frac128(u64 r, u64 m) {
    u128 num = (u128)r << 64;
    u64 hi = (u64)(num / m);
    u64 rem = (u64)(num % m);
    u64 lo = (u64)(((u128)rem << 64) / m);
    return ((u128)hi << 64) | lo;
}

/* accumulate y * (W + F/2^128) into (acc_int, acc_frac) exactly */
static inline void fx_acc(u128 *acc_int, u128 *acc_frac, u64 y, u64 W, u128 F) {
    u128 p_lo = (u128)y * (u64)F;
    u128 p_hi = (u128)y * (u64)(F >> 64);
    u128 low = p_lo + (p_hi << 64);
    u128 carry1 = low < p_lo;
    u128 ip = (p_hi >> 64) + carry1;
    *acc_frac += low;
    u128 carry2 = *acc_frac < low;
    *acc_int += (u128)y * W + ip + carry2;
}

/* ------------------------------------------------------------------ */
/* ChaCha20 counter-mode sampler                                       */
/* ------------------------------------------------------------------ */

enum { DOM_SK = 1, DOM_ENC_A = 2, DOM_ENC_E = 3, DOM_KSK_A = 4, DOM_KSK_E = 5 };

#define ROTL32(a, b) (((a) << (b)) | ((a) >> (32 - (b))))
#define QR(a, b, c, d)                                   \
    a += b; d ^= a; d = ROTL32(d, 16);                   \
    c += d; b ^= c; b = ROTL32(b, 12);                   \
    a += b; d ^= a; d = ROTL32(d, 8);                    \
    c += d; b ^= c; b = ROTL32(b, 7);

static void chacha_block(u32 out[16], u64 seed, u32 ctr, u32 dom, u32 sub, u32 x, u32 y) {
    u32 in[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                  (u32)seed, (u32)(seed >> 32), 0x243F6A88u, 0x85A308D3u,
                  0x13198A2Eu, 0x03707344u, 0xA4093822u, 0x299F31D0u,
                  ctr, (dom << 24) | (sub & 0xFFFFFFu), x, y};
    u32 s[16];
    memcpy(s, in, sizeof s);
    for (int i = 0; i < 10; i++) {
        QR(s[0], s[4], s[8], s[12]);
        QR(s[1], s[5], s[9], s[13]);
        QR(s[2], s[6], s[10], s[14]);
        QR(s[3], s[7], s[11], s[15]);
        QR(s[0], s[5], s[10], s[15]);
        QR(s[1], s[6], s[11], s[12]);
        QR(s[2], s[7], s[8], s[13]);
        QR(s[3], s[4], s[9], s[14]);
    }
    for (int i = 0; i < 16; i++) out[i] = s[i] + in[i];
}

/* uniform residues mod m: coefficient c uses words 4(c%4)..+3 of block c/4 */
static void sample_uniform(u64 *dst, u32 n, u64 m, u64 seed, u32 dom, u32 sub, u32 x, u32 y) {
    u32 blk[16];
    for (u32 c = 0; c < n; c++) {
        if ((c & 3) == 0) chacha_block(blk, seed, c >> 2, dom, sub, x, y);
        const u32 *w = blk + 4 * (c & 3);
        u128 v = ((u128)w[3] << 96) | ((u128)w[2] << 64) | ((u128)w[1] << 32) | w[0];
        dst[c] = (u64)(v % m);
    }
}

/* ternary {-1,0,1}: word c%16 of block c/16, value mod 3 -> {0, 1, -1} */
static void sample_ternary(int8_t *dst, u32 n, u64 seed, u32 dom, u32 sub, u32 x, u32 y) {
    u32 blk[16];
    for (u32 c = 0; c < n; c++) {
        if ((c & 15) == 0) chacha_block(blk, seed, c >> 4, dom, sub, x, y);
        u32 r = blk[c & 15] % 3u;
        dst[c] = r == 2 ? -1 : (int8_t)r;
    }
}

/* centered binomial, eta = 21 (sigma ~ 3.24): words 2(c%8), 2(c%8)+1 of block c/8 */
static void sample_cbd(i64 *dst, u32 n, u64 seed, u32 dom, u32 sub, u32 x, u32 y) {
    u32 blk[16];
    for (u32 c = 0; c < n; c++) {
        if ((c & 7) == 0) chacha_block(blk, seed, c >> 3, dom, sub, x, y);
        u32 w0 = blk[2 * (c & 7)] & 0x1FFFFFu, w1 = blk[2 * (c & 7) + 1] & 0x1FFFFFu;
        dst[c] = (i64)__builtin_popcount(w0) - (i64)__builtin_popcount(w1);
    }
}

/* ------------------------------------------------------------------ */
/* NTT                                                                 */
/* ------------------------------------------------------------------ */

typedef struct {
    u64 q;
    u64 psi;      /* minimal primitive 2n-th root of unity */
    u64 n_inv;
    u64 *psi_rev;     /* psi^brev(k)   */
    u64 *psi_inv_rev; /* psi^-brev(k)  */
} modtab;

static u64 min_primitive_root(u64 q, u32 n) {
    u64 two_n = 2ull * n, psi0 = 0;
    for (u64 h = 2; h < q; h++) {
        u64 c = powmod(h, (q - 1) / two_n, q);
        if (powmod(c, n, q) == q - 1) { psi0 = c; break; }
    }
    u64 sq = mulmod(psi0, psi0, q), cur = psi0, best = psi0;
    for (u32 k = 0; k < n; k++) {
        if (cur < best) best = cur;
        cur = mulmod(cur, sq, q);
    }
    return best;
}

static int modtab_init(modtab *M, u64 q, u32 n, u32 logn) {
    M->q = q;
    M->psi = min_primitive_root(q, n);
    M->n_inv = invmod(n, q);
    M->psi_rev = (u64 *)malloc(n * sizeof(u64));
    M->psi_inv_rev = (u64 *)malloc(n * sizeof(u64));
    if (!M->psi_rev || !M->psi_inv_rev) return -1;
    u64 psi_inv = invmod(M->psi, q);
    u64 *pw = (u64 *)malloc(n * sizeof(u64)), *pwi = (u64 *)malloc(n * sizeof(u64));
    pw[0] = 1; pwi[0] = 1;
    for (u32 k = 1; k < n; k++) { pw[k] = mulmod(pw[k - 1], M->psi, q); pwi[k] = mulmod(pwi[k - 1], psi_inv, q); }
    for (u32 k = 0; k < n; k++) { M->psi_rev[k] = pw[brev(k, logn)]; M->psi_inv_rev[k] = pwi[brev(k, logn)]; }
    free(pw); free(pwi);
    return 0;
}

static void modtab_free(modtab *M) { free(M->psi_rev); free(M->psi_inv_rev); }

/* natural-order coefficients -> evaluations, a[i] = A(psi^(2 brev(i) + 1)) */
static void ntt(u64 *a, const modtab *M, u32 n) {
    u64 q = M->q;
    u32 t = n;
    for (u32 m = 1; m < n; m <<= 1) {
        t >>= 1;
        for (u32 i = 0; i < m; i++) {
            u32 j1 = 2 * i * t;
            u64 S = M->psi_rev[m + i];
            for (u32 j = j1; j < j1 + t; j++) {
                u64 U = a[j], V = mulmod(a[j + t], S, q);
                a[j] = addmod(U, V, q);
                a[j + t] = submod(U, V, q);
            }
        }
    }
}

static void intt(u64 *a, const modtab *M, u32 n) {
    u64 q = M->q;
    u32 t = 1;
    for (u32 m = n; m > 1; m >>= 1) {
        u32 j1 = 0, h = m >> 1;
        for (u32 i = 0; i < h; i++) {
            u64 S = M->psi_inv_rev[h + i];
            for (u32 j = j1; j < j1 + t; j++) {
                u64 U = a[j], V = a[j + t];
                a[j] = addmod(U, V, q);
                a[j + t] = mulmod(submod(U, V, q), S, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    for (u32 j = 0; j < n; j++) a[j] = mulmod(a[j], M->n_inv, q);
}

/* ------------------------------------------------------------------ */
/* context                                                             */
/* ------------------------------------------------------------------ */

typedef struct key_node {
    u32 kid;            /* Galois element, or 0 for the relinearization key */
    u64 *data;          /* [L digits][2: b, a][L+1 primes][n], NTT domain     */
    struct key_node *next;
} key_node;

typedef struct {
    /* decryption / encoding, per plaintext modulus k */
    u64 Qtilde[FHE_MAX_Q];              /* (Q_l/q_i)^-1 mod q_i           */
    u64 decW[FHE_MAX_T][FHE_MAX_Q];     /* floor(t_k / q_i)              */
    u128 decF[FHE_MAX_T][FHE_MAX_Q];    /* frac(t_k / q_i) * 2^128        */
    u64 delta[FHE_MAX_T][FHE_MAX_Q];    /* floor(Q_l / t_k) mod q_i       */
    u64 rt[FHE_MAX_T];                  /* Q_l mod t_k                    */
    u64 msinv[FHE_MAX_Q];               /* q_{l-1}^-1 mod q_i (mod switch) */
    /* squaring: lift Q_l -> B */
    u128 invq[FHE_MAX_Q];               /* 2^128 / q_i                    */
    u64 QhatB[FHE_MAX_Q][FHE_MAX_B];    /* (Q_l/q_i) mod b_k              */
    u64 QmodB[FHE_MAX_B];
    /* squaring: scale t/Q_l in Q_l u B, result in B */
    u64 Mtq[FHE_MAX_Q];                 /* ((Q_l/q_i) B)^-1 mod q_i       */
    u64 Mtb[FHE_MAX_B];                 /* ((B/b_k) Q_l)^-1 mod b_k       */
    u64 omega[FHE_MAX_T][FHE_MAX_Q][FHE_MAX_B]; /* floor(t B / q_i) mod b_k */
    u128 theta[FHE_MAX_T][FHE_MAX_Q];   /* frac(t B / q_i) * 2^128        */
    u64 tBb[FHE_MAX_T][FHE_MAX_B];      /* t (B/b_k) mod b_k              */
} level_tab;

typedef struct {
    /* B -> Q (independent of level except through the target primes) */
    u64 Btilde[FHE_MAX_B];              /* (B/b_k)^-1 mod b_k */
    u128 invb[FHE_MAX_B];
    u64 BhatQ[FHE_MAX_B][FHE_MAX_Q];    /* (B/b_k) mod q_i    */
    u64 BmodQ[FHE_MAX_Q];
} aux_tab;

struct fhe_ctx {
    fhe_params P;
    u32 n, logn, N, L, nb, T;
    u32 nmod;          /* L + 1 + nb + T */
    modtab *M;         /* index: q_i -> i, special -> L, b_k -> L+1+k, t_k -> L+1+nb+k */
    int8_t *s;
    u64 **s_ntt;       /* per q, special, aux */
    u64 **s2_ntt;      /* per q, special */
    u32 *slot2ntt;
    u64 pmod[FHE_MAX_Q], pinv[FHE_MAX_Q];
    level_tab *lv;     /* lv[l] for l in 1..L */
    aux_tab ax;
    key_node *keys;
    u64 key_bytes;
    uint32_t noise_max;  /* largest decryption rounding distance since the last fhe_status (2^-32 units) */
    uint32_t flags;      /* bit 0: rotate_and_sum precondition violated (fhe_check_zero_tail) */
};

struct fhe_ct {
    fhe_ctx *ctx;
    u32 R, level, count;
    u64 *data;         /* [count][2][level][n] */
};

struct fhe_pt {
    fhe_ctx *ctx;
    int encoded;
    u64 *coef_t;       /* [T][n] coefficients mod t_k            */
    u64 *ntt_q;        /* [T][L][n] centered lift, NTT mod q_i     */
};

#define IDX_P(ctx) ((ctx)->L)
#define IDX_B(ctx, k) ((ctx)->L + 1 + (k))
#define IDX_T(ctx, k) ((ctx)->L + 1 + (ctx)->nb + (k))

static u64 modof(const fhe_ctx *c, u32 idx) { return c->M[idx].q; }

static void build_level(fhe_ctx *c, u32 l) {
    level_tab *T = &c->lv[l];
    const u64 *q = c->P.q;
    for (u32 i = 0; i < l; i++) {
        u64 qh = 1;
        for (u32 j = 0; j < l; j++) if (j != i) qh = mulmod(qh, q[j] % q[i], q[i]);
        T->Qtilde[i] = invmod(qh, q[i]);
        T->invq[i] = frac128(1, q[i]);
        if (l >= 2 && i < l - 1) T->msinv[i] = invmod(q[l - 1] % q[i], q[i]);
    }
    for (u32 k = 0; k < c->T; k++) {
        u64 t = c->P.t[k];
        u64 rt = 1;
        for (u32 j = 0; j < l; j++) rt = mulmod(rt, q[j] % t, t);
        T->rt[k] = rt;
        for (u32 i = 0; i < l; i++) {
            T->decW[k][i] = t / q[i];
            T->decF[k][i] = frac128(t % q[i], q[i]);
            /* floor(Q/t) = (Q - rt)/t ; mod q_i: (-rt) * t^-1 */
            T->delta[k][i] = mulmod(negmod(rt % q[i], q[i]), invmod(t % q[i], q[i]), q[i]);
        }
    }
    if (!c->nb) return;
    const u64 *b = c->P.b;
    u32 nb = c->nb;
    for (u32 k = 0; k < nb; k++) {
        u64 Qm = 1;
        for (u32 j = 0; j < l; j++) Qm = mulmod(Qm, q[j] % b[k], b[k]);
        T->QmodB[k] = Qm;
        for (u32 i = 0; i < l; i++) {
            u64 qh = 1;
            for (u32 j = 0; j < l; j++) if (j != i) qh = mulmod(qh, q[j] % b[k], b[k]);
            T->QhatB[i][k] = qh;
        }
        u64 bh = 1;
        for (u32 j = 0; j < nb; j++) if (j != k) bh = mulmod(bh, b[j] % b[k], b[k]);
        T->Mtb[k] = invmod(mulmod(bh, Qm, b[k]), b[k]);
    }
    for (u32 i = 0; i < l; i++) {
        u64 Bm = 1;
        for (u32 k = 0; k < nb; k++) Bm = mulmod(Bm, b[k] % q[i], q[i]);
        u64 qh = 1;
        for (u32 j = 0; j < l; j++) if (j != i) qh = mulmod(qh, q[j] % q[i], q[i]);
        T->Mtq[i] = invmod(mulmod(qh, Bm, q[i]), q[i]);
        for (u32 kt = 0; kt < c->T; kt++) {
            u64 t = c->P.t[kt];
            u64 tBq = mulmod(t % q[i], Bm, q[i]);            /* (t B) mod q_i */
            T->theta[kt][i] = frac128(tBq, q[i]);
            for (u32 k = 0; k < nb; k++)                        /* floor(tB/q_i) mod b_k */
                T->omega[kt][i][k] = mulmod(negmod(tBq % b[k], b[k]), invmod(q[i] % b[k], b[k]), b[k]);
        }
    }
    for (u32 kt = 0; kt < c->T; kt++) {
        u64 t = c->P.t[kt];
        for (u32 k = 0; k < nb; k++) {
            u64 bh = 1;
            for (u32 j = 0; j < nb; j++) if (j != k) bh = mulmod(bh, b[j] % b[k], b[k]);
            T->tBb[kt][k] = mulmod(t % b[k], bh, b[k]);
        }
    }
}

static void build_aux(fhe_ctx *c) {
    aux_tab *A = &c->ax;
    const u64 *b = c->P.b, *q = c->P.q;
    for (u32 k = 0; k < c->nb; k++) {
        u64 bh = 1;
        for (u32 j = 0; j < c->nb; j++) if (j != k) bh = mulmod(bh, b[j] % b[k], b[k]);
        A->Btilde[k] = invmod(bh, b[k]);
        A->invb[k] = frac128(1, b[k]);
        for (u32 i = 0; i < c->L; i++) {
            u64 h = 1;
            for (u32 j = 0; j < c->nb; j++) if (j != k) h = mulmod(h, b[j] % q[i], q[i]);
            A->BhatQ[k][i] = h;
        }
    }
    for (u32 i = 0; i < c->L; i++) {
        u64 Bm = 1;
        for (u32 k = 0; k < c->nb; k++) Bm = mulmod(Bm, b[k] % q[i], q[i]);
        A->BmodQ[i] = Bm;
    }
}

static int validate(const fhe_params *p) {
    if (p->log_n < 2 || p->log_n > 16) return fail(FHE_EINVAL, "log_n must be in [2, 16], got %u", p->log_n);
    if (p->L < 1 || p->L > FHE_MAX_Q) return fail(FHE_EINVAL, "L must be in [1, %d]", FHE_MAX_Q);
    if (p->K != 1) return fail(FHE_EINVAL, "exactly one special prime is supported (K=%u)", p->K);
    if (p->n_aux > FHE_MAX_B) return fail(FHE_EINVAL, "n_aux must be <= %d", FHE_MAX_B);
    if (p->n_aux && p->n_aux < p->L + 1) return fail(FHE_EINVAL, "n_aux must be 0 or >= L+1");
    if (p->T < 1 || p->T > FHE_MAX_T) return fail(FHE_EINVAL, "T must be in [1, %d]", FHE_MAX_T);
    u64 two_n = 2ull << p->log_n;
    u64 all[FHE_MAX_Q + FHE_MAX_P + FHE_MAX_B + FHE_MAX_T];
    u32 na = 0;
    for (u32 i = 0; i < p->L; i++) all[na++] = p->q[i];
    all[na++] = p->p[0];
    for (u32 i = 0; i < p->n_aux; i++) all[na++] = p->b[i];
    for (u32 i = 0; i < p->T; i++) all[na++] = p->t[i];
    for (u32 i = 0; i < na; i++) {
        if (all[i] >= (1ull << 61) || all[i] < 3) return fail(FHE_EINVAL, "modulus %llu outside [3, 2^61)", (unsigned long long)all[i]);
        if (!is_prime(all[i])) return fail(FHE_EINVAL, "modulus %llu is not prime", (unsigned long long)all[i]);
        if (all[i] % two_n != 1) return fail(FHE_EINVAL, "modulus %llu is not 1 mod 2n = %llu", (unsigned long long)all[i], (unsigned long long)two_n);
        for (u32 j = 0; j < i; j++)
            if (all[j] == all[i]) return fail(FHE_EINVAL, "modulus %llu repeated", (unsigned long long)all[i]);
    }
    for (u32 i = 0; i < p->L; i++)
        if (p->p[0] < p->q[i]) return fail(FHE_EINVAL, "special prime must exceed every q_i");
    return 0;
}

int fhe_ctx_create(const fhe_params *params, fhe_ctx **out) {
    int rc = validate(params);
    if (rc) return rc;
    fhe_ctx *c = (fhe_ctx *)calloc(1, sizeof(fhe_ctx));
    if (!c) return fail(FHE_ENOMEM, "out of memory");
    c->P = *params;
    c->logn = params->log_n;
    c->n = 1u << c->logn;
    c->N = c->n / 2;
    c->L = params->L;
    c->nb = params->n_aux;
    c->T = params->T;
    c->nmod = c->L + 1 + c->nb + c->T;
    c->M = (modtab *)calloc(c->nmod, sizeof(modtab));
    for (u32 i = 0; i < c->L; i++) modtab_init(&c->M[i], params->q[i], c->n, c->logn);
    modtab_init(&c->M[IDX_P(c)], params->p[0], c->n, c->logn);
    for (u32 k = 0; k < c->nb; k++) modtab_init(&c->M[IDX_B(c, k)], params->b[k], c->n, c->logn);
    for (u32 k = 0; k < c->T; k++) modtab_init(&c->M[IDX_T(c, k)], params->t[k], c->n, c->logn);

    u32 n = c->n;
    c->s = (int8_t *)malloc(n);
    sample_ternary(c->s, n, params->seed, DOM_SK, 0, 0, 0);
    u32 nks = c->L + 1 + c->nb;
    c->s_ntt = (u64 **)calloc(nks, sizeof(u64 *));
    c->s2_ntt = (u64 **)calloc(c->L + 1, sizeof(u64 *));
    for (u32 i = 0; i < nks; i++) {
        u64 q = modof(c, i);
        c->s_ntt[i] = (u64 *)malloc(n * sizeof(u64));
        for (u32 j = 0; j < n; j++) c->s_ntt[i][j] = smod(c->s[j], q);
        ntt(c->s_ntt[i], &c->M[i], n);
        if (i <= c->L) {
            c->s2_ntt[i] = (u64 *)malloc(n * sizeof(u64));
            for (u32 j = 0; j < n; j++) c->s2_ntt[i][j] = mulmod(c->s_ntt[i][j], c->s_ntt[i][j], q);
        }
    }
    c->slot2ntt = (u32 *)malloc(n * sizeof(u32));
    u64 two_n = 2ull * n, e = 1;
    for (u32 i = 0; i < c->N; i++) {
        c->slot2ntt[i] = brev((u32)((e - 1) / 2), c->logn);
        c->slot2ntt[c->N + i] = brev((u32)((two_n - e - 1) / 2), c->logn);
        e = e * 5 % two_n;
    }
    u64 P = params->p[0];
    for (u32 i = 0; i < c->L; i++) {
        c->pmod[i] = P % params->q[i];
        c->pinv[i] = invmod(c->pmod[i], params->q[i]);
    }
    c->lv = (level_tab *)calloc(c->L + 1, sizeof(level_tab));
    for (u32 l = 1; l <= c->L; l++) build_level(c, l);
    if (c->nb) build_aux(c);
    *out = c;
    return 0;
}

void fhe_ctx_destroy(fhe_ctx *c) {
    if (!c) return;
    for (u32 i = 0; i < c->nmod; i++) modtab_free(&c->M[i]);
    free(c->M);
    for (u32 i = 0; i < c->L + 1 + c->nb; i++) free(c->s_ntt[i]);
    for (u32 i = 0; i <= c->L; i++) free(c->s2_ntt[i]);
    free(c->s_ntt); free(c->s2_ntt); free(c->s); free(c->slot2ntt); free(c->lv);
    key_node *k = c->keys;
    while (k) { key_node *nx = k->next; free(k->data); free(k); k = nx; }
    free(c);
}

int fhe_sync(fhe_ctx *ctx) { (void)ctx; return 0; }
int fhe_ctx_stream(fhe_ctx *ctx, void **stream) { (void)ctx; *stream = NULL; return 0; }
int fhe_prof_enable(fhe_ctx *ctx, int on) { (void)ctx; (void)on; return 0; }
int fhe_prof_report(fhe_ctx *ctx, char *buf, uint32_t len) { (void)ctx; if (len) buf[0] = 0; return 0; }
int fhe_launch_count(fhe_ctx *ctx, uint64_t *out) { (void)ctx; *out = 0; return 0; }
int fhe_work_modmuls(fhe_ctx *ctx, double *out) { (void)ctx; *out = 0.0; return 0; }
int fhe_peak_modmul(fhe_ctx *ctx, uint32_t iters, double *out) {
    (void)ctx; (void)iters; *out = 0.0;
    return fail(FHE_EINVAL, "no device in the golden model");
}
int fhe_peak_modmul_kind(fhe_ctx *ctx, uint32_t iters, int kind, double *out) {
    (void)kind;
    return fhe_peak_modmul(ctx, iters, out);
}
int fhe_ctx_key_bytes(fhe_ctx *ctx, uint64_t *out) { *out = ctx->key_bytes; return 0; }

/* ------------------------------------------------------------------ */
/* keys                                                                */
/* ------------------------------------------------------------------ */

static u32 galois_elt(const fhe_ctx *c, u32 k) { return (u32)powmod(5, k, 2ull * c->n); }

/* out[j] = in[perm_g(j)]: NTT-domain automorphism X -> X^g */
static void automorph(const fhe_ctx *c, const u64 *in, u64 *out, u32 g) {
    u32 n = c->n, logn = c->logn;
    u64 mask = 2ull * n - 1;
    for (u32 j = 0; j < n; j++) {
        u64 e = 2ull * brev(j, logn) + 1;
        u64 eg = (e * g) & mask;
        out[j] = in[brev((u32)((eg - 1) / 2), logn)];
    }
}

static key_node *get_key(fhe_ctx *c, u32 kid) {
    for (key_node *k = c->keys; k; k = k->next) if (k->kid == kid) return k;
    u32 n = c->n, L = c->L;
    key_node *k = (key_node *)calloc(1, sizeof(key_node));
    k->kid = kid;
    size_t words = (size_t)L * 2 * (L + 1) * n;
    k->data = (u64 *)malloc(words * sizeof(u64));
    u64 *target = (u64 *)malloc(n * sizeof(u64));
    i64 *e = (i64 *)malloc(n * sizeof(i64));
    u64 *tmp = (u64 *)malloc(n * sizeof(u64));
    for (u32 j = 0; j < L; j++) {
        sample_cbd(e, n, c->P.seed, DOM_KSK_E, j, kid, 0);
        for (u32 i = 0; i <= L; i++) {
            u64 q = modof(c, i);
            u64 *bk = k->data + (((size_t)j * 2 + 0) * (L + 1) + i) * n;
            u64 *ak = k->data + (((size_t)j * 2 + 1) * (L + 1) + i) * n;
            sample_uniform(ak, n, q, c->P.seed, DOM_KSK_A, j * 64 + i, kid, 0);
            for (u32 x = 0; x < n; x++) tmp[x] = smod(e[x], q);
            ntt(tmp, &c->M[i], n);
            for (u32 x = 0; x < n; x++) bk[x] = submod(tmp[x], mulmod(ak[x], c->s_ntt[i][x], q), q);
            if (i == j) {
                if (kid == 0) memcpy(target, c->s2_ntt[i], n * sizeof(u64));
                else automorph(c, c->s_ntt[i], target, kid);
                for (u32 x = 0; x < n; x++) bk[x] = addmod(bk[x], mulmod(c->pmod[i], target[x], q), q);
            }
        }
    }
    free(target); free(e); free(tmp);
    k->next = c->keys;
    c->keys = k;
    c->key_bytes += words * sizeof(u64);
    return k;
}

int fhe_keygen_rotations(fhe_ctx *c, const uint32_t *steps, uint32_t m) {
    for (u32 i = 0; i < m; i++) {
        if (steps[i] == 0 || steps[i] >= c->N) return fail(FHE_EINVAL, "rotation step %u outside [1, %u)", steps[i], c->N);
        get_key(c, galois_elt(c, steps[i]));
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* objects                                                             */
/* ------------------------------------------------------------------ */

int fhe_ct_create(fhe_ctx *c, uint32_t R, uint32_t level, fhe_ct **out) {
    if (R < 1) return fail(FHE_EINVAL, "R must be >= 1");
    if (level < 1 || level > c->L) return fail(FHE_ELEVEL, "level %u outside [1, %u]", level, c->L);
    fhe_ct *ct = (fhe_ct *)calloc(1, sizeof(fhe_ct));
    ct->ctx = c; ct->R = R; ct->level = level; ct->count = R * c->T;
    ct->data = (u64 *)calloc((size_t)ct->count * 2 * level * c->n, sizeof(u64));
    if (!ct->data) { free(ct); return fail(FHE_ENOMEM, "out of memory"); }
    *out = ct;
    return 0;
}
void fhe_ct_destroy(fhe_ct *ct) { if (ct) { free(ct->data); free(ct); } }
uint32_t fhe_ct_level(const fhe_ct *ct) { return ct->level; }
uint32_t fhe_ct_rows(const fhe_ct *ct) { return ct->R; }

static size_t ct_words(const fhe_ct *ct) { return (size_t)ct->count * 2 * ct->level * ct->ctx->n; }
static u64 *poly(const fhe_ct *ct, u32 idx, u32 p, u32 i) {
    return ct->data + (((size_t)idx * 2 + p) * ct->level + i) * ct->ctx->n;
}

int fhe_ct_read(fhe_ctx *c, const fhe_ct *ct, uint64_t *w) { (void)c; memcpy(w, ct->data, ct_words(ct) * 8); return 0; }
int fhe_ct_write(fhe_ctx *c, fhe_ct *ct, const uint64_t *w) { (void)c; memcpy(ct->data, w, ct_words(ct) * 8); return 0; }
int fhe_ct_to_device(fhe_ctx *c, const fhe_ct *ct, void *dst) { (void)c; memcpy(dst, ct->data, ct_words(ct) * 8); return 0; }
int fhe_ct_from_device(fhe_ctx *c, fhe_ct *ct, const void *src) { (void)c; memcpy(ct->data, src, ct_words(ct) * 8); return 0; }
int fhe_ct_zero(fhe_ctx *c, fhe_ct *ct) { (void)c; memset(ct->data, 0, ct_words(ct) * 8); return 0; }

int fhe_pt_create(fhe_ctx *c, fhe_pt **out) {
    fhe_pt *pt = (fhe_pt *)calloc(1, sizeof(fhe_pt));
    pt->ctx = c;
    pt->coef_t = (u64 *)calloc((size_t)c->T * c->n, sizeof(u64));
    pt->ntt_q = (u64 *)calloc((size_t)c->T * c->L * c->n, sizeof(u64));
    *out = pt;
    return 0;
}
void fhe_pt_destroy(fhe_pt *pt) { if (pt) { free(pt->coef_t); free(pt->ntt_q); free(pt); } }

/* slots (positions r*N+i) -> coefficients mod t_k */
static void slots_to_coef(const fhe_ctx *c, u32 k, const u64 *slots, u64 *coef) {
    u64 t = c->P.t[k];
    for (u32 x = 0; x < c->n; x++) coef[c->slot2ntt[x]] = slots[x] % t;
    intt(coef, &c->M[IDX_T(c, k)], c->n);
}

static void coef_to_slots(const fhe_ctx *c, u32 k, u64 *coef, u64 *slots) {
    ntt(coef, &c->M[IDX_T(c, k)], c->n);
    for (u32 x = 0; x < c->n; x++) slots[x] = coef[c->slot2ntt[x]];
}

int fhe_encode(fhe_ctx *c, const uint64_t *slots, fhe_pt *pt) {
    u32 n = c->n;
    for (u32 k = 0; k < c->T; k++) {
        u64 t = c->P.t[k];
        u64 *coef = pt->coef_t + (size_t)k * n;
        slots_to_coef(c, k, slots + (size_t)k * n, coef);
        for (u32 i = 0; i < c->L; i++) {
            u64 q = c->P.q[i];
            u64 *dst = pt->ntt_q + ((size_t)k * c->L + i) * n;
            for (u32 x = 0; x < n; x++) {
                i64 v = coef[x] >= (t + 1) / 2 ? (i64)coef[x] - (i64)t : (i64)coef[x];
                dst[x] = smod(v, q);
            }
            ntt(dst, &c->M[i], n);
        }
    }
    pt->encoded = 1;
    return 0;
}

int fhe_pt_read(fhe_ctx *c, const fhe_pt *pt, uint64_t *w) {
    memcpy(w, pt->ntt_q, (size_t)c->T * c->L * c->n * 8);
    return 0;
}

/* round(Q_l m / t_k) mod q_i, m in [0, t) */
static inline u64 scaled_msg(const level_tab *T, u32 k, u64 t, u64 m, u32 i, u64 q) {
    u64 corr = (u64)(((u128)2 * T->rt[k] * m + t) / ((u128)2 * t));
    return addmod(mulmod(T->delta[k][i], m % q, q), corr % q, q);
}

int fhe_encrypt(fhe_ctx *c, const uint64_t *slots, uint32_t nonce, fhe_ct *ct) {
    if (ct->level != c->L) return fail(FHE_ELEVEL, "encryption target must be at the top level");
    u32 n = c->n, L = c->L;
    const level_tab *T = &c->lv[L];
    u64 *coef = (u64 *)malloc(n * 8), *tmp = (u64 *)malloc(n * 8);
    i64 *e = (i64 *)malloc(n * sizeof(i64));
    for (u32 ci = 0; ci < ct->count; ci++) {
        u32 k = ci / ct->R;
        u64 t = c->P.t[k];
        slots_to_coef(c, k, slots + (size_t)ci * n, coef);
        sample_cbd(e, n, c->P.seed, DOM_ENC_E, 0, nonce, ci);
        for (u32 i = 0; i < L; i++) {
            u64 q = c->P.q[i];
            u64 *c0 = poly(ct, ci, 0, i), *c1 = poly(ct, ci, 1, i);
            sample_uniform(c1, n, q, c->P.seed, DOM_ENC_A, i, nonce, ci);
            for (u32 x = 0; x < n; x++) tmp[x] = addmod(smod(e[x], q), scaled_msg(T, k, t, coef[x], i, q), q);
            ntt(tmp, &c->M[i], n);
            for (u32 x = 0; x < n; x++) c0[x] = submod(tmp[x], mulmod(c1[x], c->s_ntt[i][x], q), q);
        }
    }
    free(coef); free(tmp); free(e);
    return 0;
}

/* x_i = INTT(c0 + c1 s) over Q_l, [l][n] */
static void raw_one(const fhe_ctx *c, const fhe_ct *ct, u32 ci, u64 *x) {
    u32 n = c->n, l = ct->level;
    for (u32 i = 0; i < l; i++) {
        u64 q = c->P.q[i];
        const u64 *c0 = poly(ct, ci, 0, i), *c1 = poly(ct, ci, 1, i);
        u64 *xi = x + (size_t)i * n;
        for (u32 j = 0; j < n; j++) xi[j] = addmod(c0[j], mulmod(c1[j], c->s_ntt[i][j], q), q);
        intt(xi, &c->M[i], n);
    }
}

/* m = round(t x / Q_l) mod t via the 128-bit fixed-point sum of y_i t / q_i */
static void decrypt_one(fhe_ctx *c, const fhe_ct *ct, u32 ci, u64 *coef) {
    u32 n = c->n, l = ct->level, k = ci / ct->R;
    u64 t = c->P.t[k];
    const level_tab *T = &c->lv[l];
    u64 *x = (u64 *)malloc((size_t)l * n * 8);
    raw_one(c, ct, ci, x);
    for (u32 j = 0; j < n; j++) {
        u128 ai = 0, af = 0;
        for (u32 i = 0; i < l; i++) {
            u64 y = mulmod(x[(size_t)i * n + j], T->Qtilde[i], c->P.q[i]);
            fx_acc(&ai, &af, y, T->decW[k][i], T->decF[k][i]);
        }
        coef[j] = (u64)((ai + (af >> 127)) % t);
        uint32_t f = (uint32_t)(af >> 96), d = (f >> 31) ? 0u - f : f;
        if (d > c->noise_max) c->noise_max = d;
    }
    free(x);
}

int fhe_decrypt(fhe_ctx *c, const fhe_ct *ct, uint64_t *slots) {
    u64 *coef = (u64 *)malloc(c->n * 8);
    for (u32 ci = 0; ci < ct->count; ci++) {
        decrypt_one(c, ct, ci, coef);
        coef_to_slots(c, ci / ct->R, coef, slots + (size_t)ci * c->n);
    }
    free(coef);
    return 0;
}

int fhe_decrypt_slots(fhe_ctx *c, const fhe_ct *ct, uint32_t lo, uint32_t cnt, uint64_t *out) {
    if ((u64)lo + cnt > c->N) return fail(FHE_EINVAL, "decrypt_slots: [%u, %u) exceeds %u slots", lo, lo + cnt, c->N);
    u64 *coef = (u64 *)malloc(c->n * 8), *slots = (u64 *)malloc(c->n * 8);
    for (u32 ci = 0; ci < ct->count; ci++) {
        decrypt_one(c, ct, ci, coef);
        coef_to_slots(c, ci / ct->R, coef, slots);
        for (u32 r = 0; r < 2; r++)
            for (u32 x = 0; x < cnt; x++) out[((size_t)ci * 2 + r) * cnt + x] = slots[r * c->N + lo + x];
    }
    free(coef); free(slots);
    return 0;
}

int fhe_ct_copy(fhe_ctx *c, const fhe_ct *src, fhe_ct *dst) {
    if (src->R != dst->R || src->level != dst->level) return fail(FHE_ELEVEL, "ct_copy: shape/level mismatch");
    memcpy(dst->data, src->data, (size_t)src->count * 2 * src->level * c->n * 8);
    return 0;
}

/* plan capture is a device feature: the golden model evaluates eagerly */
int fhe_capture_begin(fhe_ctx *c, uint64_t arena_bytes) { (void)c; (void)arena_bytes; return fail(FHE_EINVAL, "no device in the golden model"); }
int fhe_capture_end(fhe_ctx *c, fhe_graph **out) { (void)c; *out = NULL; return fail(FHE_EINVAL, "no device in the golden model"); }
int fhe_graph_launch(fhe_ctx *c, fhe_graph *g) { (void)c; (void)g; return fail(FHE_EINVAL, "no device in the golden model"); }
int fhe_graph_nodes(fhe_graph *g, uint64_t *out) { (void)g; *out = 0; return fail(FHE_EINVAL, "no device in the golden model"); }
void fhe_graph_destroy(fhe_graph *g) { (void)g; }
int fhe_ctx_peak_bytes(fhe_ctx *c, uint64_t *out, int reset) { (void)c; (void)reset; *out = 0; return 0; }

int fhe_check_zero_tail(fhe_ctx *c, const fhe_ct *ct, uint32_t m) {
    if (m > c->N) return fail(FHE_EINVAL, "check_zero_tail: m = %u exceeds %u slots", m, c->N);
    if (m == c->N) return 0;
    u64 *coef = (u64 *)malloc(c->n * 8), *slots = (u64 *)malloc(c->n * 8);
    for (u32 ci = 0; ci < ct->count; ci++) {
        decrypt_one(c, ct, ci, coef);
        coef_to_slots(c, ci / ct->R, coef, slots);
        for (u32 x = 0; x < c->n; x++)
            if ((x % c->N) >= m && slots[x]) c->flags |= 1u;
    }
    free(coef); free(slots);
    return 0;
}

int fhe_status(fhe_ctx *c, uint32_t *noise_dist, uint32_t *flags, int reset) {
    if (noise_dist) *noise_dist = c->noise_max;
    if (flags) *flags = c->flags;
    if (reset) { c->noise_max = 0; c->flags = 0; }
    return 0;
}

int fhe_decrypt_raw(fhe_ctx *c, const fhe_ct *ct, uint64_t *out) {
    for (u32 ci = 0; ci < ct->count; ci++) raw_one(c, ct, ci, out + (size_t)ci * ct->level * c->n);
    return 0;
}

/* ------------------------------------------------------------------ */
/* evaluation                                                          */
/* ------------------------------------------------------------------ */

static int same_shape(const fhe_ct *a, const fhe_ct *b) { return a->R == b->R && a->level == b->level; }

int fhe_add(fhe_ctx *c, const fhe_ct *a, const fhe_ct *b, fhe_ct *out) {
    if (!same_shape(a, b) || !same_shape(a, out)) return fail(FHE_ELEVEL, "add: shape/level mismatch");
    for (u32 ci = 0; ci < a->count; ci++)
        for (u32 p = 0; p < 2; p++)
            for (u32 i = 0; i < a->level; i++) {
                u64 q = c->P.q[i];
                const u64 *x = poly(a, ci, p, i), *y = poly(b, ci, p, i);
                u64 *z = poly(out, ci, p, i);
                for (u32 j = 0; j < c->n; j++) z[j] = addmod(x[j], y[j], q);
            }
    return 0;
}

int fhe_mul_plain(fhe_ctx *c, const fhe_ct *a, const fhe_pt *pt, fhe_ct *out) {
    if (!same_shape(a, out)) return fail(FHE_ELEVEL, "mul_plain: shape/level mismatch");
    for (u32 ci = 0; ci < a->count; ci++) {
        u32 k = ci / a->R;
        for (u32 p = 0; p < 2; p++)
            for (u32 i = 0; i < a->level; i++) {
                u64 q = c->P.q[i];
                const u64 *x = poly(a, ci, p, i), *w = pt->ntt_q + ((size_t)k * c->L + i) * c->n;
                u64 *z = poly(out, ci, p, i);
                for (u32 j = 0; j < c->n; j++) z[j] = mulmod(x[j], w[j], q);
            }
    }
    return 0;
}

int fhe_mul_plain_acc(fhe_ctx *c, const fhe_ct *a, const fhe_pt *pt, fhe_ct *acc) {
    if (!same_shape(a, acc)) return fail(FHE_ELEVEL, "mul_plain_acc: shape/level mismatch");
    if (a == acc) return fail(FHE_EINVAL, "mul_plain_acc: the accumulator must not alias the input");
    for (u32 ci = 0; ci < a->count; ci++) {
        u32 k = ci / a->R;
        for (u32 p = 0; p < 2; p++)
            for (u32 i = 0; i < a->level; i++) {
                u64 q = c->P.q[i];
                const u64 *x = poly(a, ci, p, i), *w = pt->ntt_q + ((size_t)k * c->L + i) * c->n;
                u64 *z = poly(acc, ci, p, i);
                for (u32 j = 0; j < c->n; j++) z[j] = addmod(z[j], mulmod(x[j], w[j], q), q);
            }
    }
    return 0;
}

int fhe_mul_scalar(fhe_ctx *c, const fhe_ct *a, int64_t w, fhe_ct *out) {
    if (!same_shape(a, out)) return fail(FHE_ELEVEL, "mul_scalar: shape/level mismatch");
    for (u32 ci = 0; ci < a->count; ci++)
        for (u32 p = 0; p < 2; p++)
            for (u32 i = 0; i < a->level; i++) {
                u64 q = c->P.q[i], s = smod(w, q);
                const u64 *x = poly(a, ci, p, i);
                u64 *z = poly(out, ci, p, i);
                for (u32 j = 0; j < c->n; j++) z[j] = mulmod(x[j], s, q);
            }
    return 0;
}

int fhe_add_plain(fhe_ctx *c, const fhe_ct *a, const fhe_pt *pt, fhe_ct *out) {
    if (!same_shape(a, out)) return fail(FHE_ELEVEL, "add_plain: shape/level mismatch");
    u32 n = c->n, l = a->level;
    const level_tab *T = &c->lv[l];
    u64 *tmp = (u64 *)malloc(n * 8);
    if (out != a) memcpy(out->data, a->data, ct_words(a) * 8);
    for (u32 ci = 0; ci < a->count; ci++) {
        u32 k = ci / a->R;
        u64 t = c->P.t[k];
        const u64 *coef = pt->coef_t + (size_t)k * n;
        for (u32 i = 0; i < l; i++) {
            u64 q = c->P.q[i];
            for (u32 x = 0; x < n; x++) tmp[x] = scaled_msg(T, k, t, coef[x], i, q);
            ntt(tmp, &c->M[i], n);
            u64 *z = poly(out, ci, 0, i);
            for (u32 x = 0; x < n; x++) z[x] = addmod(z[x], tmp[x], q);
        }
    }
    free(tmp);
    return 0;
}

/*
 * Hybrid key switching, one prime per digit, one special prime P.
 *   dig_coef[j] : digit j in coefficient form, values in [0, q_j), lifted centered
 *                 into the other primes
 *   dig_ntt[j]  : the same limb in NTT form (NTT_{q_j}(dig_coef[j]))
 * out0/out1 [l][n] NTT domain: round((sum_j d_j * ksk_j) / P) over Q_l.
 */
static void keyswitch(fhe_ctx *c, u32 l, const u64 *dig_coef, const u64 *dig_ntt, const key_node *key,
                      u64 *out0, u64 *out1) {
    u32 n = c->n, L = c->L;
    u64 *acc = (u64 *)calloc((size_t)2 * (l + 1) * n, 8);
    u64 *tmp = (u64 *)malloc(n * 8);
    for (u32 ii = 0; ii <= l; ii++) {
        u32 pi = ii == l ? L : ii;            /* prime index in the key (special = L) */
        u64 q = modof(c, pi);
        u64 *a0 = acc + (size_t)(0 * (l + 1) + ii) * n, *a1 = acc + (size_t)(1 * (l + 1) + ii) * n;
        for (u32 j = 0; j < l; j++) {
            const u64 *ext;
            if (ii == j) {
                ext = dig_ntt + (size_t)j * n;
            } else {
                /* centered lift of the digit (sign-symmetric, so the lift commutes with
                 * automorphisms: hoisted rotations reproduce these words exactly) */
                const u64 *d = dig_coef + (size_t)j * n;
                const u64 qj = c->P.q[j], hj = (qj - 1) / 2;
                for (u32 x = 0; x < n; x++) tmp[x] = d[x] > hj ? smod(-(i64)(qj - d[x]), q) : d[x] % q;
                ntt(tmp, &c->M[pi], n);
                ext = tmp;
            }
            const u64 *kb = key->data + (((size_t)j * 2 + 0) * (L + 1) + pi) * n;
            const u64 *ka = key->data + (((size_t)j * 2 + 1) * (L + 1) + pi) * n;
            for (u32 x = 0; x < n; x++) {
                a0[x] = addmod(a0[x], mulmod(ext[x], kb[x], q), q);
                a1[x] = addmod(a1[x], mulmod(ext[x], ka[x], q), q);
            }
        }
    }
    /* ModDown */
    u64 P = c->P.p[0];
    for (u32 p = 0; p < 2; p++) {
        u64 *r = acc + (size_t)(p * (l + 1) + l) * n;
        intt(r, &c->M[L], n);
        u64 *dst = p == 0 ? out0 : out1;
        for (u32 i = 0; i < l; i++) {
            u64 q = c->P.q[i];
            for (u32 x = 0; x < n; x++) {
                i64 v = r[x] > (P - 1) / 2 ? -(i64)(P - r[x]) : (i64)r[x];
                tmp[x] = smod(v, q);
            }
            ntt(tmp, &c->M[i], n);
            const u64 *ai = acc + (size_t)(p * (l + 1) + i) * n;
            u64 *d = dst + (size_t)i * n;
            for (u32 x = 0; x < n; x++) d[x] = mulmod(submod(ai[x], tmp[x], q), c->pinv[i], q);
        }
    }
    free(acc); free(tmp);
}

int fhe_rotate(fhe_ctx *c, const fhe_ct *a, uint32_t k, fhe_ct *out) {
    if (k == 0 || k >= c->N) return fail(FHE_EINVAL, "rotation step %u outside [1, %u)", k, c->N);
    if (!same_shape(a, out)) return fail(FHE_ELEVEL, "rotate: shape/level mismatch");
    if (a == out) return fail(FHE_EINVAL, "rotate: out must not alias the input");
    u32 n = c->n, l = a->level;
    u32 g = galois_elt(c, k);
    key_node *key = get_key(c, g);
    u64 *c1r = (u64 *)malloc((size_t)l * n * 8), *dig = (u64 *)malloc((size_t)l * n * 8);
    u64 *o0 = (u64 *)malloc((size_t)l * n * 8), *o1 = (u64 *)malloc((size_t)l * n * 8);
    for (u32 ci = 0; ci < a->count; ci++) {
        for (u32 i = 0; i < l; i++) {
            automorph(c, poly(a, ci, 1, i), c1r + (size_t)i * n, g);
            memcpy(dig + (size_t)i * n, c1r + (size_t)i * n, n * 8);
            intt(dig + (size_t)i * n, &c->M[i], n);
        }
        keyswitch(c, l, dig, c1r, key, o0, o1);
        for (u32 i = 0; i < l; i++) {
            u64 q = c->P.q[i];
            u64 *z0 = poly(out, ci, 0, i), *z1 = poly(out, ci, 1, i);
            automorph(c, poly(a, ci, 0, i), z0, g);
            for (u32 x = 0; x < n; x++) z0[x] = addmod(z0[x], o0[(size_t)i * n + x], q);
            memcpy(z1, o1 + (size_t)i * n, n * 8);
        }
    }
    free(c1r); free(dig); free(o0); free(o1);
    return 0;
}

int fhe_mod_switch(fhe_ctx *c, const fhe_ct *a, fhe_ct *out) {
    u32 l = a->level, n = c->n;
    if (l < 2) return fail(FHE_ELEVEL, "mod_switch: already at level 1");
    if (out->level != l - 1 || out->R != a->R) return fail(FHE_ELEVEL, "mod_switch: out must have level %u", l - 1);
    const level_tab *T = &c->lv[l];
    u64 ql = c->P.q[l - 1];
    u64 *r = (u64 *)malloc(n * 8), *tmp = (u64 *)malloc(n * 8);
    for (u32 ci = 0; ci < a->count; ci++)
        for (u32 p = 0; p < 2; p++) {
            memcpy(r, poly(a, ci, p, l - 1), n * 8);
            intt(r, &c->M[l - 1], n);
            for (u32 i = 0; i < l - 1; i++) {
                u64 q = c->P.q[i];
                for (u32 x = 0; x < n; x++) {
                    i64 v = r[x] > (ql - 1) / 2 ? -(i64)(ql - r[x]) : (i64)r[x];
                    tmp[x] = smod(v, q);
                }
                ntt(tmp, &c->M[i], n);
                const u64 *src = poly(a, ci, p, i);
                u64 *dst = poly(out, ci, p, i);
                for (u32 x = 0; x < n; x++) dst[x] = mulmod(submod(src[x], tmp[x], q), T->msinv[i], q);
            }
        }
    free(r); free(tmp);
    return 0;
}

/*
 * ct x ct square, HPS-style: exact centered lift Q_l -> B, tensor in Q_l u B,
 * round(t/Q_l * d) computed into B with a 128-bit fixed-point fraction sum,
 * centered lift B -> Q_l, then relinearization of d2 with the s^2 key.
 */
int fhe_square(fhe_ctx *c, const fhe_ct *a, fhe_ct *out) {
    if (!c->nb) return fail(FHE_EINVAL, "square: context created without an auxiliary base");
    if (!same_shape(a, out)) return fail(FHE_ELEVEL, "square: shape/level mismatch");
    if (a == out) return fail(FHE_EINVAL, "square: out must not alias the input");
    u32 n = c->n, l = a->level, nb = c->nb, nt = l + nb, L = c->L;
    const level_tab *T = &c->lv[l];
    const aux_tab *A = &c->ax;
    key_node *rk = get_key(c, 0);
    u64 *X = (u64 *)malloc((size_t)2 * nt * n * 8);     /* c0, c1 over Q_l u B */
    u64 *D = (u64 *)malloc((size_t)3 * nt * n * 8);     /* d0, d1, d2          */
    u64 *E = (u64 *)malloc((size_t)3 * l * n * 8);      /* scaled, over Q_l    */
    u64 *En = (u64 *)malloc((size_t)l * n * 8);
    u64 *o0 = (u64 *)malloc((size_t)l * n * 8), *o1 = (u64 *)malloc((size_t)l * n * 8);
#define MODI(ii) ((ii) < l ? c->P.q[ii] : c->P.b[(ii) - l])
#define TABI(ii) (&c->M[(ii) < l ? (ii) : IDX_B(c, (ii) - l)])
    for (u32 ci = 0; ci < a->count; ci++) {
        u32 kt = ci / a->R;
        for (u32 p = 0; p < 2; p++) {
            u64 *Xp = X + (size_t)p * nt * n;
            for (u32 i = 0; i < l; i++) {
                memcpy(Xp + (size_t)i * n, poly(a, ci, p, i), n * 8);
                intt(Xp + (size_t)i * n, &c->M[i], n);
            }
            for (u32 x = 0; x < n; x++) {
                u64 y[FHE_MAX_Q];
                u128 ai = 0, af = 0;
                for (u32 i = 0; i < l; i++) {
                    y[i] = mulmod(Xp[(size_t)i * n + x], T->Qtilde[i], c->P.q[i]);
                    fx_acc(&ai, &af, y[i], 0, T->invq[i]);
                }
                u64 v = (u64)(ai + (af >> 127));
                for (u32 k = 0; k < nb; k++) {
                    u64 bk = c->P.b[k], s = 0;
                    for (u32 i = 0; i < l; i++) s = addmod(s, mulmod(y[i], T->QhatB[i][k], bk), bk);
                    s = submod(s, mulmod(v % bk, T->QmodB[k], bk), bk);
                    Xp[(size_t)(l + k) * n + x] = s;
                }
            }
            for (u32 ii = 0; ii < nt; ii++) ntt(Xp + (size_t)ii * n, TABI(ii), n);
        }
        for (u32 ii = 0; ii < nt; ii++) {
            u64 q = MODI(ii);
            const u64 *x0 = X + (size_t)ii * n, *x1 = X + (size_t)(nt + ii) * n;
            u64 *d0 = D + (size_t)ii * n, *d1 = D + (size_t)(nt + ii) * n, *d2 = D + (size_t)(2 * nt + ii) * n;
            for (u32 x = 0; x < n; x++) {
                d0[x] = mulmod(x0[x], x0[x], q);
                u64 m = mulmod(x0[x], x1[x], q);
                d1[x] = addmod(m, m, q);
                d2[x] = mulmod(x1[x], x1[x], q);
            }
            intt(d0, TABI(ii), n); intt(d1, TABI(ii), n); intt(d2, TABI(ii), n);
        }
        for (u32 p = 0; p < 3; p++) {
            const u64 *Dp = D + (size_t)p * nt * n;
            u64 *Ep = E + (size_t)p * l * n;
            for (u32 x = 0; x < n; x++) {
                u64 y[FHE_MAX_Q], R[FHE_MAX_B];
                u128 ai = 0, af = 0;
                for (u32 i = 0; i < l; i++) {
                    y[i] = mulmod(Dp[(size_t)i * n + x], T->Mtq[i], c->P.q[i]);
                    fx_acc(&ai, &af, y[i], 0, T->theta[kt][i]);
                }
                u128 rnd = ai + (af >> 127);
                for (u32 k = 0; k < nb; k++) {
                    u64 bk = c->P.b[k];
                    u64 s = (u64)(rnd % bk);
                    for (u32 i = 0; i < l; i++) s = addmod(s, mulmod(y[i], T->omega[kt][i][k], bk), bk);
                    u64 z = mulmod(Dp[(size_t)(l + k) * n + x], T->Mtb[k], bk);
                    s = addmod(s, mulmod(z, T->tBb[kt][k], bk), bk);
                    R[k] = s;
                }
                /* B -> Q_l, centered */
                u64 yb[FHE_MAX_B];
                ai = 0; af = 0;
                for (u32 k = 0; k < nb; k++) {
                    yb[k] = mulmod(R[k], A->Btilde[k], c->P.b[k]);
                    fx_acc(&ai, &af, yb[k], 0, A->invb[k]);
                }
                u64 v = (u64)(ai + (af >> 127));
                for (u32 i = 0; i < l; i++) {
                    u64 q = c->P.q[i], s = 0;
                    for (u32 k = 0; k < nb; k++) s = addmod(s, mulmod(yb[k], A->BhatQ[k][i], q), q);
                    s = submod(s, mulmod(v % q, A->BmodQ[i], q), q);
                    Ep[(size_t)i * n + x] = s;
                }
            }
        }
        /* relinearize: digits of e2 */
        u64 *E2 = E + (size_t)2 * l * n;
        for (u32 i = 0; i < l; i++) {
            memcpy(En + (size_t)i * n, E2 + (size_t)i * n, n * 8);
            ntt(En + (size_t)i * n, &c->M[i], n);
        }
        keyswitch(c, l, E2, En, rk, o0, o1);
        for (u32 p = 0; p < 2; p++)
            for (u32 i = 0; i < l; i++) {
                u64 q = c->P.q[i];
                u64 *z = poly(out, ci, p, i);
                memcpy(z, E + ((size_t)p * l + i) * n, n * 8);
                ntt(z, &c->M[i], n);
                const u64 *o = (p == 0 ? o0 : o1) + (size_t)i * n;
                for (u32 x = 0; x < n; x++) z[x] = addmod(z[x], o[x], q);
            }
    }
#undef MODI
#undef TABI
    free(X); free(D); free(E); free(En); free(o0); free(o1);
    (void)L;
    return 0;
}

int fhe_hoisted_dot(fhe_ctx *c, fhe_ct *const *R, const uint32_t *g, uint32_t K, fhe_pt *const *pt,
                    uint32_t S, fhe_ct *const *out) {
    if (!K) return fail(FHE_EINVAL, "hoisted_dot: K must be >= 1");
    u32 n = c->n, l = R[0]->level;
    for (u32 k = 0; k < K; k++)
        if (!same_shape(R[k], R[0]) || !(g[k] & 1)) return fail(FHE_EINVAL, "hoisted_dot: bad operand %u", k);
    u64 *tp = (u64 *)malloc((size_t)n * 8);
    for (u32 s = 0; s < S; s++) {
        if (!same_shape(out[s], R[0])) { free(tp); return fail(FHE_ELEVEL, "hoisted_dot: output shape mismatch"); }
        memset(out[s]->data, 0, ct_words(out[s]) * 8);
        for (u32 k = 0; k < K; k++)
            for (u32 ci = 0; ci < R[0]->count; ci++) {
                u32 kt = ci / R[0]->R;
                for (u32 i = 0; i < l; i++) {
                    u64 q = c->P.q[i];
                    automorph(c, pt[s]->ntt_q + ((size_t)kt * c->L + i) * n, tp, g[k]);
                    for (u32 p = 0; p < 2; p++) {
                        const u64 *x = poly(R[k], ci, p, i);
                        u64 *z = poly(out[s], ci, p, i);
                        for (u32 j = 0; j < n; j++) z[j] = addmod(z[j], mulmod(x[j], tp[j], q), q);
                    }
                }
            }
    }
    free(tp);
    return 0;
}
int fhe_rotate_many(fhe_ctx *c, fhe_ct *const *a, fhe_ct *const *out, uint32_t m, uint32_t k) {
    for (u32 i = 0; i < m; i++) { int rc = fhe_rotate(c, a[i], k, out[i]); if (rc) return rc; }
    return 0;
}
int fhe_rotate_add_many(fhe_ctx *c, fhe_ct *const *a, fhe_ct *const *out, uint32_t m, uint32_t k) {
    for (u32 i = 0; i < m; i++) {
        int rc = fhe_rotate(c, a[i], k, out[i]);
        if (rc) return rc;
        rc = fhe_add(c, a[i], out[i], out[i]);
        if (rc) return rc;
    }
    return 0;
}
int fhe_rotate_multi(fhe_ctx *c, fhe_ct *const *a, fhe_ct *const *out, const uint32_t *k, uint32_t m) {
    for (u32 i = 0; i < m; i++) { int rc = fhe_rotate(c, a[i], k[i], out[i]); if (rc) return rc; }
    return 0;
}

/* hoisting is a device-side cost optimisation; the words are those of separate rotations */
int fhe_rotate_hoisted(fhe_ctx *c, const fhe_ct *a, const uint32_t *k, uint32_t m, fhe_ct *const *out) {
    for (uint32_t j = 0; j < m; j++) {
        int rc = fhe_rotate(c, a, k[j], out[j]);
        if (rc) return rc;
    }
    return 0;
}
int fhe_mul_plain_many(fhe_ctx *c, fhe_ct *const *a, fhe_pt *const *pt, fhe_ct *const *out, uint32_t m) {
    for (u32 i = 0; i < m; i++) { int rc = fhe_mul_plain(c, a[i], pt[i], out[i]); if (rc) return rc; }
    return 0;
}
int fhe_add_many(fhe_ctx *c, fhe_ct *const *a, fhe_ct *const *b, fhe_ct *const *out, uint32_t m) {
    for (u32 i = 0; i < m; i++) { int rc = fhe_add(c, a[i], b[i], out[i]); if (rc) return rc; }
    return 0;
}

/* ---- composite entry points (same words as the sequences they stand for) ---- */

/* hesim.py:347-366: acc <- acc + rotate(acc, 2^h) for h = ceil(log2 span) - 1 .. 0 */
int fhe_rotate_and_sum(fhe_ctx *c, fhe_ct *const *a, fhe_ct *const *out, uint32_t m, uint32_t span) {
    if (span < 1 || span > c->N) return fail(FHE_EINVAL, "rotate_and_sum: span %u outside [1, %u]", span, c->N);
    u32 rounds = 0;
    while ((1u << rounds) < span) rounds++;
    for (u32 i = 0; i < m; i++) {
        if (!same_shape(a[i], out[i])) return fail(FHE_ELEVEL, "rotate_and_sum: shape/level mismatch");
        if (a[i] == out[i]) return fail(FHE_EINVAL, "rotate_and_sum: out must not alias the input");
        fhe_ct *tmp = NULL;
        int rc = fhe_ct_create(c, a[i]->R, a[i]->level, &tmp);
        if (rc) return rc;
        memcpy(out[i]->data, a[i]->data, ct_words(a[i]) * 8);
        for (u32 h = rounds; h-- > 0 && !rc;) {
            rc = fhe_rotate(c, out[i], 1u << h, tmp);
            if (!rc) rc = fhe_add(c, out[i], tmp, out[i]);
        }
        fhe_ct_destroy(tmp);
        if (rc) return rc;
    }
    return 0;
}

/* packing.py:350-368 as a pairwise tree: every level merges adjacent blocks (left, right)
 * into left + rotate(right, N - len(left)); an odd last block moves up unchanged. */
int fhe_combine(fhe_ctx *c, fhe_ct *const *cts, const uint32_t *lengths, uint32_t m, fhe_ct *out) {
    if (m < 1) return fail(FHE_EINVAL, "combine: no ciphertexts");
    u64 total = 0;
    for (u32 i = 0; i < m; i++) {
        if (!same_shape(cts[i], out)) return fail(FHE_ELEVEL, "combine: shape/level mismatch");
        if (cts[i] == out) return fail(FHE_EINVAL, "combine: out must not alias an input");
        if (lengths[i] < 1) return fail(FHE_EINVAL, "combine: payload %u is empty", i);
        total += lengths[i];
    }
    if (total > c->N) return fail(FHE_EINVAL, "combine: payload of %llu slots exceeds %u", (unsigned long long)total, c->N);
    fhe_ct **cur = (fhe_ct **)malloc(m * sizeof *cur);
    u32 *len = (u32 *)malloc(m * sizeof *len);
    char *own = (char *)calloc(m, 1);          /* 1: a temporary of this call */
    for (u32 i = 0; i < m; i++) { cur[i] = cts[i]; len[i] = lengths[i]; }
    u32 cnt = m;
    int rc = 0;
    while (cnt > 1 && !rc) {
        u32 w = 0;
        for (u32 k = 0; k + 1 < cnt && !rc; k += 2) {
            fhe_ct *dst = NULL;
            if (cnt == 2) dst = out;
            else rc = fhe_ct_create(c, out->R, out->level, &dst);
            if (rc) break;
            rc = fhe_rotate(c, cur[k + 1], c->N - len[k], dst);
            if (!rc) rc = fhe_add(c, cur[k], dst, dst);
            if (own[k]) fhe_ct_destroy(cur[k]);
            if (own[k + 1]) fhe_ct_destroy(cur[k + 1]);
            cur[w] = dst; len[w] = len[k] + len[k + 1]; own[w] = dst != out; w++;
        }
        if (!rc && (cnt & 1)) { cur[w] = cur[cnt - 1]; len[w] = len[cnt - 1]; own[w] = own[cnt - 1]; w++; }
        cnt = w;
    }
    if (!rc && m == 1) memcpy(out->data, cts[0]->data, ct_words(out) * 8);
    free(cur); free(len); free(own);
    return rc;
}

/* engine.py:178-197 (conv_conv): out[o] = sum_k w[k * O + o] * a[k] */
int fhe_ct_gemm(fhe_ctx *c, fhe_ct *const *a, uint32_t K, const int64_t *w, uint32_t O, fhe_ct *const *out) {
    if (K < 1 || O < 1) return fail(FHE_EINVAL, "ct_gemm: empty operand list");
    for (u32 k = 0; k < K; k++)
        if (!same_shape(a[k], a[0])) return fail(FHE_ELEVEL, "ct_gemm: shape/level mismatch");
    for (u32 o = 0; o < O; o++) {
        if (!same_shape(out[o], a[0])) return fail(FHE_ELEVEL, "ct_gemm: shape/level mismatch");
        for (u32 k = 0; k < K; k++)
            if (out[o] == a[k]) return fail(FHE_EINVAL, "ct_gemm: out must not alias an input");
    }
    for (u32 o = 0; o < O; o++)
        for (u32 ci = 0; ci < a[0]->count; ci++)
            for (u32 p = 0; p < 2; p++)
                for (u32 i = 0; i < a[0]->level; i++) {
                    u64 q = c->P.q[i];
                    u64 *z = poly(out[o], ci, p, i);
                    memset(z, 0, (size_t)c->n * 8);
                    for (u32 k = 0; k < K; k++) {
                        u64 s = smod(w[(size_t)k * O + o], q);
                        const u64 *x = poly(a[k], ci, p, i);
                        for (u32 j = 0; j < c->n; j++) z[j] = addmod(z[j], mulmod(x[j], s, q), q);
                    }
                }
    return 0;
}

/* stages of one rotation's key switch (include/ffconv_he.h: fhe_debug_rotate_stages) */
int fhe_debug_rotate_stages(fhe_ctx *c, const fhe_ct *a, uint32_t k, uint64_t *digits, uint64_t *ext, uint64_t *accout) {
    if (k == 0 || k >= c->N) return fail(FHE_EINVAL, "rotation step %u outside [1, %u)", k, c->N);
    u32 n = c->n, l = a->level, L = c->L;
    u32 g = galois_elt(c, k);
    key_node *key = get_key(c, g);
    u64 *c1r = (u64 *)malloc((size_t)l * n * 8);
    for (u32 ci = 0; ci < a->count; ci++) {
        u64 *dig = digits + (size_t)ci * l * n;
        u64 *ex = ext + (size_t)ci * l * (l + 1) * n;
        u64 *acc = accout + (size_t)ci * 2 * (l + 1) * n;
        memset(ex, 0, (size_t)l * (l + 1) * n * 8);
        memset(acc, 0, (size_t)2 * (l + 1) * n * 8);
        for (u32 i = 0; i < l; i++) {
            automorph(c, poly(a, ci, 1, i), c1r + (size_t)i * n, g);
            memcpy(dig + (size_t)i * n, c1r + (size_t)i * n, n * 8);
            intt(dig + (size_t)i * n, &c->M[i], n);
        }
        for (u32 ii = 0; ii <= l; ii++) {
            u32 pi = ii == l ? L : ii;
            u64 q = modof(c, pi);
            u64 *a0 = acc + (size_t)(0 * (l + 1) + ii) * n, *a1 = acc + (size_t)(1 * (l + 1) + ii) * n;
            for (u32 j = 0; j < l; j++) {
                const u64 *e;
                if (ii == j) {
                    e = c1r + (size_t)j * n;
                } else {
                    u64 *t = ex + ((size_t)j * (l + 1) + ii) * n;
                    const u64 *d = dig + (size_t)j * n;
                    const u64 qj = c->P.q[j], hj = (qj - 1) / 2;
                    for (u32 x = 0; x < n; x++) t[x] = d[x] > hj ? smod(-(i64)(qj - d[x]), q) : d[x] % q;
                    ntt(t, &c->M[pi], n);
                    e = t;
                }
                const u64 *kb = key->data + (((size_t)j * 2 + 0) * (L + 1) + pi) * n;
                const u64 *ka = key->data + (((size_t)j * 2 + 1) * (L + 1) + pi) * n;
                for (u32 x = 0; x < n; x++) {
                    a0[x] = addmod(a0[x], mulmod(e[x], kb[x], q), q);
                    a1[x] = addmod(a1[x], mulmod(e[x], ka[x], q), q);
                }
            }
        }
        for (u32 p = 0; p < 2; p++) intt(acc + (size_t)(p * (l + 1) + l) * n, &c->M[L], n);
    }
    free(c1r);
    return 0;
}
