// arith.cuh -- modular arithmetic, fixed-point sums and ChaCha20 samplers for
// the sm_100a evaluator.  Integer pipes only: 64-bit words, primes < 2^61.
//
//  * Shoup multiplication (fixed operand w with w' = floor(w 2^64 / q)) for NTT
//    twiddles and per-prime scalars: mul.lo + mul.hi + mul.lo, lazy in [0, 2q).
//  * Montgomery multiplication (R = 2^64) for operand pairs that are both
//    data (ct x pt, key inner products): operands stored pre-scaled by R.
//  * 64-bit Barrett-style reduction with mu = floor(2^64 / q).
//
// The sampler conventions (block layout, domains, CBD(21), ternary mod 3) are
// the golden spec shared with oracle/golden_rlwe.c.
#pragma once
#include <cstdint>

typedef uint64_t u64;
typedef uint32_t u32;
typedef int64_t i64;
typedef unsigned __int128 u128;

#define DEV __device__ __forceinline__
#define HD __host__ __device__ __forceinline__

struct ModInfo {
    u64 q;
    u64 qinv;      // q^-1 mod 2^64 (Montgomery)
    u64 r2;        // 2^128 mod q
    u64 mu;        // floor(2^64 / q)
    u64 ninv, ninv_sh;
    u64 w1ninv, w1ninv_sh;     // (last inverse-NTT twiddle) * n^-1: the scaling folds into the last stage
    u64 half;      // (q - 1) / 2
    u64 nq;        // -q mod 2^64 (the quotient subtraction folds into a multiply-add)
    u64 q3;        // 3q, loaded (not derived) so ptxas keeps it in a register instead of
                   // re-deriving U + 3q with an IMAD per butterfly
    const ulonglong2 *tw;      // (psi^brev(k), Shoup companion) pairs
    const ulonglong2 *itw;     // (psi^-brev(k), Shoup companion) pairs
};

DEV u64 mulhi(u64 a, u64 b) { return __umul64hi(a, b); }

// a*w mod q in [0, 2q), any 64-bit a
DEV u64 shoup_lazy(u64 a, u64 w, u64 wsh, u64 q) { return a * w - mulhi(a, wsh) * q; }
DEV u64 shoup(u64 a, u64 w, u64 wsh, u64 q) {
    u64 r = shoup_lazy(a, w, wsh, q);
    return r >= q ? r - q : r;
}
// floor(a b / 2^64) or one less: the low partial product a0 b0 is dropped
// (it only carries at most 1 into the high word).  5 IMADs instead of 7.
DEV u64 mulhi_approx(u64 a, u64 b) {
    const u32 a0 = (u32)a, a1 = (u32)(a >> 32), b0 = (u32)b, b1 = (u32)(b >> 32);
    u32 t0, t1, t2;       // t0: low word, only its carry is used
    asm("mul.lo.u32 %0, %4, %5;\n\t"
        "mul.hi.u32 %1, %4, %5;\n\t"
        "mad.lo.cc.u32 %0, %3, %6, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %6, %1;\n\t"
        "addc.u32 %2, 0, 0;\n\t"
        "mad.lo.cc.u32 %1, %4, %6, %1;\n\t"
        "madc.hi.u32 %2, %4, %6, %2;"
        : "=&r"(t0), "=&r"(t1), "=&r"(t2)
        : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
    return ((u64)t2 << 32) | t1;
}
// a*w mod q in [0, 3q) for any 64-bit a (Shoup with the approximate quotient);
// nq = -q mod 2^64 turns a*w - qhat*q into two multiply-adds.
DEV u64 shoup_approx(u64 a, u64 w, u64 wsh, u64 nq) { return a * w + mulhi_approx(a, wsh) * nq; }
// x mod q, canonical, for any 64-bit x (Barrett with mu = floor(2^64/q): x - qhat q < 3q)
DEV u64 red_any(u64 x, u64 q, u64 mu, u64 nq) {
    u64 r = x + mulhi_approx(x, mu) * nq;
    r = r >= 2 * q ? r - 2 * q : r;
    return r >= q ? r - q : r;
}
// a*b*2^-64 mod q, canonical; requires a*b < q*2^64 (e.g. b < q)
DEV u64 mont(u64 a, u64 b, u64 q, u64 qinv) {
    u64 lo = a * b, hi = mulhi(a, b);
    u64 m = lo * qinv;
    u64 mh = mulhi(m, q);
    return hi >= mh ? hi - mh : hi - mh + q;
}
// Montgomery reduction of a 128-bit value T = (hi, lo) < q 2^64: T 2^-64 mod q
DEV u64 mont_reduce(u64 hi, u64 lo, u64 q, u64 qinv) {
    u64 m = lo * qinv;
    u64 mh = mulhi(m, q);
    return hi >= mh ? hi - mh : hi - mh + q;
}
DEV void mac128(u64 &hi, u64 &lo, u64 a, u64 b) {      // (hi, lo) += a * b (exact, carry chained)
    asm("mad.lo.cc.u64 %0, %2, %3, %0;\n\t"
        "madc.hi.u64 %1, %2, %3, %1;"
        : "+l"(lo), "+l"(hi)
        : "l"(a), "l"(b));
}
DEV u64 addm(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
DEV u64 subm(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
DEV u64 negm(u64 a, u64 q) { return a ? q - a : 0; }
// x mod q for any 64-bit x
DEV u64 red64(u64 x, u64 q, u64 mu) {
    u64 r = x - mulhi(x, mu) * q;
    while (r >= q) r -= q;
    return r;
}
// a*b mod q for a, b < q (two Montgomery steps)
DEV u64 mulmod(u64 a, u64 b, const ModInfo &M) { return mont(mont(a, b, M.q, M.qinv), M.r2, M.q, M.qinv); }
DEV u64 to_mont(u64 a, const ModInfo &M) { return mont(a, M.r2, M.q, M.qinv); }
// signed -> [0, q)
DEV u64 smod(i64 v, const ModInfo &M) {
    if (v >= 0) return red64((u64)v, M.q, M.mu);
    u64 r = red64((u64)(-(v + 1)), M.q, M.mu);
    return M.q - 1 - r;
}
// x in [0, m_src) read as centered (x > (m_src-1)/2 -> x - m_src), then mod q;
// msrc_q = m_src mod q
DEV u64 centered_lift(u64 x, u64 half_src, u64 msrc_q, const ModInfo &M) {
    u64 r = red64(x, M.q, M.mu);
    return x > half_src ? subm(r, msrc_q, M.q) : r;
}
// The same lift, lazily: a representative in [0, 4q) (forward-NTT input bound).
// x + (-x/q approx) q lies in [0, 3q); the negative branch adds q - (m_src mod q).
DEV u64 centered_lift_lazy(u64 x, u64 half_src, u64 msrc_q, const ModInfo &M) {
    const u64 r = x + mulhi_approx(x, M.mu) * M.nq;
    return x > half_src ? r + (M.q - msrc_q) : r;
}
// The same lift without any multiplication, for source moduli below 8q: a centered value
// lies in [-half_src, half_src], so when half_src < 4q the non-negative ones already are
// representatives below 4q (the forward NTT's input bound) and the negative ones become so
// after adding k q, k = ceil(half_src / q) <= 4.  lift_offset returns k q - m_src (mod
// 2^64), or 0 when the source modulus is too large and the Barrett form must be used
// (0 is never a valid offset: k q = m_src has no solution for distinct primes).
DEV u64 lift_offset(u64 half_src, u64 m_src, u64 q) {
    if (half_src >= 4 * q) return 0;
    const u64 k = 1 + (half_src > q) + (half_src > 2 * q) + (half_src > 3 * q);
    return k * q - m_src;
}
DEV u64 centered_lift_add(u64 x, u64 half_src, u64 off) { return x > half_src ? x + off : x; }
// x mod q, lazily in [0, 3q), any 64-bit x
DEV u64 red_lazy(u64 x, const ModInfo &M) { return x + mulhi_approx(x, M.mu) * M.nq; }
// x (128-bit) mod q
DEV u64 mod128(u128 x, const ModInfo &M) {
    u64 hi = red64((u64)(x >> 64), M.q, M.mu), lo = red64((u64)x, M.q, M.mu);
    // 2^64 mod q = mont(r2, 1) ... use r2 = 2^128 mod q: hi * 2^64 = mont(hi, r2)
    return addm(mont(hi, M.r2, M.q, M.qinv), lo, M.q);
}

// accumulate y * (W + F / 2^128) into (ai, af) exactly (golden: fx_acc)
DEV void fx_acc(u128 &ai, u128 &af, u64 y, u64 W, u64 Fhi, u64 Flo) {
    u128 p_lo = (u128)y * Flo;
    u128 p_hi = (u128)y * Fhi;
    u128 low = p_lo + (p_hi << 64);
    u128 c1 = low < p_lo;
    u128 ip = (p_hi >> 64) + c1;
    af += low;
    u128 c2 = af < low;
    ai += (u128)y * W + ip + c2;
}

// ------------------------------------------------------------------ ChaCha20
enum { DOM_SK = 1, DOM_ENC_A = 2, DOM_ENC_E = 3, DOM_KSK_A = 4, DOM_KSK_E = 5 };

DEV u32 rotl32(u32 a, int b) { return __funnelshift_l(a, a, b); }
#define CQR(a, b, c, d)                      \
    a += b; d ^= a; d = rotl32(d, 16);       \
    c += d; b ^= c; b = rotl32(b, 12);       \
    a += b; d ^= a; d = rotl32(d, 8);        \
    c += d; b ^= c; b = rotl32(b, 7);

DEV void chacha_block(u32 out[16], u64 seed, u32 ctr, u32 dom, u32 sub, u32 x, u32 y) {
    u32 in[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                  (u32)seed, (u32)(seed >> 32), 0x243F6A88u, 0x85A308D3u,
                  0x13198A2Eu, 0x03707344u, 0xA4093822u, 0x299F31D0u,
                  ctr, (dom << 24) | (sub & 0xFFFFFFu), x, y};
    u32 s[16];
#pragma unroll
    for (int i = 0; i < 16; i++) s[i] = in[i];
#pragma unroll 1
    for (int i = 0; i < 10; i++) {
        CQR(s[0], s[4], s[8], s[12]);
        CQR(s[1], s[5], s[9], s[13]);
        CQR(s[2], s[6], s[10], s[14]);
        CQR(s[3], s[7], s[11], s[15]);
        CQR(s[0], s[5], s[10], s[15]);
        CQR(s[1], s[6], s[11], s[12]);
        CQR(s[2], s[7], s[8], s[13]);
        CQR(s[3], s[4], s[9], s[14]);
    }
#pragma unroll
    for (int i = 0; i < 16; i++) out[i] = s[i] + in[i];
}

// uniform residue for coefficient c (words 4(c%4)..+3 of block c/4)
DEV u64 sample_uniform(const ModInfo &M, u64 seed, u32 dom, u32 sub, u32 x, u32 y, u32 c) {
    u32 blk[16];
    chacha_block(blk, seed, c >> 2, dom, sub, x, y);
    const int o = 4 * (c & 3);
    u128 v = ((u128)blk[o + 3] << 96) | ((u128)blk[o + 2] << 64) | ((u128)blk[o + 1] << 32) | blk[o];
    return mod128(v, M);
}
DEV int sample_ternary(u64 seed, u32 dom, u32 sub, u32 x, u32 y, u32 c) {
    u32 blk[16];
    chacha_block(blk, seed, c >> 4, dom, sub, x, y);
    u32 r = blk[c & 15] % 3u;
    return r == 2 ? -1 : (int)r;
}
DEV int sample_cbd(u64 seed, u32 dom, u32 sub, u32 x, u32 y, u32 c) {
    u32 blk[16];
    chacha_block(blk, seed, c >> 3, dom, sub, x, y);
    u32 w0 = blk[2 * (c & 7)] & 0x1FFFFFu, w1 = blk[2 * (c & 7) + 1] & 0x1FFFFFu;
    return __popc(w0) - __popc(w1);
}

DEV u32 brev_n(u32 x, int logn) { return __brev(x) >> (32 - logn); }
// NTT-domain automorphism X -> X^g: out[j] = in[perm(j)]
DEV u32 galois_perm(u32 j, u32 g, int logn) {
    u32 e = 2u * brev_n(j, logn) + 1u;
    u32 eg = (u32)(((u64)e * g) & ((2ull << logn) - 1));
    return brev_n((eg - 1u) >> 1, logn);
}
