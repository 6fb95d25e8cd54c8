// ntt_core.cuh -- shared-memory negacyclic NTT cores for one polynomial row per CTA.
//
// Forward (Cooley-Tukey): natural-order coefficients -> evaluations in
// bit-reversed order, a[i] = A(psi^(2 brev(i) + 1)).  Inverse (Gentleman-Sande):
// bit-reversed evaluations -> natural coefficients, scaled by n^-1.  Same
// ordering and twiddles (minimal primitive 2n-th root) as oracle/golden_rlwe.c.
//
// Layout: every thread owns E = 2^W words in registers and runs up to W
// butterfly stages per pass; passes exchange through shared memory padded one
// word per 2^W (conflict-free for 64-bit accesses).  n >= 2^12 uses W = 5
// (radix-32, 512 threads x 128 registers for n = 2^14, 132 KB of shared memory)
// for inverse transforms, W = 4 (1024 x 64) for forward ones: standalone 46 % / 40 %
// of the integer peak (fwd W5 / inv W5) vs 45 % / 35 % at W = 4, but the fused
// forward kernels (ModUp, rescale) run faster at W = 4 (profiles/r01_*).  Values are kept lazily in [0, 4q)
// (forward, Harvey) / [0, 2q) (inverse) and reduced once at the end.
#pragma once
#include "arith.cuh"

#ifndef NTT_W_FWD
#define NTT_W_FWD 4
#endif
#ifndef NTT_W_INV
#define NTT_W_INV 5
#endif

// default radix per pass: 2^5 (512 threads, 32 words each) for the large rings,
// 2^4 below; overridable for experiments (csrc/ntt_bench.cu)
template <int LOGN>
struct DefaultW {      // forward transforms
    static constexpr int value = LOGN < 4 ? LOGN : (LOGN >= 12 ? NTT_W_FWD : 4);
};
template <int LOGN>
struct DefaultWInv {   // inverse transforms
    static constexpr int value = LOGN < 4 ? LOGN : (LOGN >= 12 ? NTT_W_INV : 4);
};


template <int LOGN, int WW = DefaultW<LOGN>::value>
struct NttCfg {
    static constexpr int N = 1 << LOGN;
    static constexpr int W = WW;                        // stages per pass
    static constexpr int E = 1 << W;                    // words per thread
    static constexpr int TH = N / E;                    // threads per row
    static constexpr int NP = (LOGN + W - 1) / W;       // passes
    static constexpr int SMEM_WORDS = N + (N >> W) + 1;
    // one pad word per 2^W: every pass's access pattern is conflict-free for 64-bit words
    static DEV int pad(int i) { return i + (i >> W); }
};
template <int LOGN> using FwdCfg = NttCfg<LOGN, DefaultW<LOGN>::value>;
template <int LOGN> using InvCfg = NttCfg<LOGN, DefaultWInv<LOGN>::value>;

// insert the W bits of e at bit position f0 of the thread index
template <int W>
DEV int fidx(int tid, int e, int f0) {
    int lo = tid & ((1 << f0) - 1), hi = tid >> f0;
    return (hi << (f0 + W)) | (e << f0) | lo;
}

// Forward. In: v[] holds element fidx(tid, e, LOGN - W) (i.e. v[e] = a[(e << (LOGN-W)) | tid])
// with values < 4q.  Out: canonical values in sm[C::pad(i)], bit-reversed order; ends
// with __syncthreads().
template <int LOGN, int WW = DefaultW<LOGN>::value>
DEV void ntt_fwd_core(u64 (&v)[NttCfg<LOGN, WW>::E], u64 *sm, const ModInfo &M, int tid) {
    using C = NttCfg<LOGN, WW>;
    constexpr int W = C::W, E = C::E, NP = C::NP;
    const u64 q = M.q, q2 = 2 * q;
#pragma unroll
    for (int p = 0; p < NP; p++) {
        const int s0 = p * W;
        const int f0 = (LOGN - s0 - W) > 0 ? (LOGN - s0 - W) : 0;
        const int k = (LOGN - s0) < W ? (LOGN - s0) : W;
        if (p > 0) {
#pragma unroll
            for (int e = 0; e < E; e++) v[e] = sm[C::pad(fidx<W>(tid, e, f0))];
            __syncthreads();
        }
#pragma unroll
        for (int ls = 0; ls < k; ls++) {
            const int s = s0 + ls;
            const int b = LOGN - s - 1 - f0;
#pragma unroll
            for (int e = 0; e < E; e++) {
                if (e & (1 << b)) continue;
                const int e2 = e | (1 << b);
                const u32 g = (1u << s) + ((u32)fidx<W>(tid, e, f0) >> (LOGN - s));
                const ulonglong2 tw = __ldg(M.tw + g);
                const u64 w = tw.x, wsh = tw.y;
                u64 U = v[e];
                U = U >= q2 ? U - q2 : U;
                u64 V = shoup_lazy(v[e2], w, wsh, q);
                v[e] = U + V;
                v[e2] = U - V + q2;
            }
        }
        if (p == NP - 1) {
#pragma unroll
            for (int e = 0; e < E; e++) {
                u64 x = v[e];
                x = x >= q2 ? x - q2 : x;
                v[e] = x >= q ? x - q : x;
            }
        }
#pragma unroll
        for (int e = 0; e < E; e++) sm[C::pad(fidx<W>(tid, e, f0))] = v[e];
        __syncthreads();
    }
}

// Inverse. In: canonical (or < 2q) values in sm[C::pad(i)], bit-reversed order, synced.
// Out: v[e] = a[(e << (LOGN-W)) | tid] canonical, scaled by n^-1.  Shared memory is
// free for reuse only after a __syncthreads() by the caller.
template <int LOGN, int WW = DefaultWInv<LOGN>::value>
DEV void ntt_inv_core(u64 (&v)[NttCfg<LOGN, WW>::E], u64 *sm, const ModInfo &M, int tid, u32 g_perm = 0) {
    using C = NttCfg<LOGN, WW>;
    constexpr int W = C::W, E = C::E, NP = C::NP, N = C::N;
    const u64 q = M.q, q2 = 2 * q;
#pragma unroll
    for (int p = 0; p < NP; p++) {
        const int lt0 = p * W;                                   // log2 t of the first stage
        const int f0 = (lt0 + W) <= LOGN ? lt0 : LOGN - W;
        const int k = (LOGN - lt0) < W ? (LOGN - lt0) : W;
        if (p == 0 && g_perm) {
#pragma unroll
            for (int e = 0; e < E; e++) v[e] = sm[C::pad(galois_perm(fidx<W>(tid, e, f0), g_perm, LOGN))];
        } else {
#pragma unroll
            for (int e = 0; e < E; e++) v[e] = sm[C::pad(fidx<W>(tid, e, f0))];
        }
        if (p < NP - 1) __syncthreads();
#pragma unroll
        for (int ls = 0; ls < k; ls++) {
            const int lt = lt0 + ls;
            const int b = lt - f0;
            const int h = N >> (lt + 1);
#pragma unroll
            for (int e = 0; e < E; e++) {
                if (e & (1 << b)) continue;
                const int e2 = e | (1 << b);
                const u32 g = (u32)h + ((u32)fidx<W>(tid, e, f0) >> (lt + 1));
                const ulonglong2 tw = __ldg(M.itw + g);
                const u64 w = tw.x, wsh = tw.y;
                u64 U = v[e], V = v[e2];
                u64 s = U + V;
                v[e] = s >= q2 ? s - q2 : s;
                v[e2] = shoup_lazy(U - V + q2, w, wsh, q);
            }
        }
        if (p < NP - 1) {
#pragma unroll
            for (int e = 0; e < E; e++) sm[C::pad(fidx<W>(tid, e, f0))] = v[e];
            __syncthreads();
        }
    }
#pragma unroll
    for (int e = 0; e < E; e++) v[e] = shoup(v[e], M.ninv, M.ninv_sh, q);
}

