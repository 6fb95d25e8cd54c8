// ntt_core.cuh -- shared-memory negacyclic NTT cores for one polynomial row per CTA.
//
// Forward (Cooley-Tukey): natural-order coefficients -> evaluations in
// bit-reversed order, a[i] = A(psi^(2 brev(i) + 1)).  Inverse (Gentleman-Sande):
// bit-reversed evaluations -> natural coefficients, scaled by n^-1.  Same
// ordering and twiddles (minimal primitive 2n-th root) as oracle/golden_rlwe.c.
//
// Layout: every thread owns E = 2^W words in registers and runs up to W
// butterfly stages per pass; passes exchange through shared memory padded one
// word per 2^W (conflict-free for 64-bit accesses).  Default W = 4 (radix-16,
// 1024 threads x 64 registers for n = 2^14, 139 KB of shared memory) for both
// directions and every fused row kernel: radix-32 passes (W = 5, kept as a per-kernel
// knob) measured slower once the warp-local exchange fences were in.
// Butterfly values are kept lazily bounded (FwdLazy / InvLazy below) and reduced
// once at the end.
#pragma once
#include "arith.cuh"

// Lazy-reduction schedule.  Butterfly values are bounded, not reduced: with
// LIM = 2^clz(q) (so LIM q < 2^64), a forward (Cooley-Tukey) stage adds < 3q to
// every value (approximate-quotient Shoup products lie in [0, 3q)) and the U
// operands are conditionally reduced by (LIM/2) q only in the stages where the
// bound would pass LIM q; an inverse (Gentleman-Sande) stage doubles the bound of
// the sums, which are conditionally reduced once it reaches LIM/2.  Bounds are
// tracked in units of q, uniformly over the CTA, so the reduction choice is a
// uniform branch per stage.  A forward NTT never reduces for q < 2^58; neither
// does an inverse one for the 40-bit primes of configs[1].  The outputs are
// canonical, hence bit-identical to the exact butterflies of the golden model.
struct FwdLazy {
    u64 nq, q3, cq;
    int lim, B;          // LIM, and the current bound of every value (units of q)
    bool red;            // this stage reduces its U operands by cq
    DEV explicit FwdLazy(const ModInfo &M) : nq(M.nq), q3(M.q3), B(4), red(false) {
        const int z = min(__clzll(M.q), 24);
        lim = 1 << z;
        cq = M.q << (z - 1);
    }
    // inputs < 4q; call once per stage, before its butterflies
    DEV void stage() {
        red = B + 3 > lim;
        B = red ? max((lim >> 1) + 1, B - (lim >> 1)) + 3 : B + 3;
    }
    // approximate conditional subtraction on the high words: u >= cq is certain when
    // hi(u) > hi(cq); otherwise u < cq + 2^32 < cq + q (reductions only happen for
    // q >= 2^58, where LIM q would otherwise overflow), hence the "+ 1" in stage()
    DEV u64 cred(u64 u) const { return (u32)(u >> 32) > (u32)(cq >> 32) ? u - cq : u; }
    DEV void bfly(u64 &a, u64 &b, const ulonglong2 &tw) const {
        const u64 U = a, V = shoup_approx(b, tw.x, tw.y, nq);
        a = U + V;
        b = U - V + q3;
    }
};
struct InvLazy {
    u64 q, nq, Bq;       // Bq = (input bound) * q
    int lgB, sB;         // log2 of the largest bound, log2 of the current bound
    bool red;            // this stage reduces its sums by Bq
    DEV explicit InvLazy(const ModInfo &M) : q(M.q), nq(M.nq), Bq(2 * M.q), sB(1), red(false) {
        lgB = min(__clzll(M.q), 24) - 1;
    }
    // inputs < 2q; call once per stage, before its butterflies
    DEV void stage() {
        Bq = q << sB;
        red = sB + 1 > lgB;
        if (!red) sB++;
    }
    DEV u64 cred(u64 s) const { return s >= Bq ? s - Bq : s; }
    DEV void bfly(u64 &a, u64 &b, const ulonglong2 &tw) const {
        const u64 U = a, V = b;
        a = U + V;
        b = shoup_approx(U - V + Bq, tw.x, tw.y, nq);
    }
    // last stage (one twiddle w1 for every butterfly) with the n^-1 scaling folded in:
    // canonical outputs (U + V) n^-1 and (U - V) w1 n^-1
    DEV void last(u64 &a, u64 &b, const ModInfo &M) const {
        const u64 U = a, V = b;
        a = shoup(U + V, M.ninv, M.ninv_sh, q);
        b = shoup(U - V + Bq, M.w1ninv, M.w1ninv_sh, q);
    }
};

#ifndef NTT_EXP
#define NTT_EXP 0
#endif
#ifndef NTT_W_FWD
#define NTT_W_FWD 4
#endif
#ifndef NTT_W_INV
#define NTT_W_INV 4
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


// The twiddles of one stage for one thread are D = 2^(W - b - 1) consecutive table
// entries starting at an even index (b: the stage's butterfly bit within the thread's
// words); pairs of (w, w') entries are fetched with one 256-bit load.
// L1 policy (NTT_L1_POLICY=1): the twiddles of the early stages (tables of at most
// NTT_TW_KEEP_LOG entries, shared by many threads and rows) are loaded evict-last, the
// large late-stage tables and the streamed row data no-allocate, so the rows streaming
// through an SM do not evict the twiddles every CTA keeps re-reading.
#ifndef NTT_L1_POLICY
#define NTT_L1_POLICY 1
#endif
#ifndef NTT_TW_KEEP_LOG
#define NTT_TW_KEEP_LOG 11
#endif
DEV void ldg_tw2(const ulonglong2 *p, ulonglong2 &a, ulonglong2 &b, bool keep) {
#if NTT_L1_POLICY
    if (keep)
        asm("ld.global.nc.L1::evict_last.v4.u64 {%0, %1, %2, %3}, [%4];"
            : "=l"(a.x), "=l"(a.y), "=l"(b.x), "=l"(b.y)
            : "l"(p));
    else
        asm("ld.global.nc.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
            : "=l"(a.x), "=l"(a.y), "=l"(b.x), "=l"(b.y)
            : "l"(p));
#else
    asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
        : "=l"(a.x), "=l"(a.y), "=l"(b.x), "=l"(b.y)
        : "l"(p));
#endif
}
DEV ulonglong2 ldg_tw1(const ulonglong2 *p, bool keep) {
#if NTT_L1_POLICY
    ulonglong2 a;
    if (keep) asm("ld.global.nc.L1::evict_last.v2.u64 {%0, %1}, [%2];" : "=l"(a.x), "=l"(a.y) : "l"(p));
    else asm("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(a.x), "=l"(a.y) : "l"(p));
    return a;
#else
    return __ldg(p);
#endif
}
// streamed row data (read once per row): no L1 allocation under the policy
DEV u64 ld_stream(const u64 *p) {
#if NTT_L1_POLICY
    u64 x;
    asm volatile("ld.global.L1::no_allocate.u64 %0, [%1];" : "=l"(x) : "l"(p));
    return x;
#else
    return *p;
#endif
}
// logt: log2 of the stage's twiddle-table length (the stage index)
template <int ND>
DEV void fetch_tw(ulonglong2 (&tw)[ND], const ulonglong2 *p, int D, int logt = 0) {
    const bool keep = logt <= NTT_TW_KEEP_LOG;
    if (D == 1) {
        tw[0] = ldg_tw1(p, keep);
    } else {
#pragma unroll
        for (int d = 0; d < ND; d += 2)
            if (d < D) ldg_tw2(p + d, tw[d], tw[d + 1], keep);
    }
}

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
// CANON = false: the outputs are left lazy; the return value is their bound in
// units of q (every output < bound * q <= 2^64), for callers that absorb it.
// OUT selects where the last pass leaves its results:
//   OUT_SMEM  shared memory, fenced by __syncthreads() (any thread may read any word);
//   OUT_REGS  the registers (no final store and barrier): v[e] = out[(tid << W) | e], E
//             consecutive words per thread (store_keep / load_keep below);
//   OUT_WARP  shared memory, fenced by __syncwarp() only: a warp's 32 E words are one
//             contiguous chunk written by that warp alone, so each warp reads back ITS chunk
//             (warp_chunk_base + k * 32 + lane: coalesced global accesses) without waiting
//             for the others -- the warps' epilogues and the next row's first pass overlap.
// PRESYNC (persistent callers of OUT_WARP): a barrier before the first shared-memory store
// of the row, so no warp is still reading its chunk of the previous row.
enum { OUT_SMEM = 0, OUT_REGS = 1, OUT_WARP = 2 };
template <int LOGN, int WW = DefaultW<LOGN>::value, bool CANON = true, int OUT = OUT_SMEM, bool PRESYNC = false>
DEV int ntt_fwd_core(u64 (&v)[NttCfg<LOGN, WW>::E], u64 *sm, const ModInfo &M, int tid) {
    using C = NttCfg<LOGN, WW>;
    constexpr int W = C::W, E = C::E, NP = C::NP;
    FwdLazy Lz(M);
#pragma unroll
    for (int p = 0; p < NP; p++) {
        const int s0 = p * W;
        const int f0 = (LOGN - s0 - W) > 0 ? (LOGN - s0 - W) : 0;
        const int k = (LOGN - s0) < W ? (LOGN - s0) : W;
        // The exchange into the last pass is warp-local: in pass NP-2 a warp writes exactly the
        // 32 E consecutive words it reads (and rewrites) in pass NP-1, so both of its fences
        // are warp barriers and the warps drift apart (one's exchange under another's
        // butterflies).  WL: the configuration has whole warps.
        constexpr bool WL = C::TH >= 32 && NP >= 2;
        if (p > 0) {
#pragma unroll
            for (int e = 0; e < E; e++) v[e] = sm[C::pad(fidx<W>(tid, e, f0))];
            if (WL && p == NP - 1) __syncwarp();
            else __syncthreads();
        }
#pragma unroll
        for (int ls = 0; ls < k; ls++) {
            const int s = s0 + ls;
            const int b = LOGN - s - 1 - f0;
            Lz.stage();
            if (Lz.red) {
#pragma unroll
                for (int e = 0; e < E; e++)
                    if (!(e & (1 << b))) v[e] = Lz.cred(v[e]);
            }
            ulonglong2 tw[E / 2];
#if NTT_EXP == 1      // timing experiment: no twiddle loads (results are garbage)
#pragma unroll
            for (int d = 0; d < E / 2; d++) tw[d] = make_ulonglong2(M.ninv + d, M.ninv_sh + s);
#else
            fetch_tw(tw, M.tw + (1u << s) + ((u32)fidx<W>(tid, 0, f0) >> (LOGN - s)), E >> (b + 1), s);
#endif
#pragma unroll
            for (int e = 0; e < E; e++) {
                if (e & (1 << b)) continue;
#if NTT_EXP == 2      // timing experiment: no butterfly arithmetic (results are garbage)
                v[e] ^= tw[e >> (b + 1)].x;
                v[e | (1 << b)] += tw[e >> (b + 1)].y;
#else
                Lz.bfly(v[e], v[e | (1 << b)], tw[e >> (b + 1)]);
#endif
            }
        }
        if (CANON && p == NP - 1) {
#pragma unroll
            for (int e = 0; e < E; e++) v[e] = red_any(v[e], M.q, M.mu, M.nq);
        }
        if (OUT == OUT_REGS && p == NP - 1) break;
        if (PRESYNC && p == 0) __syncthreads();
#pragma unroll
        for (int e = 0; e < E; e++) sm[C::pad(fidx<W>(tid, e, f0))] = v[e];
        if ((OUT == OUT_WARP && p == NP - 1 && NP > 1) || (WL && p == NP - 2)) __syncwarp();
        else __syncthreads();
    }
    return CANON ? 1 : Lz.B;
}
// first word of the chunk the thread's warp owns after an OUT_WARP transform
template <int W>
DEV int warp_chunk_base(int tid) { return (tid & ~31) << W; }
// E consecutive words of one thread to / from global memory with 32-byte accesses
// (p 32-byte aligned for E >= 4)
#ifndef NTT_STORE_VEC
#define NTT_STORE_VEC 4     // words per store of store_keep: 4 (32-byte stores, measured best) or 2 (16-byte)
#endif
template <int E>
DEV void store_keep(u64 *p, const u64 (&v)[E]) {
    if constexpr (E % 4 == 0 && NTT_STORE_VEC == 4) {
#pragma unroll
        for (int e = 0; e < E; e += 4)
            asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p + e), "l"(v[e]), "l"(v[e + 1]), "l"(v[e + 2]),
                         "l"(v[e + 3])
                         : "memory");
    } else if constexpr (E % 2 == 0) {
        // 16-byte stores: the two outputs of one last-stage butterfly, where the register
        // allocator can place them without staging moves
#pragma unroll
        for (int e = 0; e < E; e += 2) *reinterpret_cast<ulonglong2 *>(p + e) = make_ulonglong2(v[e], v[e + 1]);
    } else {
#pragma unroll
        for (int e = 0; e < E; e++) p[e] = v[e];
    }
}
template <int E>
DEV void load_keep(u64 (&v)[E], const u64 *p) {
    if constexpr (E % 4 == 0) {
#pragma unroll
        for (int e = 0; e < E; e += 4)
            asm("ld.global.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
                : "=l"(v[e]), "=l"(v[e + 1]), "=l"(v[e + 2]), "=l"(v[e + 3])
                : "l"(p + e));
    } else {
#pragma unroll
        for (int e = 0; e < E; e++) v[e] = p[e];
    }
}

// Inverse. In: canonical (or < 2q) values in sm[C::pad(i)], bit-reversed order, synced.
// Out: v[e] = a[(e << (LOGN-W)) | tid] canonical, scaled by n^-1.  Shared memory is
// free for reuse only after a __syncthreads() by the caller.
template <int LOGN, int WW = DefaultWInv<LOGN>::value>
DEV void ntt_inv_core(u64 (&v)[NttCfg<LOGN, WW>::E], u64 *sm, const ModInfo &M, int tid, u32 g_perm = 0) {
    using C = NttCfg<LOGN, WW>;
    constexpr int W = C::W, E = C::E, NP = C::NP, N = C::N;
    InvLazy Lz(M);
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
        // Mirror image of the forward core: passes 0 and 1 both work on the warp's own 32 E
        // consecutive words, so the fences around that exchange are warp barriers (pass 0's
        // only when it does not gather through an automorphism).
        constexpr bool WL = C::TH >= 32 && NP >= 3 && 2 * W <= LOGN;
        if (p < NP - 1) {
            if (WL && (p == 1 || (p == 0 && !g_perm))) __syncwarp();
            else __syncthreads();
        }
#pragma unroll
        for (int ls = 0; ls < k; ls++) {
            const int lt = lt0 + ls;
            const int b = lt - f0;
            const int h = N >> (lt + 1);
            Lz.stage();
            if (lt == LOGN - 1) {          // last stage: twiddle itw[1] for all, n^-1 folded in
#pragma unroll
                for (int e = 0; e < E; e++)
                    if (!(e & (1 << b))) Lz.last(v[e], v[e | (1 << b)], M);
                continue;
            }
            ulonglong2 tw[E / 2];
            fetch_tw(tw, M.itw + (u32)h + ((u32)fidx<W>(tid, 0, f0) >> (lt + 1)), E >> (b + 1), LOGN - 1 - lt);
#pragma unroll
            for (int e = 0; e < E; e++) {
                if (e & (1 << b)) continue;
                Lz.bfly(v[e], v[e | (1 << b)], tw[e >> (b + 1)]);
            }
            if (Lz.red) {
#pragma unroll
                for (int e = 0; e < E; e++)
                    if (!(e & (1 << b))) v[e] = Lz.cred(v[e]);
            }
        }
        if (p < NP - 1) {
#pragma unroll
            for (int e = 0; e < E; e++) sm[C::pad(fidx<W>(tid, e, f0))] = v[e];
            if (WL && p == 0) __syncwarp();
            else __syncthreads();
        }
    }
}


// ------------------------------------------------------------------------------
// Rows longer than one CTA's shared memory (n = 2^15, 2^16): one thread-block
// cluster of CR = n / 2^14 CTAs per row; CTA `rank` owns words
// [rank * 2^14, (rank + 1) * 2^14) in its shared memory (distributed shared memory,
// DSMEM).  Forward: the first W stages (the only ones whose butterflies span CTAs)
// run on each thread's own words straight from the global load, the results are
// stored into their owners' shared memory, and the remaining stages run per CTA
// as in the single-CTA core.  Inverse: mirror image (local passes, then one pass
// that reads its words from the owners' shared memory).  Same transform, order and
// twiddles as the single-CTA cores, so every ring size is bit-identical to the
// golden model.  For n <= 2^14 RowCfg is the single-CTA configuration (CR = 1).
#include <cooperative_groups.h>

#ifndef NTT_LOGL
#define NTT_LOGL 14      // rows up to 2^NTT_LOGL words run on one CTA
#endif
#ifndef NTT_LOGL_BIG
#define NTT_LOGL_BIG 14  // words per CTA of the cluster rows (n = 2^15, 2^16)
#endif
// WO != 0 overrides the radix of single-CTA rows, per kernel (FwdW5 for k_modup /
// k_ntt_rows, RescaleW for k_rescale: all radix-16 now, see the header comment)
template <int LOGN, bool INV, int WO = 0>
struct RowCfg {
    static constexpr int LOGL = LOGN > 14 ? NTT_LOGL_BIG : (LOGN > NTT_LOGL ? NTT_LOGL : LOGN);    // log2 words per CTA
    static constexpr int CL = LOGN - LOGL;                // log2 CTAs per row
    static constexpr int CR = 1 << CL;
#ifndef NTT_WO_CLUSTER
#define NTT_WO_CLUSTER 0   // 1: the radix override applies to cluster rows too
#endif
    using Loc = NttCfg<LOGL, (WO && (CL == 0 || NTT_WO_CLUSTER)) ? WO : (INV ? DefaultWInv<LOGL>::value : DefaultW<LOGL>::value)>;
    static constexpr int W = Loc::W, E = Loc::E, TH = Loc::TH, NL = Loc::N, N = 1 << LOGN;
    static constexpr int SMEM_WORDS = Loc::SMEM_WORDS;
    static_assert(CL <= 3 && CL <= W, "clusters of at most 8 CTAs");
    static DEV int pad(int i) { return Loc::pad(i); }
    static DEV int rank() {
        if constexpr (CL > 0) return (int)(blockIdx.x & (CR - 1));
        else return 0;
    }
    static DEV int row() { return (int)(blockIdx.x >> CL); }     // row index (blockIdx.x of the 1-CTA layout)
    static DEV int base() { return rank() << LOGL; }             // global index of local word 0
    // global element index of v[e] (forward input / inverse output)
    static DEV int io(int tid, int e) { return (e << (LOGN - W)) | (rank() * TH + tid); }
};

template <int LOGN, bool CANON = true, int WO = 0>
DEV int ntt_fwd_cluster(u64 (&v)[RowCfg<LOGN, false, WO>::E], u64 *sm, const ModInfo &M, int tid) {
    namespace cg = cooperative_groups;
    using R = RowCfg<LOGN, false, WO>;
    constexpr int W = R::W, E = R::E, LOGL = R::LOGL, CL = R::CL;
    FwdLazy Lz(M);
    const int rank = R::rank(), gtid = rank * R::TH + tid;
    cg::cluster_group cl = cg::this_cluster();
    // stages 0 .. W-1: the pair partner differs in bit W-1-s of e
#pragma unroll
    for (int s = 0; s < W; s++) {
        const int b = W - 1 - s;
        Lz.stage();
        if (Lz.red) {
#pragma unroll
            for (int e = 0; e < E; e++)
                if (!(e & (1 << b))) v[e] = Lz.cred(v[e]);
        }
        ulonglong2 tw[E / 2];
        fetch_tw(tw, M.tw + (1 << s), E >> (b + 1), s);
#pragma unroll
        for (int e = 0; e < E; e++) {
            if (e & (1 << b)) continue;
            Lz.bfly(v[e], v[e | (1 << b)], tw[e >> (b + 1)]);
        }
    }
    cl.sync();   // every CTA of the cluster is resident before remote stores
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int owner = e >> (W - CL);
        const int local = ((e & ((1 << (W - CL)) - 1)) << (LOGN - W)) | gtid;
        u64 *dst = cl.map_shared_rank(sm, owner);
        dst[R::pad(local)] = v[e];
    }
    cl.sync();
    // local stages: global stage s = sl + CL, sl = W - CL .. LOGL - 1
    constexpr int S0 = W - CL;
    constexpr int NP = (LOGL - S0 + W - 1) / W;
#pragma unroll
    for (int p = 0; p < NP; p++) {
        const int s0 = S0 + p * W;
        const int f0 = (LOGL - s0 - W) > 0 ? (LOGL - s0 - W) : 0;
        const int k = (LOGL - s0) < W ? (LOGL - s0) : W;
        // warp-local exchange into the last local pass, as in the single-CTA core
        constexpr bool WL = R::TH >= 32 && NP >= 2;
#pragma unroll
        for (int e = 0; e < E; e++) v[e] = sm[R::pad(fidx<W>(tid, e, f0))];
        if (WL && p == NP - 1) __syncwarp();
        else __syncthreads();
#pragma unroll
        for (int ls = 0; ls < k; ls++) {
            const int sl = s0 + ls;
            const int b = LOGL - sl - 1 - f0;
            Lz.stage();
            if (Lz.red) {
#pragma unroll
                for (int e = 0; e < E; e++)
                    if (!(e & (1 << b))) v[e] = Lz.cred(v[e]);
            }
            ulonglong2 tw[E / 2];
            fetch_tw(tw, M.tw + (1u << (sl + CL)) + ((u32)rank << sl) + ((u32)fidx<W>(tid, 0, f0) >> (LOGL - sl)),
                     E >> (b + 1), sl + CL);
#pragma unroll
            for (int e = 0; e < E; e++) {
                if (e & (1 << b)) continue;
                Lz.bfly(v[e], v[e | (1 << b)], tw[e >> (b + 1)]);
            }
        }
        if (CANON && p == NP - 1) {
#pragma unroll
            for (int e = 0; e < E; e++) v[e] = red_any(v[e], M.q, M.mu, M.nq);
        }
#pragma unroll
        for (int e = 0; e < E; e++) sm[R::pad(fidx<W>(tid, e, f0))] = v[e];
        if (WL && p == NP - 2) __syncwarp();
        else __syncthreads();
    }
    return CANON ? 1 : Lz.B;
}

// In: this CTA's words (global base() + x) canonical in sm[pad(x)], synced.
// Out: v[e] = a[R::io(tid, e)] canonical, scaled by n^-1; ends with a cluster barrier.
template <int LOGN>
DEV void ntt_inv_cluster(u64 (&v)[RowCfg<LOGN, true>::E], u64 *sm, const ModInfo &M, int tid) {
    namespace cg = cooperative_groups;
    using R = RowCfg<LOGN, true>;
    constexpr int W = R::W, E = R::E, LOGL = R::LOGL, CL = R::CL, N = R::N;
    InvLazy Lz(M);
    const int rank = R::rank(), gtid = rank * R::TH + tid;
    cg::cluster_group cl = cg::this_cluster();
    constexpr int LT = LOGL - W + CL;            // local stages lt = 0 .. LT-1
    constexpr int NP = (LT + W - 1) / W;
#pragma unroll
    for (int p = 0; p < NP; p++) {
        const int lt0 = p * W;
        const int k = (LT - lt0) < W ? (LT - lt0) : W;
        const int f0 = lt0 < LOGL - W ? lt0 : LOGL - W;
        // warp-local exchange between the first two local passes, as in the single-CTA core
        constexpr bool WL = R::TH >= 32 && NP >= 3 && 2 * W <= LOGL;
#pragma unroll
        for (int e = 0; e < E; e++) v[e] = sm[R::pad(fidx<W>(tid, e, f0))];
        if (WL && p <= 1) __syncwarp();
        else __syncthreads();
#pragma unroll
        for (int ls = 0; ls < k; ls++) {
            const int lt = lt0 + ls;
            const int b = lt - f0;
            Lz.stage();
            ulonglong2 tw[E / 2];
            fetch_tw(tw, M.itw + (u32)(N >> (lt + 1)) + ((u32)rank << (LOGL - lt - 1)) + ((u32)fidx<W>(tid, 0, f0) >> (lt + 1)),
                     E >> (b + 1), LOGN - 1 - lt);
#pragma unroll
            for (int e = 0; e < E; e++) {
                if (e & (1 << b)) continue;
                Lz.bfly(v[e], v[e | (1 << b)], tw[e >> (b + 1)]);
            }
            if (Lz.red) {
#pragma unroll
                for (int e = 0; e < E; e++)
                    if (!(e & (1 << b))) v[e] = Lz.cred(v[e]);
            }
        }
#pragma unroll
        for (int e = 0; e < E; e++) sm[R::pad(fidx<W>(tid, e, f0))] = v[e];
        if (WL && p == 0) __syncwarp();
        else __syncthreads();
    }
    cl.sync();   // all local stages of the row are done
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int owner = e >> (W - CL);
        const int local = ((e & ((1 << (W - CL)) - 1)) << (LOGN - W)) | gtid;
        const u64 *src = cl.map_shared_rank(sm, owner);
        v[e] = src[R::pad(local)];
    }
    // stages lt = LOGN - W + b: the pair partner differs in bit b of e
#pragma unroll
    for (int b = 0; b < W; b++) {
        const int lt = LOGN - W + b;
        Lz.stage();
        if (lt == LOGN - 1) {              // last stage: n^-1 folded in
#pragma unroll
            for (int e = 0; e < E; e++)
                if (!(e & (1 << b))) Lz.last(v[e], v[e | (1 << b)], M);
            continue;
        }
        ulonglong2 tw[E / 2];
        fetch_tw(tw, M.itw + (N >> (lt + 1)), E >> (b + 1), LOGN - 1 - lt);
#pragma unroll
        for (int e = 0; e < E; e++) {
            if (e & (1 << b)) continue;
            Lz.bfly(v[e], v[e | (1 << b)], tw[e >> (b + 1)]);
        }
        if (Lz.red) {
#pragma unroll
            for (int e = 0; e < E; e++)
                if (!(e & (1 << b))) v[e] = Lz.cred(v[e]);
        }
    }
    cl.sync();   // no CTA leaves or reuses its shared memory while another reads it
}

// Row-size dispatch used by the row kernels.
template <int LOGN, bool CANON = true, int WO = 0>
DEV int ntt_fwd_row(u64 (&v)[RowCfg<LOGN, false, WO>::E], u64 *sm, const ModInfo &M, int tid) {
    if constexpr (RowCfg<LOGN, false, WO>::CL == 0)
        return ntt_fwd_core<LOGN, RowCfg<LOGN, false, WO>::W, CANON>(v, sm, M, tid);
    else return ntt_fwd_cluster<LOGN, CANON, WO>(v, sm, M, tid);
}
#ifndef NTT_W_FUSED_FWD
#define NTT_W_FUSED_FWD 4
#endif
template <int LOGN>
struct FwdW5 {       // radix override for k_modup / k_ntt_rows
    static constexpr int value = LOGN >= 12 ? NTT_W_FUSED_FWD : 0;
};
template <int LOGN>
DEV void ntt_inv_row(u64 (&v)[RowCfg<LOGN, true>::E], u64 *sm, const ModInfo &M, int tid) {
    if constexpr (RowCfg<LOGN, true>::CL == 0) ntt_inv_core<LOGN>(v, sm, M, tid);
    else ntt_inv_cluster<LOGN>(v, sm, M, tid);
}
