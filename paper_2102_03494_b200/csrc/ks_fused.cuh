// ks_fused.cuh -- key switching with ModUp fused into the key inner product,
// accumulators in Tensor Memory (TMEM).
//
// Hybrid key switching (one prime per digit, one special prime P) needs, for every
// output prime i of a ciphertext, acc_p[i] = sum_j NTT_i(lift_i(digit_j)) * key_p[j][i]
// (p = 0, 1).  The unfused path writes every extended digit NTT_i(lift_i(digit_j))
// to HBM (k_modup: l^2 rows per ciphertext) and reads it back (k_ks_inner,
// k_ks_special).  Here one CTA owns one (ciphertext, output prime) pair and walks the
// digits: it lifts digit j into prime i, transforms it in shared memory and
// multiply-accumulates it with both key halves straight out of shared memory.  The
// two accumulator rows (2 x n words = 256 KB at n = 2^14) do not fit in registers
// or shared memory next to the NTT's working set, so they live in TMEM -- the 256 KB
// per-SM tensor memory that tcgen05 MMAs accumulate into, used here as the
// accumulator store of a modular inner product (tcgen05.ld / tcgen05.st, 32x32b
// shape: each thread owns one TMEM lane and 4 columns per coefficient it handles).
// The extended digits never reach HBM.
//
// CTA work (l q primes + the special prime per ciphertext):
//   output prime i < l : l - 1 forward NTTs (digit j = i is the ciphertext's own NTT-form
//                        limb, read through the rotation's automorphism), then the
//                        key-switch addends are folded in as
//                        y * (P mod q_i) and acc_p[i] is stored (NTT form)
//   special prime      : l forward NTTs; both accumulators are stored (NTT form) and a
//                        k_intt_rows launch takes them to coefficient form for the
//                        ModDown rescale
// Blocks 0 .. S-1 are the (slightly heavier) special-prime items, so the hardware's
// in-order block dispatch schedules them first.
//
// Arithmetic: acc <- acc + Mont(x, key) mod q with x the lazy NTT output (< 2^64) and
// key < q in Montgomery form, i.e. canonical partial sums of x * key * 2^-64; the sum
// equals the unfused path's single Montgomery reduction of the 128-bit sum, so the
// words are bit-identical to the golden model.
#pragma once
#include "kernels.cuh"

// ------------------------------------------------------------------ TMEM helpers
DEV u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }

DEV void tmem_alloc(u32 *slot, u32 ncols) {           // one full warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
DEV void tmem_dealloc(u32 taddr, u32 ncols) {         // the allocating warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
DEV void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DEV void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 16 consecutive 32-bit columns of this thread's lane
DEV void tmem_ld16(u32 ta, u32 (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
        "[%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(ta)
        : "memory");
}
DEV void tmem_st16(u32 ta, const u32 (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16};" ::"r"(ta),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

// 8 consecutive 32-bit columns (two accumulator pairs)
DEV void tmem_ld8(u32 ta, u32 (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta)
                 : "memory");
}
DEV void tmem_st8(u32 ta, const u32 (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(ta), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
template <int CH>
DEV void tmem_ld(u32 ta, u32 (&r)[4 * CH]) {
    if constexpr (CH == 4) tmem_ld16(ta, r);
    else tmem_ld8(ta, r);
}
template <int CH>
DEV void tmem_st(u32 ta, const u32 (&r)[4 * CH]) {
    if constexpr (CH == 4) tmem_st16(ta, r);
    else tmem_st8(ta, r);
}

// Row configuration of the fused kernel: the ModUp rows' configuration (radix-32
// single-CTA rows from 2^12, radix-16 thread-block-cluster rows for 2^15 / 2^16, where
// every CTA owns 2^14 words and keeps their accumulators in its own TMEM); at least one
// full warp (tcgen05.ld/st are warp-collective).
template <int LOGN>
struct KsfCfg {
    static_assert(LOGN >= 9 && LOGN <= 16, "fused key switching: rows of 2^9 .. 2^16 words");
    static constexpr int WO = FwdW5<LOGN>::value;
    using C = RowCfg<LOGN, false, WO>;
    static constexpr int E = C::E, TH = C::TH, N = C::N, NL = C::NL, W = C::W;
    static constexpr int WARPS = TH / 32;
    static constexpr int COLS_PER_THREAD = 4 * E;                       // two u64 accumulators per word
    static constexpr int BLOCKS = (WARPS + 3) / 4;                      // column blocks (warps sharing a lane quarter)
    static constexpr int NEED = COLS_PER_THREAD * BLOCKS;
    static constexpr u32 NCOLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
    static_assert(NEED <= 512, "accumulators exceed TMEM");
    // words per TMEM access: 4 (16 columns) with 128 registers per thread, 2 (8 columns)
    // with 64 (the 1024-thread radix-16 rows)
    static constexpr int CH = TH <= 512 ? 4 : 2;
    static_assert(E % CH == 0, "TMEM accesses move CH words at a time");
    static_assert(TH >= 32, "at least one full warp");
};

// acc_p += Mont(x_e, key_p[j][i]) for this thread's words x = tid + e TH.  DIAG: the
// digit is the input's own NTT-form limb (read through X -> X^dperm), else the
// transformed digit in shared memory.  FIRST: the accumulators start here.
template <int LOGN, bool DIAG>
DEV void ksf_mac(u32 tbase, bool first, const u64 *sm, const u64 *dg, u32 dperm, const u64 *k0, const u64 *k1,
                 u64 q, u64 qinv, int tid) {
    using F = KsfCfg<LOGN>;
    using C = typename F::C;
    constexpr int E = F::E, TH = F::TH, CH = F::CH;
    // rolled over the CH-word chunks (the kernel's code must stay within the instruction
    // cache next to the unrolled NTT passes); the chunk's key words are loaded before
    // its TMEM accumulators so both latencies overlap
#pragma unroll 1
    for (int c = 0; c < E / CH; c++) {
        u64 xv[CH], kv0[CH], kv1[CH];
#pragma unroll
        for (int k = 0; k < CH; k++) {
            const int x = tid + (CH * c + k) * TH;                  // local word
            const u32 gx = (u32)(C::base() + x);                      // word of the row
            kv0[k] = __ldg(k0 + gx);
            kv1[k] = __ldg(k1 + gx);
            xv[k] = DIAG ? dg[dperm ? galois_perm(gx, dperm, LOGN) : gx] : sm[C::pad(x)];
        }
        u32 r[4 * CH];
        if (!first) tmem_ld<CH>(tbase + 4 * CH * c, r);
        u64 p0[CH], p1[CH];
#pragma unroll
        for (int k = 0; k < CH; k++) {
            p0[k] = mont(xv[k], kv0[k], q, qinv);
            p1[k] = mont(xv[k], kv1[k], q, qinv);
        }
        if (!first) {
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < CH; k++) {
                p0[k] = addm(((u64)r[4 * k + 1] << 32) | r[4 * k], p0[k], q);
                p1[k] = addm(((u64)r[4 * k + 3] << 32) | r[4 * k + 2], p1[k], q);
            }
        }
#pragma unroll
        for (int k = 0; k < CH; k++) {
            r[4 * k] = (u32)p0[k];
            r[4 * k + 1] = (u32)(p0[k] >> 32);
            r[4 * k + 2] = (u32)p1[k];
            r[4 * k + 3] = (u32)(p1[k] >> 32);
        }
        tmem_st<CH>(tbase + 4 * CH * c, r);
    }
    tmem_wait_st();
}

// per-item operands, kept in shared memory: the radix-32 transform needs the whole
// register budget (512 threads x 128), so nothing else stays live across it
struct KsfItem {
    const u64 *coef, *key, *dg;
    u32 dperm, tslot;
    int s, i;
};

template <int LOGN>
__global__ void __launch_bounds__(KsfCfg<LOGN>::TH, 1)
    k_ks_fused(const DigitTab dt, u64 *__restrict__ Acc, int S, int l, int L, int special_id,
               const ModInfo *__restrict__ mods, const KsAdd ka) {
    using F = KsfCfg<LOGN>;
    using C = typename F::C;
    constexpr int E = F::E, TH = F::TH, CH = F::CH;
    constexpr u32 n = F::N;
    extern __shared__ u64 sm[];
    __shared__ KsfItem it;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) {
        // item: blocks [0, S) are the special-prime rows, then (s, i) for the q primes
        const int b = C::row();
        const int s = b < S ? b : (b - S) / l, i = b < S ? l : (b - S) % l;
        it.s = s;
        it.i = i;
        it.coef = dt.coef[s];
        it.key = dt.key[s];
        it.dg = dt.ntt[s] + (u32)i * n;
        it.dperm = dt.dperm[s];
    }
    if (warp == 0) tmem_alloc(&it.tslot, F::NCOLS);
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const int i = it.i;
    const bool special = i == l;
    const u32 kstride = 2u * (L + 1) * n;                 // digit j -> j + 1
    const u32 kpair = (u32)(L + 1) * n;                    // key half 0 -> 1
    auto tb = [&]() { return it.tslot + ((u32)((warp & 3) * 32) << 16) + (u32)((warp >> 2) * F::COLS_PER_THREAD); };
    // the prime's row in the key layout
    auto krow = [&](int j) { return it.key + (u32)j * kstride + (special ? (u32)L : (u32)i) * n; };

    if (!special) {
        const ModInfo &Mq = mods[i];
        ksf_mac<LOGN, true>(tb(), true, sm, it.dg, it.dperm, krow(i), krow(i) + kpair, Mq.q, Mq.qinv, tid);
    }
#pragma unroll 1
    for (int j = 0; j < l; j++) {
        if (j == it.i) continue;
        {
            const ModInfo M = mods[special ? special_id : i];
            const ModInfo &Sj = mods[j];
            const u64 half_j = Sj.half, qj_mod = red64(Sj.q, M.q, M.mu);
            const u64 *src = it.coef + (u32)j * n;
            u64 v[E];
#pragma unroll
            for (int e = 0; e < E; e++) v[e] = centered_lift_lazy(src[C::io(tid, e)], half_j, qj_mod, M);
            ntt_fwd_row<LOGN, false, F::WO>(v, sm, M, tid);   // ends with __syncthreads
        }
        const ModInfo &Mq = mods[it.i == l ? special_id : it.i];
        const u64 *k0 = krow(j);
        ksf_mac<LOGN, false>(tb(), special && j == 0, sm, nullptr, 0, k0, k0 + kpair, Mq.q, Mq.qinv, tid);
        __syncthreads();                                  // the next transform reuses shared memory
    }
    const int s = it.s;
    const ModInfo M = mods[special ? special_id : i];
    const u64 q = M.q, qinv = M.qinv;
    const u32 tbase = tb();

    if (!special) {
        // key-switch addends folded in: ModDown(acc + P y) = ModDown(acc) + y exactly
        const u64 pr = ka.pr[i];
        const u64 *ad = ka.add[s];
        const u64 *ac = ka.acc[s];
        const u32 ag = ka.add_g[s];
        const int pmask = ka.add_pmask;
        const long long aps = ka.add_pstride, cps = ka.acc_pstride;
        u64 *o0 = Acc + ((u32)s * 2 * (l + 1) + (u32)i) * n;
        u64 *o1 = o0 + (u32)(l + 1) * n;
#pragma unroll 1
        for (int c = 0; c < E / CH; c++) {
            u32 r[4 * CH];
            tmem_ld<CH>(tbase + 4 * CH * c, r);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < CH; k++) {
                const u32 x = (u32)(C::base() + tid + (CH * c + k) * TH);
                u64 a0 = ((u64)r[4 * k + 1] << 32) | r[4 * k], a1 = ((u64)r[4 * k + 3] << 32) | r[4 * k + 2];
                if (ad) {
                    const u32 xa = ag ? galois_perm(x, ag, LOGN) : x;
                    if (pmask & 1) a0 = addm(a0, mont(ad[(u32)i * n + xa], pr, q, qinv), q);
                    if (pmask & 2) a1 = addm(a1, mont(ad[aps + (u32)i * n + xa], pr, q, qinv), q);
                }
                if (ac) {
                    a0 = addm(a0, mont(ac[(u32)i * n + x], pr, q, qinv), q);
                    a1 = addm(a1, mont(ac[cps + (u32)i * n + x], pr, q, qinv), q);
                }
                o0[x] = a0;
                o1[x] = a1;
            }
        }
    } else {
        // special prime: both accumulators (NTT form) for the inverse transform that
        // precedes the ModDown rescale (a radix-16 k_intt_rows launch: the radix-32
        // inverse core does not fit this kernel's register budget)
        u64 *o0 = Acc + ((u32)s * 2 * (l + 1) + (u32)l) * n;
        u64 *o1 = o0 + (u32)(l + 1) * n;
#pragma unroll 1
        for (int c = 0; c < E / CH; c++) {
            u32 r[4 * CH];
            tmem_ld<CH>(tbase + 4 * CH * c, r);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < CH; k++) {
                const u32 x = (u32)(C::base() + tid + (CH * c + k) * TH);
                o0[x] = ((u64)r[4 * k + 1] << 32) | r[4 * k];
                o1[x] = ((u64)r[4 * k + 3] << 32) | r[4 * k + 2];
            }
        }
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(it.tslot, F::NCOLS);
}
