// ntt4.cuh -- two-kernel ("four-step") negacyclic NTT for large rings.
//
// n = 2^LOGN = 2^LA * 2^LB.  Index j = hi * 2^LB + lo.  The Cooley-Tukey stages
// s < LA touch only the hi bits ("columns": fixed lo), stages s >= LA only the lo
// bits ("rows": fixed hi).  Kernel A runs the column stages for 16 adjacent
// columns per CTA, kernel B the row stages for 16 adjacent rows per CTA; each
// thread owns 8 words (radix-8 register passes, smem exchange within the CTA).
// The Gentleman-Sande inverse runs the row stages first, then the columns.
// Exactly the same butterflies, twiddles, lazy ranges and output ordering as the
// single-CTA cores (ntt_core.cuh), so the results are bit-identical; what changes
// is the shape of the work: 256-thread CTAs with 16-32 KB of shared memory, many
// resident per SM, and no row-size limit (n = 2^15, 2^16 rows do not fit one CTA).
#pragma once
#include "ntt_core.cuh"

template <int LOGN>
struct Ntt4Cfg {
    static constexpr int LA = (LOGN + 1) / 2;          // column (hi) stages
    static constexpr int LB = LOGN - LA;               // row (lo) stages
    static constexpr int N = 1 << LOGN;
    static constexpr int C = 16;                       // columns / rows per CTA
    static constexpr int TA = (1 << LA) / 8;           // threads per column
    static constexpr int TB = (1 << LB) / 8;           // threads per row
    static constexpr int THA = C * TA, THB = C * TB;
    static constexpr int CTAS_PER_ROW_A = (1 << LB) / C;
    static constexpr int CTAS_PER_ROW_B = (1 << LA) / C;
};

// local index of element e (3 bits) in a sub-NTT of 2^M points for a pass whose
// 3-bit field starts at bit f0; tau = thread within the sub-NTT
DEV int lidx(int tau, int e, int f0) {
    int lo = tau & ((1 << f0) - 1), hi = tau >> f0;
    return (hi << (f0 + 3)) | (e << f0) | lo;
}
DEV int pad4(int i) { return i + (i >> 4); }

// ------------------------------------------------------------------ forward
// Column stages s in [0, LA): element (u = hi, col).  v[] in: loaded for pass 0,
// v[e] = x[(e << (LA-3)) | tau]; out: lazy values in [0, 4q) for local index
// lidx(tau, e, 0) of the last pass.  Twiddles are shared by every column and are
// staged once per CTA in shared memory (tws).
template <int M>
DEV void sub_fwd_cols(u64 (&v)[8], u64 *sm, const ulonglong2 *tws, int tau, int col, int C, u64 q) {
    constexpr int NP = (M + 2) / 3;
    const u64 q2 = 2 * q;
#pragma unroll
    for (int p = 0; p < NP; p++) {
        const int s0 = 3 * p;
        const int f0 = (M - s0 - 3) > 0 ? (M - s0 - 3) : 0;
        const int k = (M - s0) < 3 ? (M - s0) : 3;
        if (p > 0) {
#pragma unroll
            for (int e = 0; e < 8; e++) v[e] = sm[pad4(lidx(tau, e, f0) * C + col)];
            __syncthreads();
        }
#pragma unroll
        for (int ls = 0; ls < k; ls++) {
            const int s = s0 + ls;
            const int b = M - s - 1 - f0;
#pragma unroll
            for (int e = 0; e < 8; e++) {
                if (e & (1 << b)) continue;
                const int e2 = e | (1 << b);
                const ulonglong2 tw = tws[(1 << s) + (lidx(tau, e, f0) >> (M - s))];
                u64 U = v[e];
                U = U >= q2 ? U - q2 : U;
                const u64 V = shoup_lazy(v[e2], tw.x, tw.y, q);
                v[e] = U + V;
                v[e2] = U - V + q2;
            }
        }
        if (p < NP - 1) {
#pragma unroll
            for (int e = 0; e < 8; e++) sm[pad4(lidx(tau, e, f0) * C + col)] = v[e];
            __syncthreads();
        }
    }
}

// Row stages s in [LA, LOGN) for row `hi`: local index u = lo bits.
template <int LOGN, int M>
DEV void sub_fwd_rows(u64 (&v)[8], u64 *sm, const ulonglong2 *tw, int tau, int row, int hi, u64 q) {
    constexpr int NP = (M + 2) / 3;
    constexpr int LA = LOGN - M;
    constexpr int RS = (1 << M) + ((1 << M) >> 4);     // padded row stride in shared memory
    const u64 q2 = 2 * q;
#pragma unroll
    for (int p = 0; p < NP; p++) {
        const int s0 = 3 * p;
        const int f0 = (M - s0 - 3) > 0 ? (M - s0 - 3) : 0;
        const int k = (M - s0) < 3 ? (M - s0) : 3;
        if (p > 0) {
#pragma unroll
            for (int e = 0; e < 8; e++) v[e] = sm[row * RS + pad4(lidx(tau, e, f0))];
            __syncthreads();
        }
#pragma unroll
        for (int ls = 0; ls < k; ls++) {
            const int sl = s0 + ls;                       // local stage
            const int s = LA + sl;                        // global stage
            const int b = M - sl - 1 - f0;
#pragma unroll
            for (int e = 0; e < 8; e++) {
                if (e & (1 << b)) continue;
                const int e2 = e | (1 << b);
                const u32 g = (1u << s) + ((u32)hi << sl) + ((u32)lidx(tau, e, f0) >> (M - sl));
                const ulonglong2 t = __ldg(tw + g);
                u64 U = v[e];
                U = U >= q2 ? U - q2 : U;
                const u64 V = shoup_lazy(v[e2], t.x, t.y, q);
                v[e] = U + V;
                v[e2] = U - V + q2;
            }
        }
        if (p < NP - 1) {
#pragma unroll
            for (int e = 0; e < 8; e++) sm[row * RS + pad4(lidx(tau, e, f0))] = v[e];
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------------ inverse
// Row stages first: log2 t = lt in [0, LB) (bit lt of lo), input bit-reversed
// order values < 2q; out: v[e] for local index lidx(tau, e, f0_last) in [0, 2q).
template <int LOGN, int M>
DEV void sub_inv_rows(u64 (&v)[8], u64 *sm, const ulonglong2 *itw, int tau, int row, int hi, u64 q) {
    constexpr int NP = (M + 2) / 3;
    constexpr int RS = (1 << M) + ((1 << M) >> 4);
    constexpr int N = 1 << LOGN;
    const u64 q2 = 2 * q;
#pragma unroll
    for (int p = 0; p < NP; p++) {
        const int lt0 = 3 * p;
        const int f0 = (lt0 + 3) <= M ? lt0 : M - 3;
        const int k = (M - lt0) < 3 ? (M - lt0) : 3;
        if (p > 0) {
#pragma unroll
            for (int e = 0; e < 8; e++) v[e] = sm[row * RS + pad4(lidx(tau, e, f0))];
            __syncthreads();
        }
#pragma unroll
        for (int ls = 0; ls < k; ls++) {
            const int lt = lt0 + ls;
            const int b = lt - f0;
            const u32 h = (u32)(N >> (lt + 1));
#pragma unroll
            for (int e = 0; e < 8; e++) {
                if (e & (1 << b)) continue;
                const int e2 = e | (1 << b);
                // j >> (lt+1) = (hi << (M - lt - 1)) | (u >> (lt + 1))
                const u32 g = h + ((u32)hi << (M - lt - 1)) + ((u32)lidx(tau, e, f0) >> (lt + 1));
                const ulonglong2 t = __ldg(itw + g);
                const u64 U = v[e], V = v[e2];
                const u64 sum = U + V;
                v[e] = sum >= q2 ? sum - q2 : sum;
                v[e2] = shoup_lazy(U - V + q2, t.x, t.y, q);
            }
        }
        if (p < NP - 1) {
#pragma unroll
            for (int e = 0; e < 8; e++) sm[row * RS + pad4(lidx(tau, e, f0))] = v[e];
            __syncthreads();
        }
    }
}

// Column stages last: lt in [LB, LOGN), bit (lt - LB) of u = hi.  Twiddles shared
// by every column (tws = itw + 1 ... staged per CTA, indexed by h + (u >> (lt+1-LB))).
template <int LOGN, int M>
DEV void sub_inv_cols(u64 (&v)[8], u64 *sm, const ulonglong2 *tws, int tau, int col, int C, u64 q) {
    constexpr int NP = (M + 2) / 3;
    const u64 q2 = 2 * q;
#pragma unroll
    for (int p = 0; p < NP; p++) {
        const int lt0 = 3 * p;                            // local log2 t
        const int f0 = (lt0 + 3) <= M ? lt0 : M - 3;
        const int k = (M - lt0) < 3 ? (M - lt0) : 3;
        if (p > 0) {
#pragma unroll
            for (int e = 0; e < 8; e++) v[e] = sm[pad4(lidx(tau, e, f0) * C + col)];
            __syncthreads();
        }
#pragma unroll
        for (int ls = 0; ls < k; ls++) {
            const int lt = lt0 + ls;
            const int b = lt - f0;
            const int h = (1 << M) >> (lt + 1);            // global h = N >> (LB + lt + 1) = 2^(M - lt - 1)
#pragma unroll
            for (int e = 0; e < 8; e++) {
                if (e & (1 << b)) continue;
                const int e2 = e | (1 << b);
                const ulonglong2 t = tws[h + (lidx(tau, e, f0) >> (lt + 1))];
                const u64 U = v[e], V = v[e2];
                const u64 sum = U + V;
                v[e] = sum >= q2 ? sum - q2 : sum;
                v[e2] = shoup_lazy(U - V + q2, t.x, t.y, q);
            }
        }
        if (p < NP - 1) {
#pragma unroll
            for (int e = 0; e < 8; e++) sm[pad4(lidx(tau, e, f0) * C + col)] = v[e];
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------- bench kernels
// Row r of `rows` polynomials; plain load / store, used by fhe_bench_ntt (W = 100).
template <int LOGN>
__global__ void __launch_bounds__(Ntt4Cfg<LOGN>::THA) k4_fwd_cols(const u64 *in, u64 *tmp, const ModInfo *mods,
                                                               int mid) {
    using C4 = Ntt4Cfg<LOGN>;
    constexpr int LA = C4::LA, LB = C4::LB, C = C4::C;
    __shared__ u64 sm[C * (1 << LA) + (C * (1 << LA) >> 4) + 1];
    __shared__ ulonglong2 tws[1 << LA];
    const int r = blockIdx.x / C4::CTAS_PER_ROW_A, cb = blockIdx.x % C4::CTAS_PER_ROW_A;
    const int col = threadIdx.x % C, tau = threadIdx.x / C;
    const ModInfo &M = mods[mid];
    for (int i = threadIdx.x; i < (1 << LA); i += blockDim.x) tws[i] = M.tw[i];
    const u64 *src = in + (long long)r * C4::N + cb * C + col;
    u64 v[8];
#pragma unroll
    for (int e = 0; e < 8; e++) v[e] = src[(long long)((e << (LA - 3)) | tau) << LB];
    __syncthreads();
    sub_fwd_cols<LA>(v, sm, tws, tau, col, C, M.q);
    u64 *dst = tmp + (long long)r * C4::N + cb * C + col;
    const int f0 = 0;
#pragma unroll
    for (int e = 0; e < 8; e++) dst[(long long)lidx(tau, e, f0) << LB] = v[e];
}

template <int LOGN>
__global__ void __launch_bounds__(Ntt4Cfg<LOGN>::THB) k4_fwd_rows(const u64 *tmp, u64 *out, const ModInfo *mods,
                                                               int mid) {
    using C4 = Ntt4Cfg<LOGN>;
    constexpr int LB = C4::LB, C = C4::C;
    constexpr int RS = (1 << LB) + ((1 << LB) >> 4);
    __shared__ u64 sm[C * RS];
    const int r = blockIdx.x / C4::CTAS_PER_ROW_B, hb = blockIdx.x % C4::CTAS_PER_ROW_B;
    const int row = threadIdx.x / C4::TB, tau = threadIdx.x % C4::TB;
    const int hi = hb * C + row;
    const ModInfo &M = mods[mid];
    const u64 *src = tmp + (long long)r * C4::N + ((long long)hi << LB);
    u64 v[8];
#pragma unroll
    for (int e = 0; e < 8; e++) v[e] = src[(e << (LB - 3)) | tau];
    sub_fwd_rows<LOGN, LB>(v, sm, M.tw, tau, row, hi, M.q);
    const u64 q = M.q, q2 = 2 * q;
    u64 *dst = out + (long long)r * C4::N + ((long long)hi << LB);
#pragma unroll
    for (int e = 0; e < 8; e++) {
        u64 x = v[e];
        x = x >= q2 ? x - q2 : x;
        dst[lidx(tau, e, 0)] = x >= q ? x - q : x;
    }
}

template <int LOGN>
__global__ void __launch_bounds__(Ntt4Cfg<LOGN>::THB) k4_inv_rows(const u64 *in, u64 *tmp, const ModInfo *mods,
                                                               int mid) {
    using C4 = Ntt4Cfg<LOGN>;
    constexpr int LB = C4::LB, C = C4::C;
    constexpr int RS = (1 << LB) + ((1 << LB) >> 4);
    __shared__ u64 sm[C * RS];
    const int r = blockIdx.x / C4::CTAS_PER_ROW_B, hb = blockIdx.x % C4::CTAS_PER_ROW_B;
    const int row = threadIdx.x / C4::TB, tau = threadIdx.x % C4::TB;
    const int hi = hb * C + row;
    const ModInfo &M = mods[mid];
    const u64 *src = in + (long long)r * C4::N + ((long long)hi << LB);
    u64 v[8];
#pragma unroll
    for (int e = 0; e < 8; e++) v[e] = src[lidx(tau, e, 0)];
    sub_inv_rows<LOGN, LB>(v, sm, M.itw, tau, row, hi, M.q);
    u64 *dst = tmp + (long long)r * C4::N + ((long long)hi << LB);
    const int fl = (LB - 3);
#pragma unroll
    for (int e = 0; e < 8; e++) dst[lidx(tau, e, fl)] = v[e];
}

template <int LOGN>
__global__ void __launch_bounds__(Ntt4Cfg<LOGN>::THA) k4_inv_cols(const u64 *tmp, u64 *out, const ModInfo *mods,
                                                               int mid) {
    using C4 = Ntt4Cfg<LOGN>;
    constexpr int LA = C4::LA, LB = C4::LB, C = C4::C;
    __shared__ u64 sm[C * (1 << LA) + (C * (1 << LA) >> 4) + 1];
    __shared__ ulonglong2 tws[1 << LA];
    const int r = blockIdx.x / C4::CTAS_PER_ROW_A, cb = blockIdx.x % C4::CTAS_PER_ROW_A;
    const int col = threadIdx.x % C, tau = threadIdx.x / C;
    const ModInfo &M = mods[mid];
    for (int i = threadIdx.x; i < (1 << LA); i += blockDim.x) tws[i] = M.itw[i];   // h < 2^LA
    const u64 *src = tmp + (long long)r * C4::N + cb * C + col;
    u64 v[8];
#pragma unroll
    for (int e = 0; e < 8; e++) v[e] = src[(long long)lidx(tau, e, 0) << LB];
    __syncthreads();
    sub_inv_cols<LOGN, LA>(v, sm, tws, tau, col, C, M.q);
    u64 *dst = out + (long long)r * C4::N + cb * C + col;
    const int fl = LA - 3;
#pragma unroll
    for (int e = 0; e < 8; e++)
        dst[(long long)lidx(tau, e, fl) << LB] = shoup(v[e], M.ninv, M.ninv_sh, M.q);
}

