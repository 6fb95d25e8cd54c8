// ffconv_he.cu -- host side of the sm_100a packed RNS-BFV evaluator: context,
// tables, memory, and the C ABI of include/ffconv_he.h.
//
// One context = one CUDA stream; every entry point enqueues asynchronously except
// read/decrypt/sync, which block.  Ciphertexts live in stream-ordered pool
// allocations, limb-major [T*R][2][level][n] uint64 in the NTT domain.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "ffconv_he.h"
#include "kernels.cuh"
#include "ks_fused.cuh"

// =================================================================== errors
static thread_local char g_err[512];
static int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}
#define CU(call)                                                                             \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(FHE_EDEVICE, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                 \
    } while (0)
#define CHECK_LAUNCH() CU(cudaGetLastError())
#define TRY(x)                  \
    do {                        \
        int rc_ = (x);          \
        if (rc_) return rc_;    \
    } while (0)

extern "C" const char *fhe_last_error(void) { return g_err; }
extern "C" const char *fhe_backend_name(void) { return "cuda-sm100a"; }

// ============================================================ host arithmetic
namespace hm {
static u64 mul(u64 a, u64 b, u64 m) { return (u64)((u128)a * b % m); }
static u64 pw(u64 a, u64 e, u64 m) {
    u64 r = 1 % m;
    a %= m;
    while (e) {
        if (e & 1) r = mul(r, a, m);
        a = mul(a, a, m);
        e >>= 1;
    }
    return r;
}
static u64 inv(u64 a, u64 m) { return pw(a % m, m - 2, m); }
static u64 neg(u64 a, u64 m) { return a % m ? m - a % m : 0; }
static u64 shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
static u64 mont(u64 x, u64 q) { return (u64)(((u128)(x % q) << 64) % q); }
static void frac128(u64 r, u64 m, u64 &hi, u64 &lo) {   // floor(r 2^128 / m), r < m
    u128 num = (u128)r << 64;
    hi = (u64)(num / m);
    u64 rem = (u64)(num % m);
    lo = (u64)(((u128)rem << 64) / m);
}
static int is_prime(u64 n) {
    static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (u64 b : bases) {
        if (n == b) return 1;
        if (n % b == 0) return 0;
    }
    u64 d = n - 1;
    int s = 0;
    while (!(d & 1)) { d >>= 1; s++; }
    for (u64 b : bases) {
        u64 x = pw(b, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s; r++) {
            x = mul(x, x, n);
            if (x == n - 1) { comp = false; break; }
        }
        if (comp) return 0;
    }
    return 1;
}
static u32 brev(u32 x, u32 bits) {
    u32 r = 0;
    for (u32 i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}
static u64 min_root(u64 q, u32 n) {      // minimal primitive 2n-th root of unity
    u64 two_n = 2ull * n, psi0 = 0;
    for (u64 h = 2; h < q; h++) {
        u64 c = pw(h, (q - 1) / two_n, q);
        if (pw(c, n, q) == q - 1) { psi0 = c; break; }
    }
    u64 sq = mul(psi0, psi0, q), cur = psi0, best = psi0;
    for (u32 k = 0; k < n; k++) {
        if (cur < best) best = cur;
        cur = mul(cur, sq, q);
    }
    return best;
}
}  // namespace hm

// ================================================================== context
struct KeyBuf {
    u64 *d = nullptr;   // [L][2][L+1][n], Montgomery form
    u64 last = 0;       // key-use tick of the last launch sequence that referenced it
};

struct Arena;

struct fhe_ctx {
    fhe_params P{};
    int dev = 0;
    cudaStream_t st = nullptr;
    u32 n = 0, logn = 0, N = 0, L = 0, nb = 0, T = 0, nmod = 0;
    int special_id = 0, b_id0 = 0, t_id0 = 0;
    std::vector<u64> mods;             // modulus value per id
    std::vector<ModInfo> hmods;        // with device twiddle pointers
    ModInfo *d_mods = nullptr;
    u64 *d_tw = nullptr;
    u64 *d_s_can = nullptr, *d_s_m = nullptr, *d_s2_m = nullptr;   // [L+1+nb][n], s2 rows [L+1]
    unsigned char *d_sk_ids = nullptr;
    u32 *d_slot2ntt = nullptr, *d_ntt2slot = nullptr;
    std::vector<LevelDev> hlv;         // index by level 1..L
    LevelDev *d_lv = nullptr;
    AuxDev hax{};
    AuxDev *d_ax = nullptr;
    u64 *d_pmod = nullptr;             // P mod prime_i, i in [0, L]
    u32 *d_status = nullptr;           // [0] largest decryption rounding distance (2^-32 units)
                                       // [1] sticky flags: bit 0 rotate_and_sum precondition violated
    u64 pinv[MAXQ]{}, pinv_sh[MAXQ]{};
    u64 pmont[MAXQ]{};                  // P * 2^64 mod q_i (key-switch addends, KsAdd)
    std::unordered_map<u32, KeyBuf> keys;
    u64 key_bytes = 0;
    // Keys are regenerated deterministically (seed, Galois element), so the store is a
    // cache: beyond key_budget bytes the least recently used keys not referenced by
    // the current launch sequence are freed (configs[3] touches ~7,000 steps).
    u64 key_budget = 0;
    u64 key_tick = 1;
    u64 key_evictions = 0;
    std::vector<u64 *> key_free;        // buffers of evicted keys, reused (cudaFree is slow and synchronizing)
    // copy engine: pinned host buffers in fhe_encrypt / fhe_decrypt are copied on their own
    // stream through double-buffered device staging, overlapping the compute stream
    // (separate H2D and D2H streams: PCIe is full duplex; NIO staging slots so a whole
    // chunked batch can be in flight while the previous one is evaluated)
    static constexpr int NIO = 8;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    u64 *io_in[NIO]{}, *io_out[NIO]{};
    size_t io_in_words[NIO]{}, io_out_words[NIO]{};
    cudaEvent_t ev_in_ready[NIO]{}, ev_in_free[NIO]{}, ev_out_ready[NIO]{}, ev_out_free[NIO]{};
    int io_in_next = 0, io_out_next = 0;
    // pinned staging for plaintext encoding (two slots, so encode never waits for the stream)
    u64 *enc_stage[2]{};
    cudaEvent_t enc_ev[2]{};
    int enc_next = 0;
    // workspaces (key switching: one set per lane; lanes = streams the sub-batches rotate over)
    int S = 1;                          // key-switching sub-batch
    u64 *w_D = nullptr, *w_Ext = nullptr, *w_Acc = nullptr;   // current set
    static constexpr int MAXLANES = 4;
    int lanes = 2;                      // FHE_LANES (1..4)
    u64 *ws_D[MAXLANES]{}, *ws_Ext[MAXLANES]{}, *ws_Acc[MAXLANES]{};
    cudaStream_t streams[MAXLANES]{};
    cudaEvent_t ev_fork = nullptr, ev_key = nullptr, ev_join[MAXLANES]{};
    u64 *w_sq = nullptr;
    size_t w_sq_words = 0;
    u64 *w_tmp = nullptr;
    size_t w_tmp_words = 0;
    // plan capture (fhe_capture_begin/end): allocations come from cap_arena, frees of
    // pool memory are deferred to the end of the capture
    Arena *cap_arena = nullptr;
    std::vector<void *> deferred_free;
    size_t live_bytes = 0, peak_bytes = 0;   // pool-allocated ciphertext bytes (arena sizing)
    // profiling
    bool prof = false;
    u64 launches = 0;
    double alg_mm = 0;                  // algorithmic modmuls issued (fhe_work_modmuls)
    // ct-GEMM weight tables ([L][K][O] residues, Montgomery form), keyed by content
    std::unordered_map<u64, u64 *> gemm_tabs;
    struct Rec { const char *name; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> ev_pool;
};

// bracket one launch with events when profiling is on
struct ProfScope {
    fhe_ctx *c;
    const char *name;
    cudaEvent_t a = nullptr;
    ProfScope(fhe_ctx *c_, const char *n) : c(c_), name(n) {
        c->launches++;
        if (!c->prof) return;
        a = take();
        cudaEventRecord(a, c->st);
    }
    cudaEvent_t take() {
        if (c->ev_pool.empty()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            return e;
        }
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    ~ProfScope() {
        if (!c->prof) return;
        cudaEvent_t b = take();
        cudaEventRecord(b, c->st);
        c->recs.push_back({name, a, b});
    }
};

// Device memory of ciphertexts created while a plan walk is captured into a CUDA graph:
// one device slab with a best-fit extent allocator (free extents split and coalesce, so
// the mixed ciphertext sizes of a level-scheduled walk reuse each other's memory).  The
// graph replays the same addresses, so the arena lives as long as the graph or any
// handle into it.
struct Arena {
    u64 *base = nullptr;
    size_t words = 0;
    std::map<size_t, size_t> free_ext;  // offset -> length (words), disjoint, coalesced
    long refs = 0;                      // live ciphertext handles into the arena
    bool orphaned = false;              // its graph was destroyed
    static size_t round(size_t w) { return (w + 31) & ~(size_t)31; }     // 256-byte blocks
    u64 *alloc(size_t w) {
        w = round(w);
        auto best = free_ext.end();
        for (auto it = free_ext.begin(); it != free_ext.end(); ++it)
            if (it->second >= w && (best == free_ext.end() || it->second < best->second)) best = it;
        if (best == free_ext.end()) return nullptr;
        const size_t off = best->first, len = best->second;
        free_ext.erase(best);
        if (len > w) free_ext[off + w] = len - w;
        return base + off;
    }
    void release(u64 *p, size_t w) {
        w = round(w);
        size_t off = (size_t)(p - base);
        auto nx = free_ext.lower_bound(off);
        if (nx != free_ext.begin()) {
            auto pv = std::prev(nx);
            if (pv->first + pv->second == off) { off = pv->first; w += pv->second; free_ext.erase(pv); }
        }
        if (nx != free_ext.end() && off + w == nx->first) { w += nx->second; free_ext.erase(nx); }
        free_ext[off] = w;
    }
};

struct fhe_graph {
    fhe_ctx *ctx;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t exec = nullptr;
    Arena *arena = nullptr;
};

struct fhe_ct {
    fhe_ctx *ctx;
    u32 R, level, count;
    u64 *d;
    Arena *arena;                       // non-null: arena memory (captured plan)
};

struct fhe_pt {
    fhe_ctx *ctx;
    u64 *coef_t;   // [T][n]
    u64 *ntt_m;    // [T][L][n] Montgomery form
    int encoded;
};

static size_t ct_words(const fhe_ct *ct) { return (size_t)ct->count * 2 * ct->level * ct->ctx->n; }

static inline long long nblocks(long long total, int bs = 256) {
    long long b = (total + bs - 1) / bs;
    return b > 148 * 16 ? 148 * 16 : (b < 1 ? 1 : b);
}
#define EW(kernel, total, ...)                                                 \
    do {                                                                       \
        ProfScope ps_(c, #kernel);                                             \
        kernel<<<(unsigned)nblocks(total), 256, 0, c->st>>>(__VA_ARGS__);      \
    } while (0)

// ----------------------------------------------------- row-kernel dispatch
static std::mutex g_attr_mu;
static std::unordered_set<const void *> g_attr_done;

template <int LOGN, bool INV = false, int WO = 0, typename... KArgs, typename... Args>
static void launch_row(fhe_ctx *c, const char *name, void (*kern)(KArgs...), dim3 grid, cudaStream_t st,
                       Args... args) {
    ProfScope ps_(c, name);
    using C = RowCfg<LOGN, INV, WO>;
    const size_t smem = (size_t)C::SMEM_WORDS * sizeof(u64);
    c->alg_mm += (double)grid.x * grid.y * grid.z * (C::N / 2) * LOGN;      // one (I)NTT per row
    {
        std::lock_guard<std::mutex> lk(g_attr_mu);
        if (!g_attr_done.count((const void *)kern)) {
            cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            g_attr_done.insert((const void *)kern);
        }
    }
    if constexpr (C::CR == 1) {
        kern<<<grid, C::TH, smem, st>>>(args...);
    } else {
        // one thread-block cluster of CR CTAs per row (distributed shared memory)
        grid.x *= C::CR;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(C::TH);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C::CR;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
    }
}

#define LOGN_SWITCH(logn, ...)                                   \
    switch (logn) {                                              \
        case 2: { constexpr int LG = 2; __VA_ARGS__; } break;    \
        case 3: { constexpr int LG = 3; __VA_ARGS__; } break;    \
        case 4: { constexpr int LG = 4; __VA_ARGS__; } break;    \
        case 5: { constexpr int LG = 5; __VA_ARGS__; } break;    \
        case 6: { constexpr int LG = 6; __VA_ARGS__; } break;    \
        case 7: { constexpr int LG = 7; __VA_ARGS__; } break;    \
        case 8: { constexpr int LG = 8; __VA_ARGS__; } break;    \
        case 9: { constexpr int LG = 9; __VA_ARGS__; } break;    \
        case 10: { constexpr int LG = 10; __VA_ARGS__; } break;  \
        case 11: { constexpr int LG = 11; __VA_ARGS__; } break;  \
        case 12: { constexpr int LG = 12; __VA_ARGS__; } break;  \
        case 13: { constexpr int LG = 13; __VA_ARGS__; } break;  \
        case 14: { constexpr int LG = 14; __VA_ARGS__; } break;  \
        case 15: { constexpr int LG = 15; __VA_ARGS__; } break;  \
        case 16: { constexpr int LG = 16; __VA_ARGS__; } break;  \
        default: break;                                          \
    }

static int ntt_rows(fhe_ctx *c, int rows, const NttRowsArgs &a, const char *name = "k_ntt_rows") {
    if (rows <= 0) return 0;
    LOGN_SWITCH(c->logn, launch_row<LG, false, FwdW5<LG>::value>(c, name, k_ntt_rows<LG>, dim3(rows), c->st, a, c->d_mods));
    CHECK_LAUNCH();
    return 0;
}
static int intt_rows(fhe_ctx *c, int rows, const InttRowsArgs &a, const char *name = "k_intt_rows") {
    if (rows <= 0) return 0;
    LOGN_SWITCH(c->logn, launch_row<LG, true>(c, name, k_intt_rows<LG>, dim3(rows), c->st, a, c->d_mods));
    CHECK_LAUNCH();
    return 0;
}

static NttRowsArgs nargs(const u64 *src, u64 *dst, long long stride) {
    NttRowsArgs a;
    memset(&a, 0, sizeof a);
    a.src = src; a.dst = dst; a.rdiv = 1; a.sA = stride; a.dA = stride;
    a.div = 1; a.period = 1; a.div2 = 1; a.period2 = 1;
    return a;
}
static InttRowsArgs iargs(const u64 *src, u64 *dst, long long stride) {
    InttRowsArgs a;
    memset(&a, 0, sizeof a);
    a.src = src; a.dst = dst; a.rdiv = 1; a.sA = stride; a.dA = stride;
    a.div = 1; a.period = 1;
    return a;
}
static void map_range(ModMap &m, u32 period, int base) { for (u32 i = 0; i < period; i++) m.id[i] = (unsigned char)(base + i); }
static void map_q(ModMap &m, u32 l) { map_range(m, l, 0); }

static int ensure_tmp(fhe_ctx *c, size_t words) {
    if (words <= c->w_tmp_words) return 0;
    if (c->cap_arena) return fail(FHE_EINVAL, "workspace growth inside a capture (warm the walk up first)");
    if (c->w_tmp) CU(cudaFreeAsync(c->w_tmp, c->st));
    CU(cudaMallocAsync((void **)&c->w_tmp, words * 8, c->st));
    c->w_tmp_words = words;
    return 0;
}

// ------------------------------------------------------------- validation
static int validate(const fhe_params *p) {
    if (p->log_n < 2 || p->log_n > 16) return fail(FHE_EINVAL, "log_n must be in [2, 16] (got %u)", p->log_n);
    if (p->L < 1 || p->L > FHE_MAX_Q) return fail(FHE_EINVAL, "L must be in [1, %d]", FHE_MAX_Q);
    if (p->K != 1) return fail(FHE_EINVAL, "exactly one special prime is supported (K=%u)", p->K);
    if (p->n_aux > FHE_MAX_B) return fail(FHE_EINVAL, "n_aux must be <= %d", FHE_MAX_B);
    if (p->n_aux && p->n_aux < p->L + 1) return fail(FHE_EINVAL, "n_aux must be 0 or >= L+1");
    if (p->T < 1 || p->T > FHE_MAX_T) return fail(FHE_EINVAL, "T must be in [1, %d]", FHE_MAX_T);
    u64 two_n = 2ull << p->log_n;
    std::vector<u64> all;
    for (u32 i = 0; i < p->L; i++) all.push_back(p->q[i]);
    all.push_back(p->p[0]);
    for (u32 i = 0; i < p->n_aux; i++) all.push_back(p->b[i]);
    for (u32 i = 0; i < p->T; i++) all.push_back(p->t[i]);
    for (size_t i = 0; i < all.size(); i++) {
        if (all[i] >= (1ull << 61) || all[i] < 3) return fail(FHE_EINVAL, "modulus %llu outside [3, 2^61)", (unsigned long long)all[i]);
        if (!hm::is_prime(all[i])) return fail(FHE_EINVAL, "modulus %llu is not prime", (unsigned long long)all[i]);
        if (all[i] % two_n != 1) return fail(FHE_EINVAL, "modulus %llu is not 1 mod 2n = %llu", (unsigned long long)all[i], (unsigned long long)two_n);
        for (size_t j = 0; j < i; j++)
            if (all[j] == all[i]) return fail(FHE_EINVAL, "modulus %llu repeated", (unsigned long long)all[i]);
    }
    for (u32 i = 0; i < p->L; i++)
        if (p->p[0] < p->q[i]) return fail(FHE_EINVAL, "special prime must exceed every q_i");
    // the key-switching inner product accumulates L products < q^2 in 128 bits
    if ((u128)p->p[0] * p->L >= ((u128)1 << 64)) return fail(FHE_EINVAL, "L * max modulus must stay below 2^64");
    return 0;
}

// ------------------------------------------------------------- tables
static void build_level(fhe_ctx *c, u32 l, LevelDev &T) {
    memset(&T, 0, sizeof T);
    const u64 *q = c->P.q;
    for (u32 i = 0; i < l; i++) {
        u64 qh = 1;
        for (u32 j = 0; j < l; j++) if (j != i) qh = hm::mul(qh, q[j] % q[i], q[i]);
        T.Qtilde_m[i] = hm::mont(hm::inv(qh, q[i]), q[i]);
        hm::frac128(1, q[i], T.invq_hi[i], T.invq_lo[i]);
        if (l >= 2 && i < l - 1) {
            T.msinv[i] = hm::inv(q[l - 1] % q[i], q[i]);
            T.msinv_sh[i] = hm::shoup(T.msinv[i], q[i]);
            T.qlast_mod[i] = q[l - 1] % q[i];
        }
    }
    T.half_last = (q[l - 1] - 1) / 2;
    for (u32 k = 0; k < c->T; k++) {
        u64 t = c->P.t[k], rt = 1;
        for (u32 j = 0; j < l; j++) rt = hm::mul(rt, q[j] % t, t);
        T.rt[k] = rt;
        T.rtF[k] = (u64)(((u128)rt << 64) / t);
        for (u32 i = 0; i < l; i++) {
            T.decW[k][i] = t / q[i];
            hm::frac128(t % q[i], q[i], T.decFhi[k][i], T.decFlo[k][i]);
            u64 delta = hm::mul(hm::neg(rt, q[i]), hm::inv(t % q[i], q[i]), q[i]);
            T.delta_m[k][i] = hm::mont(delta, q[i]);
        }
    }
    if (!c->nb) return;
    const u64 *b = c->P.b;
    u32 nb = c->nb;
    for (u32 k = 0; k < nb; k++) {
        u64 Qm = 1;
        for (u32 j = 0; j < l; j++) Qm = hm::mul(Qm, q[j] % b[k], b[k]);
        T.QmodB_m[k] = hm::mont(Qm, b[k]);
        for (u32 i = 0; i < l; i++) {
            u64 qh = 1;
            for (u32 j = 0; j < l; j++) if (j != i) qh = hm::mul(qh, q[j] % b[k], b[k]);
            T.QhatB_m[i][k] = hm::mont(qh, b[k]);
        }
        u64 bh = 1;
        for (u32 j = 0; j < nb; j++) if (j != k) bh = hm::mul(bh, b[j] % b[k], b[k]);
        T.Mtb_m[k] = hm::mont(hm::inv(hm::mul(bh, Qm, b[k]), b[k]), b[k]);
    }
    for (u32 i = 0; i < l; i++) {
        u64 Bm = 1;
        for (u32 k = 0; k < nb; k++) Bm = hm::mul(Bm, b[k] % q[i], q[i]);
        u64 qh = 1;
        for (u32 j = 0; j < l; j++) if (j != i) qh = hm::mul(qh, q[j] % q[i], q[i]);
        T.Mtq_m[i] = hm::mont(hm::inv(hm::mul(qh, Bm, q[i]), q[i]), q[i]);
        for (u32 kt = 0; kt < c->T; kt++) {
            u64 t = c->P.t[kt];
            u64 tBq = hm::mul(t % q[i], Bm, q[i]);
            hm::frac128(tBq, q[i], T.theta_hi[kt][i], T.theta_lo[kt][i]);
            for (u32 k = 0; k < nb; k++) {
                u64 om = hm::mul(hm::neg(tBq % b[k], b[k]), hm::inv(q[i] % b[k], b[k]), b[k]);
                T.omega_m[kt][i][k] = hm::mont(om, b[k]);
            }
        }
    }
    for (u32 kt = 0; kt < c->T; kt++) {
        u64 t = c->P.t[kt];
        for (u32 k = 0; k < nb; k++) {
            u64 bh = 1;
            for (u32 j = 0; j < nb; j++) if (j != k) bh = hm::mul(bh, b[j] % b[k], b[k]);
            T.tBb_m[kt][k] = hm::mont(hm::mul(t % b[k], bh, b[k]), b[k]);
        }
    }
}

static void build_aux(fhe_ctx *c, AuxDev &A) {
    memset(&A, 0, sizeof A);
    const u64 *b = c->P.b, *q = c->P.q;
    for (u32 k = 0; k < c->nb; k++) {
        u64 bh = 1;
        for (u32 j = 0; j < c->nb; j++) if (j != k) bh = hm::mul(bh, b[j] % b[k], b[k]);
        A.Btilde_m[k] = hm::mont(hm::inv(bh, b[k]), b[k]);
        hm::frac128(1, b[k], A.invb_hi[k], A.invb_lo[k]);
        for (u32 i = 0; i < c->L; i++) {
            u64 h = 1;
            for (u32 j = 0; j < c->nb; j++) if (j != k) h = hm::mul(h, b[j] % q[i], q[i]);
            A.BhatQ_m[k][i] = hm::mont(h, q[i]);
        }
    }
    for (u32 i = 0; i < c->L; i++) {
        u64 Bm = 1;
        for (u32 k = 0; k < c->nb; k++) Bm = hm::mul(Bm, b[k] % q[i], q[i]);
        A.BmodQ_m[i] = hm::mont(Bm, q[i]);
    }
}

static int setup_moduli(fhe_ctx *c) {
    u32 n = c->n;
    c->nmod = c->L + 1 + c->nb + c->T;
    c->special_id = c->L;
    c->b_id0 = c->L + 1;
    c->t_id0 = c->L + 1 + c->nb;
    c->mods.clear();
    for (u32 i = 0; i < c->L; i++) c->mods.push_back(c->P.q[i]);
    c->mods.push_back(c->P.p[0]);
    for (u32 i = 0; i < c->nb; i++) c->mods.push_back(c->P.b[i]);
    for (u32 i = 0; i < c->T; i++) c->mods.push_back(c->P.t[i]);
    std::vector<u64> tw((size_t)c->nmod * 4 * n);
    CU(cudaMalloc((void **)&c->d_tw, tw.size() * 8));
    c->hmods.resize(c->nmod);
    std::vector<u64> pw(n), pwi(n);
    for (u32 id = 0; id < c->nmod; id++) {
        u64 q = c->mods[id];
        u64 psi = hm::min_root(q, n), psi_inv = hm::inv(psi, q);
        pw[0] = 1; pwi[0] = 1;
        for (u32 k = 1; k < n; k++) { pw[k] = hm::mul(pw[k - 1], psi, q); pwi[k] = hm::mul(pwi[k - 1], psi_inv, q); }
        u64 *base = tw.data() + (size_t)id * 4 * n;
        for (u32 k = 0; k < n; k++) {
            u64 w = pw[hm::brev(k, c->logn)], wi = pwi[hm::brev(k, c->logn)];
            base[2 * k] = w;
            base[2 * k + 1] = hm::shoup(w, q);
            base[2 * n + 2 * k] = wi;
            base[2 * n + 2 * k + 1] = hm::shoup(wi, q);
        }
        ModInfo &M = c->hmods[id];
        M.q = q;
        u64 x = q;                         // Newton: q^-1 mod 2^64
        for (int it = 0; it < 6; it++) x *= 2 - q * x;
        M.qinv = x;
        u64 r1 = (u64)(((u128)1 << 64) % q);
        M.r2 = hm::mul(r1, r1, q);
        M.mu = (u64)(((u128)1 << 64) / q);
        M.ninv = hm::inv(n, q);
        M.ninv_sh = hm::shoup(M.ninv, q);
        M.w1ninv = hm::mul(pwi[hm::brev(1, c->logn)], M.ninv, q);
        M.w1ninv_sh = hm::shoup(M.w1ninv, q);
        M.half = (q - 1) / 2;
        M.nq = (u64)0 - q;
        M.q3 = 3 * q;
        u64 *dbase = c->d_tw + (size_t)id * 4 * n;
        M.tw = (const ulonglong2 *)dbase;
        M.itw = (const ulonglong2 *)(dbase + 2 * n);
    }
    CU(cudaMemcpy(c->d_tw, tw.data(), tw.size() * 8, cudaMemcpyHostToDevice));
    CU(cudaMalloc((void **)&c->d_mods, c->nmod * sizeof(ModInfo)));
    CU(cudaMemcpy(c->d_mods, c->hmods.data(), c->nmod * sizeof(ModInfo), cudaMemcpyHostToDevice));
    return 0;
}

static int setup_secret(fhe_ctx *c) {
    u32 n = c->n, nks = c->L + 1 + c->nb;
    std::vector<unsigned char> ids(nks);
    for (u32 r = 0; r < nks; r++) ids[r] = (unsigned char)r;   // q..., special, aux... (ids coincide)
    CU(cudaMalloc((void **)&c->d_sk_ids, nks));
    CU(cudaMemcpy(c->d_sk_ids, ids.data(), nks, cudaMemcpyHostToDevice));
    CU(cudaMalloc((void **)&c->d_s_can, (size_t)nks * n * 8));
    CU(cudaMalloc((void **)&c->d_s_m, (size_t)nks * n * 8));
    CU(cudaMalloc((void **)&c->d_s2_m, (size_t)(c->L + 1) * n * 8));
    long long total = (long long)nks * n;
    EW(k_sk_prep, total, c->d_s_can, total, (int)c->logn, c->P.seed, c->d_sk_ids, c->d_mods);
    CHECK_LAUNCH();
    NttRowsArgs a = nargs(c->d_s_can, c->d_s_can, n);
    a.period = nks;
    map_range(a.map, nks, 0);
    TRY(ntt_rows(c, nks, a));
    EW(k_sk_finish, total, c->d_s_can, c->d_s_m, c->d_s2_m, total, (int)(c->L + 1), (int)c->logn, c->d_sk_ids,
       c->d_mods);
    CHECK_LAUNCH();
    // P mod prime_i and P^-1 mod q_i
    std::vector<u64> pm(c->L + 1);
    u64 P = c->P.p[0];
    for (u32 i = 0; i <= c->L; i++) pm[i] = P % c->mods[i];
    for (u32 i = 0; i < c->L; i++) {
        c->pinv[i] = hm::inv(pm[i], c->P.q[i]);
        c->pinv_sh[i] = hm::shoup(c->pinv[i], c->P.q[i]);
        c->pmont[i] = hm::mont(pm[i], c->P.q[i]);
    }
    CU(cudaMalloc((void **)&c->d_pmod, (c->L + 1) * 8));
    CU(cudaMemcpy(c->d_pmod, pm.data(), (c->L + 1) * 8, cudaMemcpyHostToDevice));
    CU(cudaMalloc((void **)&c->d_status, 2 * sizeof(u32)));
    CU(cudaMemset(c->d_status, 0, 2 * sizeof(u32)));
    return 0;
}

static int setup_workspace(fhe_ctx *c) {
    size_t n = c->n, L = c->L;
    size_t per_ct = n * (L + L * (L + 1) + 2 * (L + 1)) * 8;
    // sub-batch: as many ciphertexts as 1.25 GB of workspace per lane holds, at most MAXS
    // (128 measured best at configs[1]: fewer partial waves of the row kernels;
    // profiles/r02_subbatch.json)
    // (rings 2^15 / 2^16 keep the 512 MB budget: their ciphertext objects are GBs and
    // the engine's output groups are sized against what the workspaces leave)
    size_t budget = (c->logn > 14 ? 512ull : 1280ull) << 20;
    const char *env = getenv("FHE_KS_BATCH");
    int S = env ? atoi(env) : (int)(budget / per_ct);
    if (!env && S < 8) S = 8;          // large rings: keep >= 8 ciphertexts per sub-batch
    if (S < 1) S = 1;
    if (S > MAXS) S = MAXS;
    c->S = S;
    const char *lenv = getenv("FHE_LANES");
    c->lanes = lenv ? std::max(1, std::min(fhe_ctx::MAXLANES, atoi(lenv))) : 2;
    for (int k = 0; k < c->lanes; k++) {
        CU(cudaMalloc((void **)&c->ws_D[k], S * L * n * 8));
        CU(cudaMalloc((void **)&c->ws_Ext[k], S * L * (L + 1) * n * 8));
        CU(cudaMalloc((void **)&c->ws_Acc[k], S * 2 * (L + 1) * n * 8));
    }
    c->w_D = c->ws_D[0]; c->w_Ext = c->ws_Ext[0]; c->w_Acc = c->ws_Acc[0];
    for (int k = 1; k < c->lanes; k++) {
        CU(cudaStreamCreateWithFlags(&c->streams[k], cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&c->ev_join[k], cudaEventDisableTiming));
    }
    CU(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&c->ev_key, cudaEventDisableTiming));
    CU(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    for (int j = 0; j < fhe_ctx::NIO; j++) {
        CU(cudaEventCreateWithFlags(&c->ev_in_ready[j], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->ev_in_free[j], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->ev_out_ready[j], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->ev_out_free[j], cudaEventDisableTiming));
    }
    {
        // key cache budget: FHE_KEY_BUDGET_MB, default 40 % of device memory
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        const char *kenv = getenv("FHE_KEY_BUDGET_MB");
        c->key_budget = kenv ? (u64)atoll(kenv) << 20 : (u64)(tot / 5 * 2);
    }
    if (c->nb) {
        size_t l = L, nb = c->nb;
        c->w_sq_words = S * n * (2 * l + 2 * nb + 3 * (l + nb) + 3 * l + 3 * l);
        CU(cudaMalloc((void **)&c->w_sq, c->w_sq_words * 8));
    }
    return 0;
}

extern "C" int fhe_ctx_create(const fhe_params *params, fhe_ctx **out) {
    TRY(validate(params));
    fhe_ctx *c = new fhe_ctx();
    c->P = *params;
    c->dev = params->device;
    c->logn = params->log_n;
    c->n = 1u << c->logn;
    c->N = c->n / 2;
    c->L = params->L;
    c->nb = params->n_aux;
    c->T = params->T;
    int rc = 0;
    do {
        if (cudaSetDevice(c->dev) != cudaSuccess) { rc = fail(FHE_EDEVICE, "cannot select CUDA device %d", c->dev); break; }
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, c->dev) != cudaSuccess) { rc = fail(FHE_EDEVICE, "no CUDA device"); break; }
        if (prop.major != 10) { rc = fail(FHE_EDEVICE, "device %s is sm_%d%d; this build targets sm_100a", prop.name, prop.major, prop.minor); break; }
        if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) { rc = fail(FHE_EDEVICE, "stream creation failed"); break; }
        c->streams[0] = c->st;
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, c->dev) == cudaSuccess) {
            u64 thresh = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh);
        }
        if ((rc = setup_moduli(c))) break;
        // slot maps
        std::vector<u32> s2n(c->n), n2s(c->n);
        u64 two_n = 2ull * c->n, e = 1;
        for (u32 i = 0; i < c->N; i++) {
            s2n[i] = hm::brev((u32)((e - 1) / 2), c->logn);
            s2n[c->N + i] = hm::brev((u32)((two_n - e - 1) / 2), c->logn);
            e = e * 5 % two_n;
        }
        for (u32 x = 0; x < c->n; x++) n2s[s2n[x]] = x;
        if (cudaMalloc((void **)&c->d_slot2ntt, c->n * 4) || cudaMalloc((void **)&c->d_ntt2slot, c->n * 4)) { rc = fail(FHE_ENOMEM, "cudaMalloc"); break; }
        cudaMemcpy(c->d_slot2ntt, s2n.data(), c->n * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(c->d_ntt2slot, n2s.data(), c->n * 4, cudaMemcpyHostToDevice);
        c->hlv.resize(c->L + 1);
        for (u32 l = 1; l <= c->L; l++) build_level(c, l, c->hlv[l]);
        if (cudaMalloc((void **)&c->d_lv, (c->L + 1) * sizeof(LevelDev)) != cudaSuccess) { rc = fail(FHE_ENOMEM, "cudaMalloc"); break; }
        cudaMemcpy(c->d_lv, c->hlv.data(), (c->L + 1) * sizeof(LevelDev), cudaMemcpyHostToDevice);
        if (c->nb) {
            build_aux(c, c->hax);
            cudaMalloc((void **)&c->d_ax, sizeof(AuxDev));
            cudaMemcpy(c->d_ax, &c->hax, sizeof(AuxDev), cudaMemcpyHostToDevice);
        }
        if ((rc = setup_secret(c))) break;
        if ((rc = setup_workspace(c))) break;
        if (cudaStreamSynchronize(c->st) != cudaSuccess) { rc = fail(FHE_EDEVICE, "context setup failed: %s", cudaGetErrorString(cudaGetLastError())); break; }
    } while (0);
    if (rc) {
        fhe_ctx_destroy(c);
        return rc;
    }
    *out = c;
    return 0;
}

extern "C" void fhe_ctx_destroy(fhe_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->dev);
    if (c->st) cudaStreamSynchronize(c->st);
    for (auto &kv : c->keys) cudaFree(kv.second.d);
    for (auto &kv : c->gemm_tabs) cudaFree(kv.second);
    for (u64 *d : c->key_free) cudaFree(d);
    for (int j = 0; j < 2; j++) {
        if (c->enc_stage[j]) cudaFreeHost(c->enc_stage[j]);
        if (c->enc_ev[j]) cudaEventDestroy(c->enc_ev[j]);
    }
    if (c->h2d) { cudaStreamSynchronize(c->h2d); cudaStreamDestroy(c->h2d); }
    if (c->d2h) { cudaStreamSynchronize(c->d2h); cudaStreamDestroy(c->d2h); }
    for (int j = 0; j < fhe_ctx::NIO; j++) {
        if (c->io_in[j]) cudaFree(c->io_in[j]);
        if (c->io_out[j]) cudaFree(c->io_out[j]);
        cudaEvent_t evs[] = {c->ev_in_ready[j], c->ev_in_free[j], c->ev_out_ready[j], c->ev_out_free[j]};
        for (cudaEvent_t e : evs) if (e) cudaEventDestroy(e);
    }
    void *bufs[] = {c->d_mods, c->d_tw, c->d_s_can, c->d_s_m, c->d_s2_m, c->d_sk_ids, c->d_slot2ntt,
                    c->d_ntt2slot, c->d_lv, c->d_ax, c->d_pmod, c->w_sq, c->d_status};
    for (void *b : bufs) if (b) cudaFree(b);
    for (int k = 0; k < fhe_ctx::MAXLANES; k++) {
        void *wb[] = {c->ws_D[k], c->ws_Ext[k], c->ws_Acc[k]};
        for (void *b : wb) if (b) cudaFree(b);
    }
    for (int k = 1; k < fhe_ctx::MAXLANES; k++) {
        if (c->streams[k]) { cudaStreamSynchronize(c->streams[k]); cudaStreamDestroy(c->streams[k]); }
        if (c->ev_join[k]) cudaEventDestroy(c->ev_join[k]);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_key) cudaEventDestroy(c->ev_key);
    if (c->w_tmp) cudaFreeAsync(c->w_tmp, c->st);
    if (c->st) { cudaStreamSynchronize(c->st); cudaStreamDestroy(c->st); }
    delete c;
}

extern "C" int fhe_sync(fhe_ctx *c) {
    CU(cudaStreamSynchronize(c->st));
    if (c->h2d) CU(cudaStreamSynchronize(c->h2d));
    if (c->d2h) CU(cudaStreamSynchronize(c->d2h));
    return 0;
}

static bool is_pinned(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return at.type == cudaMemoryTypeHost;
}

// (re)size a device staging buffer once no copy uses it
static int ensure_stage(fhe_ctx *c, u64 **buf, size_t *have, size_t words) {
    if (*have >= words) return 0;
    CU(cudaStreamSynchronize(c->h2d));
    CU(cudaStreamSynchronize(c->d2h));
    CU(cudaStreamSynchronize(c->st));
    if (*buf) CU(cudaFree(*buf));
    CU(cudaMalloc((void **)buf, words * 8));
    *have = words;
    return 0;
}

extern "C" int fhe_ctx_stream(fhe_ctx *c, void **stream) {
    *stream = (void *)c->st;
    return 0;
}

extern "C" int fhe_peak_modmul_kind(fhe_ctx *c, uint32_t iters, int kind, double *out) {
    if (kind != 0 && kind != 1) return fail(FHE_EINVAL, "peak kind must be 0 (exact Shoup) or 1 (approximate-quotient Shoup)");
    auto kern = kind ? k_peak_modmul<1> : k_peak_modmul<0>;
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->dev));
    const int blocks = sms * 8, threads = 256;
    u64 q = c->P.q[0], w = q / 3 + 7, wsh = hm::shoup(w, q);
    u64 *sink;
    CU(cudaMallocAsync((void **)&sink, 8, c->st));
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    kern<<<blocks, threads, 0, c->st>>>(sink, iters / 8 + 1, q, w, wsh);   // warm-up
    CU(cudaEventRecord(e0, c->st));
    kern<<<blocks, threads, 0, c->st>>>(sink, iters, q, w, wsh);
    CU(cudaEventRecord(e1, c->st));
    CU(cudaEventSynchronize(e1));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CU(cudaFreeAsync(sink, c->st));
    *out = (double)blocks * threads * 8.0 * iters / (ms * 1e-3);
    return 0;
}
extern "C" int fhe_peak_modmul(fhe_ctx *c, uint32_t iters, double *out) { return fhe_peak_modmul_kind(c, iters, 0, out); }

extern "C" int fhe_prof_enable(fhe_ctx *c, int on) {
    c->prof = on != 0;
    return 0;
}

extern "C" int fhe_prof_report(fhe_ctx *c, char *buf, uint32_t len) {
    CU(cudaStreamSynchronize(c->st));
    std::vector<std::pair<std::string, std::pair<long, double>>> agg;
    for (auto &r : c->recs) {
        float ms = 0;
        cudaEventElapsedTime(&ms, r.a, r.b);
        bool found = false;
        for (auto &x : agg)
            if (x.first == r.name) { x.second.first++; x.second.second += ms; found = true; break; }
        if (!found) agg.push_back({r.name, {1, (double)ms}});
        c->ev_pool.push_back(r.a);
        c->ev_pool.push_back(r.b);
    }
    c->recs.clear();
    std::string out;
    char line[256];
    for (auto &x : agg) {
        snprintf(line, sizeof line, "%s %ld %.6f\n", x.first.c_str(), x.second.first, x.second.second);
        out += line;
    }
    if (len) {
        strncpy(buf, out.c_str(), len - 1);
        buf[len - 1] = 0;
    }
    return 0;
}

extern "C" int fhe_work_modmuls(fhe_ctx *c, double *out) {
    *out = c->alg_mm;
    return 0;
}

extern "C" int fhe_launch_count(fhe_ctx *c, uint64_t *out) {
    *out = c->launches;
    return 0;
}

extern "C" int fhe_ctx_key_bytes(fhe_ctx *c, uint64_t *out) {
    *out = c->key_bytes;
    return 0;
}

// ===================================================================== keys
static u32 galois_elt(const fhe_ctx *c, u32 k) { return (u32)hm::pw(5, k, 2ull * c->n); }

static int evict_keys(fhe_ctx *c, size_t need) {
    if (c->key_bytes + need <= c->key_budget) return 0;
    // free down to 3/4 of the budget in one go (one device sync per eviction round)
    const u64 target = c->key_budget / 4 * 3;
    std::vector<std::pair<u64, u32>> lru;
    for (auto &kv : c->keys)
        if (kv.second.last < c->key_tick && kv.first != 0) lru.push_back({kv.second.last, kv.first});
    if (lru.empty()) return 0;                 // everything is pinned: exceed the budget
    std::sort(lru.begin(), lru.end());
    CU(cudaDeviceSynchronize());               // in-flight sub-batches may still read them
    const size_t words = (size_t)c->L * 2 * (c->L + 1) * c->n;
    for (auto &e : lru) {
        if (c->key_bytes + need <= target) break;
        c->key_free.push_back(c->keys[e.second].d);
        c->keys.erase(e.second);
        c->key_bytes -= words * 8;
        c->key_evictions++;
    }
    return 0;
}

static int get_key(fhe_ctx *c, u32 kid, const u64 **out) {
    auto it = c->keys.find(kid);
    if (it != c->keys.end()) {
        it->second.last = c->key_tick;
        *out = it->second.d;
        return 0;
    }
    if (c->cap_arena) return fail(FHE_EINVAL, "key for Galois element %u was not generated before the capture", kid);
    size_t n = c->n, L = c->L;
    size_t words = L * 2 * (L + 1) * n;
    TRY(evict_keys(c, words * 8));
    KeyBuf kb;
    if (!c->key_free.empty()) {
        kb.d = c->key_free.back();
        c->key_free.pop_back();
    } else {
        CU(cudaMalloc((void **)&kb.d, words * 8));
    }
    kb.last = c->key_tick;
    // generate on stream 0 (the shared w_tmp lives there); the other lanes wait for it
    cudaStream_t caller = c->st;
    c->st = c->streams[0];
    TRY(ensure_tmp(c, L * (L + 1) * n));
    long long total = (long long)L * (L + 1) * n;
    EW(k_key_prep, total, c->w_tmp, total, (int)L, (int)c->logn, c->P.seed, kid, c->special_id, c->d_mods);
    CHECK_LAUNCH();
    NttRowsArgs a = nargs(c->w_tmp, c->w_tmp, n);
    a.period = L + 1;
    map_range(a.map, L + 1, 0);   // ids 0..L-1 = q, L = special
    TRY(ntt_rows(c, (int)(L * (L + 1)), a));
    EW(k_key_finish, total, c->w_tmp, kb.d, c->d_s_m, c->d_s_can, c->d_s2_m, c->d_pmod, total, (int)L,
       (int)c->logn, c->P.seed, kid, c->special_id, c->d_mods);
    CHECK_LAUNCH();
    c->st = caller;
    if (c->lanes > 1) {
        // every later launch on the other lanes (not only the caller's: a cached key is
        // reused by the next sub-batch without a wait) is ordered after the generation
        CU(cudaEventRecord(c->ev_key, c->streams[0]));
        for (int k = 1; k < c->lanes; k++) CU(cudaStreamWaitEvent(c->streams[k], c->ev_key, 0));
    }
    c->keys[kid] = kb;
    c->key_bytes += words * 8;
    *out = kb.d;
    return 0;
}

extern "C" int fhe_keygen_rotations(fhe_ctx *c, const uint32_t *steps, uint32_t m) {
    for (u32 i = 0; i < m; i++) {
        if (steps[i] == 0 || steps[i] >= c->N) return fail(FHE_EINVAL, "rotation step %u outside [1, %u)", steps[i], c->N);
        const u64 *k;
        c->key_tick++;
        TRY(get_key(c, galois_elt(c, steps[i]), &k));
    }
    return 0;
}

// ================================================================== objects
static bool same_shape_rl(const fhe_ct *a, const fhe_ct *b) { return a->R == b->R && a->level == b->level; }

extern "C" int fhe_ct_create(fhe_ctx *c, uint32_t R, uint32_t level, fhe_ct **out) {
    if (R < 1) return fail(FHE_EINVAL, "R must be >= 1");
    if (level < 1 || level > c->L) return fail(FHE_ELEVEL, "level %u outside [1, %u]", level, c->L);
    fhe_ct *ct = new fhe_ct{c, R, level, R * c->T, nullptr, nullptr};
    const size_t words = ct_words(ct);
    if (Arena *a = c->cap_arena) {
        ct->d = a->alloc(words);
        if (!ct->d) {
            delete ct;
            return fail(FHE_ENOMEM, "capture arena exhausted (%zu words); capture with a larger arena", a->words);
        }
        ct->arena = a;
        a->refs++;
        *out = ct;
        return 0;
    }
    cudaError_t e = cudaMallocAsync((void **)&ct->d, words * 8, c->st);
    if (e != cudaSuccess) {
        // The stream-ordered pool keeps freed blocks (release threshold: never) and fragments
        // when ciphertext sizes mix (level schedule, GB-sized objects at ring 2^16): wait for
        // the pending frees, hand the unused reservations back and try once more.
        cudaGetLastError();
        cudaDeviceSynchronize();
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, c->dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
        e = cudaMallocAsync((void **)&ct->d, words * 8, c->st);
    }
    if (e != cudaSuccess) {
        size_t fr = 0, tot = 0;
        cudaGetLastError();
        cudaMemGetInfo(&fr, &tot);
        delete ct;
        return fail(FHE_ENOMEM, "ciphertext allocation of %zu bytes failed: %s (device: %zu MB free of %zu MB; live ciphertexts %zu MB, keys %llu MB)",
                    words * 8, cudaGetErrorString(e), fr >> 20, tot >> 20, c->live_bytes >> 20,
                    (unsigned long long)(c->key_bytes >> 20));
    }
    c->live_bytes += words * 8;
    c->peak_bytes = std::max(c->peak_bytes, c->live_bytes);
    *out = ct;
    return 0;
}
static void arena_release(Arena *a) {
    if (a->orphaned && a->refs == 0) {
        cudaDeviceSynchronize();
        cudaFree(a->base);
        delete a;
    }
}
extern "C" void fhe_ct_destroy(fhe_ct *ct) {
    if (!ct) return;
    fhe_ctx *c = ct->ctx;
    if (Arena *a = ct->arena) {
        // during its capture the block returns to the free list (later captured work
        // reuses it in stream order); afterwards the graph keeps writing it
        if (a == c->cap_arena) a->release(ct->d, ct_words(ct));
        a->refs--;
        arena_release(a);
    } else if (c->cap_arena) {
        c->deferred_free.push_back(ct->d);               // no pool frees inside a capture
        c->live_bytes -= ct_words(ct) * 8;
    } else {
        cudaFreeAsync(ct->d, c->streams[0]);
        c->live_bytes -= ct_words(ct) * 8;
    }
    delete ct;
}

extern "C" int fhe_ct_copy(fhe_ctx *c, const fhe_ct *src, fhe_ct *dst) {
    if (!same_shape_rl(src, dst)) return fail(FHE_ELEVEL, "ct_copy: shape/level mismatch");
    CU(cudaMemcpyAsync(dst->d, src->d, ct_words(src) * 8, cudaMemcpyDeviceToDevice, c->st));
    return 0;
}

extern "C" int fhe_ctx_peak_bytes(fhe_ctx *c, uint64_t *out, int reset) {
    *out = c->peak_bytes;
    if (reset) c->peak_bytes = c->live_bytes;
    return 0;
}

extern "C" int fhe_capture_begin(fhe_ctx *c, uint64_t arena_bytes) {
    if (c->cap_arena) return fail(FHE_EINVAL, "capture_begin: a capture is already running");
    if (c->prof) return fail(FHE_EINVAL, "capture_begin: profiling is on");
    for (int k = 0; k < c->lanes; k++) CU(cudaStreamSynchronize(c->streams[k]));
    Arena *a = new Arena();
    a->words = arena_bytes / 8 & ~(size_t)31;
    a->free_ext[0] = a->words;
    if (cudaMalloc((void **)&a->base, a->words * 8) != cudaSuccess) {
        delete a;
        cudaGetLastError();
        return fail(FHE_ENOMEM, "capture arena of %llu bytes", (unsigned long long)arena_bytes);
    }
    cudaError_t e = cudaStreamBeginCapture(c->streams[0], cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) {
        cudaFree(a->base);
        delete a;
        return fail(FHE_EDEVICE, "cudaStreamBeginCapture: %s", cudaGetErrorString(e));
    }
    c->st = c->streams[0];
    c->cap_arena = a;
    return 0;
}

extern "C" int fhe_capture_end(fhe_ctx *c, fhe_graph **out) {
    Arena *a = c->cap_arena;
    if (!a) return fail(FHE_EINVAL, "capture_end: no capture is running");
    c->cap_arena = nullptr;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(c->streams[0], &g);
    for (void *p : c->deferred_free) cudaFreeAsync(p, c->streams[0]);
    c->deferred_free.clear();
    if (e != cudaSuccess || !g) {
        a->orphaned = true;
        arena_release(a);
        return fail(FHE_EDEVICE, "cudaStreamEndCapture: %s (an operation in the walk is not capturable)",
                    cudaGetErrorString(e));
    }
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, g, 0);
    if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        a->orphaned = true;
        arena_release(a);
        return fail(FHE_EDEVICE, "cudaGraphInstantiate: %s", cudaGetErrorString(e));
    }
    size_t nodes = 0;
    cudaGraphGetNodes(g, nullptr, &nodes);
    *out = new fhe_graph{c, g, exec, a};
    return 0;
}

extern "C" int fhe_graph_launch(fhe_ctx *c, fhe_graph *g) {
    if (c->cap_arena) return fail(FHE_EINVAL, "graph_launch inside a capture");
    ProfScope ps_(c, "graph");
    CU(cudaGraphLaunch(g->exec, c->st));
    return 0;
}

extern "C" int fhe_graph_nodes(fhe_graph *g, uint64_t *out) {
    size_t n = 0;
    if (cudaGraphGetNodes(g->g, nullptr, &n) != cudaSuccess) return fail(FHE_EDEVICE, "cudaGraphGetNodes");
    *out = n;
    return 0;
}

extern "C" void fhe_graph_destroy(fhe_graph *g) {
    if (!g) return;
    cudaStreamSynchronize(g->ctx->streams[0]);
    cudaGraphExecDestroy(g->exec);
    cudaGraphDestroy(g->g);
    g->arena->orphaned = true;
    arena_release(g->arena);
    delete g;
}
extern "C" uint32_t fhe_ct_level(const fhe_ct *ct) { return ct->level; }
extern "C" uint32_t fhe_ct_rows(const fhe_ct *ct) { return ct->R; }

extern "C" int fhe_ct_read(fhe_ctx *c, const fhe_ct *ct, uint64_t *w) {
    CU(cudaMemcpyAsync(w, ct->d, ct_words(ct) * 8, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    return 0;
}
extern "C" int fhe_ct_write(fhe_ctx *c, fhe_ct *ct, const uint64_t *w) {
    CU(cudaMemcpyAsync(ct->d, w, ct_words(ct) * 8, cudaMemcpyHostToDevice, c->st));
    CU(cudaStreamSynchronize(c->st));
    return 0;
}
extern "C" int fhe_ct_to_device(fhe_ctx *c, const fhe_ct *ct, void *dst) {
    CU(cudaMemcpyAsync(dst, ct->d, ct_words(ct) * 8, cudaMemcpyDeviceToDevice, c->st));
    CU(cudaStreamSynchronize(c->st));
    return 0;
}
extern "C" int fhe_ct_from_device(fhe_ctx *c, fhe_ct *ct, const void *src) {
    CU(cudaMemcpyAsync(ct->d, src, ct_words(ct) * 8, cudaMemcpyDeviceToDevice, c->st));
    CU(cudaStreamSynchronize(c->st));
    return 0;
}
extern "C" int fhe_ct_zero(fhe_ctx *c, fhe_ct *ct) {
    CU(cudaMemsetAsync(ct->d, 0, ct_words(ct) * 8, c->st));
    return 0;
}

extern "C" int fhe_pt_create(fhe_ctx *c, fhe_pt **out) {
    if (c->cap_arena) return fail(FHE_EINVAL, "plaintext creation inside a capture (warm the walk up first)");
    fhe_pt *pt = new fhe_pt{c, nullptr, nullptr, 0};
    size_t n = c->n;
    if (cudaMallocAsync((void **)&pt->coef_t, c->T * n * 8, c->st) != cudaSuccess ||
        cudaMallocAsync((void **)&pt->ntt_m, (size_t)c->T * c->L * n * 8, c->st) != cudaSuccess) {
        delete pt;
        return fail(FHE_ENOMEM, "plaintext allocation failed");
    }
    *out = pt;
    return 0;
}
extern "C" void fhe_pt_destroy(fhe_pt *pt) {
    if (!pt) return;
    if (pt->ctx->cap_arena) {
        pt->ctx->deferred_free.push_back(pt->coef_t);
        pt->ctx->deferred_free.push_back(pt->ntt_m);
        delete pt;
        return;
    }
    // stream 0 explicitly: a finalizer may run while a call has switched c->st to lane 1
    cudaFreeAsync(pt->coef_t, pt->ctx->streams[0]);
    cudaFreeAsync(pt->ntt_m, pt->ctx->streams[0]);
    delete pt;
}

// slots [rows][n] (device) -> coefficients mod t_{(r / div) % T} (device)
static int slots_to_coef(fhe_ctx *c, const u64 *slots, u64 *coef, int rows, u32 div) {
    InttRowsArgs a = iargs(slots, coef, c->n);
    a.div = div;
    a.period = c->T;
    map_range(a.map, c->T, c->t_id0);
    a.gather = 1;
    a.tab = c->d_ntt2slot;
    a.reduce = 1;
    return intt_rows(c, rows, a);
}

extern "C" int fhe_encode(fhe_ctx *c, const uint64_t *slots, fhe_pt *pt) {
    size_t n = c->n;
    TRY(ensure_tmp(c, c->T * n));
    // host slots -> pinned slot (after its previous copy completed) -> device, asynchronously
    const int j = c->enc_next;
    c->enc_next ^= 1;
    if (!c->enc_stage[j]) {
        CU(cudaMallocHost((void **)&c->enc_stage[j], c->T * n * 8));
        CU(cudaEventCreateWithFlags(&c->enc_ev[j], cudaEventDisableTiming));
    } else {
        CU(cudaEventSynchronize(c->enc_ev[j]));
    }
    memcpy(c->enc_stage[j], slots, c->T * n * 8);
    CU(cudaMemcpyAsync(c->w_tmp, c->enc_stage[j], c->T * n * 8, cudaMemcpyHostToDevice, c->st));
    CU(cudaEventRecord(c->enc_ev[j], c->st));
    TRY(slots_to_coef(c, c->w_tmp, pt->coef_t, (int)c->T, 1));
    // centered lift t_k -> q_i, NTT, Montgomery form; row r = k*L + i
    NttRowsArgs a = nargs(pt->coef_t, pt->ntt_m, 0);
    a.rdiv = c->L; a.sA = n; a.sB = 0; a.dA = (long long)c->L * n; a.dB = n;
    a.div = 1; a.period = c->L; map_q(a.map, c->L);
    a.div2 = c->L; a.period2 = c->T; map_range(a.srcmap, c->T, c->t_id0);
    a.load = 2; a.epi = 1;
    TRY(ntt_rows(c, (int)(c->T * c->L), a));
    pt->encoded = 1;
    return 0;
}

extern "C" int fhe_pt_read(fhe_ctx *c, const fhe_pt *pt, uint64_t *w) {
    size_t words = (size_t)c->T * c->L * c->n;
    TRY(ensure_tmp(c, words));
    EW(k_from_mont, (long long)words, pt->ntt_m, c->w_tmp, (long long)words, (int)c->L, (int)c->logn, c->d_mods);
    CHECK_LAUNCH();
    CU(cudaMemcpyAsync(w, c->w_tmp, words * 8, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    return 0;
}

// ============================================================ client side
extern "C" int fhe_encrypt(fhe_ctx *c, const uint64_t *slots, uint32_t nonce, fhe_ct *ct) {
    if (ct->level != c->L) return fail(FHE_ELEVEL, "encryption target must be at the top level");
    size_t n = c->n, L = c->L, cnt = ct->count;
    TRY(ensure_tmp(c, cnt * n * (2 + L)));
    u64 *s_dev = c->w_tmp, *m = c->w_tmp + cnt * n, *tmp = m + cnt * n;
    const bool async = is_pinned(slots);
    int j = 0;
    if (async) {
        // pinned input: H2D on the copy stream into staging slot j, the compute stream waits
        j = c->io_in_next;
        c->io_in_next = (j + 1) % fhe_ctx::NIO;
        TRY(ensure_stage(c, &c->io_in[j], &c->io_in_words[j], cnt * n));
        s_dev = c->io_in[j];
        CU(cudaStreamWaitEvent(c->h2d, c->ev_in_free[j], 0));
        CU(cudaMemcpyAsync(s_dev, slots, cnt * n * 8, cudaMemcpyHostToDevice, c->h2d));
        CU(cudaEventRecord(c->ev_in_ready[j], c->h2d));
        CU(cudaStreamWaitEvent(c->st, c->ev_in_ready[j], 0));
    } else {
        CU(cudaMemcpyAsync(s_dev, slots, cnt * n * 8, cudaMemcpyHostToDevice, c->st));
    }
    TRY(slots_to_coef(c, s_dev, m, (int)cnt, ct->R));
    if (async) CU(cudaEventRecord(c->ev_in_free[j], c->st));
    const long long total8 = (long long)cnt * ((n + 7) / 8);
    EW(k_enc_prep, total8, m, tmp, total8, (int)L, (int)ct->R, (int)c->logn, c->P.seed, nonce, c->d_lv + L, c->t_id0,
       c->d_mods);
    CHECK_LAUNCH();
    // NTT of every (ci, i) row, the uniform a and c0 = v - a s in its epilogue (epi 3)
    NttRowsArgs a = nargs(tmp, ct->d, n);
    a.period = L;
    map_q(a.map, L);
    a.rdiv = (u32)L;
    a.sA = (long long)L * n; a.sB = (long long)n;
    a.dA = (long long)2 * L * n; a.dB = (long long)n;
    a.epi = 3;
    a.seed = c->P.seed;
    a.nonce = nonce;
    a.s_m = c->d_s_m;
    a.c1off = (long long)L * n;
    TRY(ntt_rows(c, (int)(cnt * L), a));
    if (!async) CU(cudaStreamSynchronize(c->st));      // pageable input: the host buffer may be reused
    return 0;
}

// x = INTT(c0 + c1 s) into dst [count][l][n]
static int raw_decrypt(fhe_ctx *c, const fhe_ct *ct, u64 *dst) {
    size_t n = c->n, l = ct->level;
    // row r = (ci, i): c0 + c1 s computed while staging the inverse NTT (gather mode 3)
    InttRowsArgs a = iargs(ct->d, dst, n);
    a.rdiv = (u32)l;
    a.sA = (long long)2 * l * n; a.sB = (long long)n;
    a.dA = (long long)l * n; a.dB = (long long)n;
    a.period = l;
    map_q(a.map, l);
    a.gather = 3;
    a.c1off = (long long)l * n;
    a.s_m = c->d_s_m;
    return intt_rows(c, (int)(ct->count * l), a);
}

// decrypted slot values mod t_k in NTT order, [cnt][n], into m (scratch X: [cnt][l][n])
static int decode_ntt_order(fhe_ctx *c, const fhe_ct *ct, u64 *X, u64 *m) {
    size_t n = c->n, l = ct->level, cnt = ct->count;
    TRY(raw_decrypt(c, ct, X));
    long long total = (long long)cnt * n;
    EW(k_dec_scale, total, X, m, total, (int)l, (int)ct->R, (int)c->logn, c->d_lv + l, c->t_id0, c->d_mods,
       c->d_status);
    CHECK_LAUNCH();
    NttRowsArgs a = nargs(m, m, n);
    a.div = ct->R;
    a.period = c->T;
    map_range(a.map, c->T, c->t_id0);
    return ntt_rows(c, (int)cnt, a);
}

extern "C" int fhe_decrypt(fhe_ctx *c, const fhe_ct *ct, uint64_t *slots) {
    size_t n = c->n, l = ct->level, cnt = ct->count;
    TRY(ensure_tmp(c, cnt * n * (l + 2)));
    u64 *X = c->w_tmp, *m = X + cnt * l * n, *o = m + cnt * n;
    TRY(decode_ntt_order(c, ct, X, m));
    long long total = (long long)cnt * n;
    if (is_pinned(slots)) {
        // pinned output: gather into staging slot j, D2H on the copy stream; valid after fhe_sync
        const int j = c->io_out_next;
        c->io_out_next = (j + 1) % fhe_ctx::NIO;
        TRY(ensure_stage(c, &c->io_out[j], &c->io_out_words[j], cnt * n));
        CU(cudaStreamWaitEvent(c->st, c->ev_out_free[j], 0));
        EW(k_gather_slots, total, m, c->io_out[j], total, (int)c->logn, c->d_slot2ntt);
        CHECK_LAUNCH();
        CU(cudaEventRecord(c->ev_out_ready[j], c->st));
        CU(cudaStreamWaitEvent(c->d2h, c->ev_out_ready[j], 0));
        CU(cudaMemcpyAsync(slots, c->io_out[j], cnt * n * 8, cudaMemcpyDeviceToHost, c->d2h));
        CU(cudaEventRecord(c->ev_out_free[j], c->d2h));
        return 0;
    }
    EW(k_gather_slots, total, m, o, total, (int)c->logn, c->d_slot2ntt);
    CHECK_LAUNCH();
    CU(cudaMemcpyAsync(slots, o, cnt * n * 8, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    return 0;
}

extern "C" int fhe_decrypt_slots(fhe_ctx *c, const fhe_ct *ct, uint32_t lo, uint32_t cnt, uint64_t *out) {
    if ((u64)lo + cnt > c->N) return fail(FHE_EINVAL, "decrypt_slots: [%u, %u) exceeds %u slots", lo, lo + cnt, c->N);
    if (!cnt) return 0;
    size_t n = c->n, l = ct->level, nct = ct->count;
    TRY(ensure_tmp(c, nct * n * (l + 1) + nct * 2 * cnt));
    u64 *X = c->w_tmp, *m = X + nct * l * n, *o = m + nct * n;
    TRY(decode_ntt_order(c, ct, X, m));
    const long long total = (long long)nct * 2 * cnt;
    EW(k_gather_slot_range, total, m, o, total, (int)c->logn, lo, cnt, c->d_slot2ntt);
    CHECK_LAUNCH();
    CU(cudaMemcpyAsync(out, o, total * 8, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    return 0;
}

extern "C" int fhe_check_zero_tail(fhe_ctx *c, const fhe_ct *ct, uint32_t m) {
    if (m > c->N) return fail(FHE_EINVAL, "check_zero_tail: m = %u exceeds %u slots", m, c->N);
    if (m == c->N) return 0;
    size_t n = c->n, l = ct->level, cnt = ct->count;
    TRY(ensure_tmp(c, cnt * n * (l + 1)));
    u64 *X = c->w_tmp, *mc = X + cnt * l * n;
    TRY(decode_ntt_order(c, ct, X, mc));
    long long total = (long long)cnt * n;
    EW(k_tail_check, total, mc, total, (int)c->logn, m, c->d_ntt2slot, c->d_status + 1);
    CHECK_LAUNCH();
    return 0;
}

extern "C" int fhe_status(fhe_ctx *c, uint32_t *noise_dist, uint32_t *flags, int reset) {
    u32 h[2];
    CU(cudaStreamSynchronize(c->st));
    CU(cudaMemcpy(h, c->d_status, sizeof h, cudaMemcpyDeviceToHost));
    if (reset) CU(cudaMemset(c->d_status, 0, sizeof h));
    if (noise_dist) *noise_dist = h[0];
    if (flags) *flags = h[1];
    return 0;
}

extern "C" int fhe_decrypt_raw(fhe_ctx *c, const fhe_ct *ct, uint64_t *out) {
    size_t words = (size_t)ct->count * ct->level * c->n;
    TRY(ensure_tmp(c, words));
    TRY(raw_decrypt(c, ct, c->w_tmp));
    CU(cudaMemcpyAsync(out, c->w_tmp, words * 8, cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    return 0;
}

// =============================================================== evaluation
static bool same_shape(const fhe_ct *a, const fhe_ct *b) { return a->R == b->R && a->level == b->level; }

extern "C" int fhe_add(fhe_ctx *c, const fhe_ct *a, const fhe_ct *b, fhe_ct *out) {
    if (!same_shape(a, b) || !same_shape(a, out)) return fail(FHE_ELEVEL, "add: shape/level mismatch");
    long long total = (long long)ct_words(a);
    EW(k_add, total, a->d, b->d, out->d, total, (int)a->level, (int)c->logn, c->d_mods);
    CHECK_LAUNCH();
    return 0;
}

static int mul_plain_rows(fhe_ctx *c, const fhe_ct *a, const fhe_pt *pt, fhe_ct *out, const u64 *acc) {
    const int rows = (int)(a->count * 2 * a->level);
    const unsigned bx = (unsigned)std::max<size_t>(1, (c->n / 2 + 255) / 256);
    dim3 grid(bx, (unsigned)std::min(rows, 65535));
    ProfScope ps_(c, "k_mul_plain");
    k_mul_plain<<<grid, 256, 0, c->st>>>(a->d, pt->ntt_m, out->d, acc, rows, (int)a->level, (int)c->L, (int)a->R,
                                        (int)c->logn, c->d_mods);
    CHECK_LAUNCH();
    return 0;
}

extern "C" int fhe_mul_plain(fhe_ctx *c, const fhe_ct *a, const fhe_pt *pt, fhe_ct *out) {
    if (!same_shape(a, out)) return fail(FHE_ELEVEL, "mul_plain: shape/level mismatch");
    if (!pt->encoded) return fail(FHE_EINVAL, "mul_plain: plaintext was never encoded");
    return mul_plain_rows(c, a, pt, out, nullptr);
}

extern "C" int fhe_mul_plain_acc(fhe_ctx *c, const fhe_ct *a, const fhe_pt *pt, fhe_ct *acc) {
    if (!same_shape(a, acc)) return fail(FHE_ELEVEL, "mul_plain_acc: shape/level mismatch");
    if (!pt->encoded) return fail(FHE_EINVAL, "mul_plain_acc: plaintext was never encoded");
    if (a == acc) return fail(FHE_EINVAL, "mul_plain_acc: the accumulator must not alias the input");
    return mul_plain_rows(c, a, pt, acc, acc->d);
}

extern "C" int fhe_mul_scalar(fhe_ctx *c, const fhe_ct *a, int64_t w, fhe_ct *out) {
    if (!same_shape(a, out)) return fail(FHE_ELEVEL, "mul_scalar: shape/level mismatch");
    ScalarTab st;
    memset(&st, 0, sizeof st);
    for (u32 i = 0; i < a->level; i++) {
        u64 q = c->P.q[i];
        u64 v = w >= 0 ? (u64)w % q : hm::neg((u64)(-(w + 1)) % q + 1, q);
        st.w[i] = v;
        st.wsh[i] = hm::shoup(v, q);
    }
    long long total = (long long)ct_words(a);
    EW(k_mul_scalar, total, a->d, out->d, total, (int)a->level, (int)c->logn, st, c->d_mods);
    CHECK_LAUNCH();
    return 0;
}

extern "C" int fhe_add_plain(fhe_ctx *c, const fhe_ct *a, const fhe_pt *pt, fhe_ct *out) {
    if (!same_shape(a, out)) return fail(FHE_ELEVEL, "add_plain: shape/level mismatch");
    if (!pt->encoded) return fail(FHE_EINVAL, "add_plain: plaintext was never encoded");
    size_t n = c->n, l = a->level;
    TRY(ensure_tmp(c, c->T * l * n));
    long long total = (long long)c->T * l * n;
    EW(k_scaled_msg, total, pt->coef_t, c->w_tmp, total, (int)l, 1, (int)c->logn, c->d_lv + l, c->t_id0, c->d_mods);
    CHECK_LAUNCH();
    NttRowsArgs na = nargs(c->w_tmp, c->w_tmp, n);
    na.period = l;
    map_q(na.map, l);
    TRY(ntt_rows(c, (int)(c->T * l), na));
    long long tw = (long long)ct_words(a);
    EW(k_add_pt, tw, a->d, c->w_tmp, out->d, tw, (int)l, (int)a->R, (int)c->logn, c->d_mods);
    CHECK_LAUNCH();
    return 0;
}

// ---------------------------------------------------------- key switching
// Digits of S cts: dt.coef[s] + j n (coefficient form), dt.ntt[s] + j n (NTT
// form).  Result: out[s][p][i] = ModDown(sum_j digit_j * key_j)[p][i] + add[s][p][i].
struct KsOut {
    u64 *out[MAXS];
    const u64 *add[MAXS];
    long long out_pstride, add_pstride;
    int add_pmask;
    u32 add_g[MAXS];
    const u64 *acc[MAXS];      // rotate-and-add: the input ct, added to both polys
    long long acc_pstride;
};

// ModUp: every off-diagonal (digit, prime) pair of S cts into Ext
template <int LOGN>
static void launch_modup_persist(fhe_ctx *c, int S, u32 l, const DigitTab &dt) {
    static int sms = 0;
    if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->dev);
    const int rows = S * (int)(l * l);
    launch_row<LOGN, false, FwdW5<LOGN>::value>(c, "k_modup", k_modup_persist<LOGN>, dim3(std::min(rows, sms)), c->st,
                                                 dt, c->w_Ext, (int)l, c->special_id, rows, c->d_mods);
    c->alg_mm += (double)(rows - std::min(rows, sms)) * (c->n / 2) * c->logn;   // launch_row counted one row per CTA
}

static int keyswitch_modup(fhe_ctx *c, int S, u32 l, const DigitTab &dt) {
    static int persist = -1;     // FHE_MODUP_PERSIST: persistent ModUp CTAs (single-CTA rows)
    if (persist < 0) { const char *e = getenv("FHE_MODUP_PERSIST"); persist = e ? atoi(e) : 1; }
    if (persist && c->logn <= 14 && c->logn >= 12 && c->logn <= NTT_LOGL) {
        if (c->logn == 14) launch_modup_persist<14>(c, S, l, dt);
        else if (c->logn == 13) launch_modup_persist<13>(c, S, l, dt);
        else launch_modup_persist<12>(c, S, l, dt);
        CHECK_LAUNCH();
        return 0;
    }
    c->alg_mm -= (double)S * l * (c->n / 2) * c->logn;      // the diagonal rows return at once
    LOGN_SWITCH(c->logn, launch_row<LG, false, FwdW5<LG>::value>(c, "k_modup", k_modup<LG>, dim3(S, l, l + 1), c->st, dt, c->w_Ext, (int)l, c->special_id,
                                        c->d_mods));
    CHECK_LAUNCH();
    return 0;
}

// inner product with the keys + ModDown (+ epilogue adds) for S items whose extended
// digits are in Ext (item s reads block s, or dt.esrc[s] through dt.perm[s])
static int keyswitch_tail(fhe_ctx *c, int S, u32 l, const DigitTab &dt, const KsOut &ko) {
    size_t n = c->n;
    int L = (int)c->L;
    // inner-product variant, env FHE_KS_VARIANT (profiles/r02_subbatch.json):
    //   0..3  register keys: (4 cts/thread, 1 CTA/SM min), (2, 1), (4, 4) [the round-2 default until the
    //         last session], (2, 4)
    //   6     key words in the thread's own shared-memory column, 8 cts/thread, 5 CTAs/SM
    //   7, 9  shared-memory keys + the next ciphertext's digits prefetched (two operand sets in flight),
    //         4 CTAs/SM, 8 / 16 cts/thread.  9 is the default: k_ks_inner -6 % at configs[1] (164.1K vs
    //         162.1K rot/s), -11 % at configs[2] (7.44 vs 7.12 images/s on the same box)
    // Levels above 12 (more than 48 KB of static shared memory) use variant 2.
    static int ksv = -1;
    if (ksv < 0) { const char *e = getenv("FHE_KS_VARIANT"); ksv = e ? atoi(e) : 9; }
    const bool ksm = (ksv == 6 || ksv == 7 || ksv == 9) && l <= 12;
    const int G = ksm ? (ksv == 9 ? 16 : 8) : (ksv == 1 || ksv == 3) ? 2 : 4;
    c->alg_mm += (double)S * (2.0 * l * (l + 1) + 2.0 * l) * n;   // key inner product + ModDown scaling
    long long tot = (long long)((S + G - 1) / G) * l * n;
    // fold the addends into the inner product while its Montgomery input bound holds
    // ((l + 2) q_i < 2^64: l digit terms + 2 addend terms, each < q_i^2); else the
    // rescale epilogue adds them
    u64 maxq = 0;
    for (u32 i = 0; i < l; i++) maxq = std::max<u64>(maxq, c->P.q[i]);
    const bool fold = (u128)(l + 2) * maxq < ((u128)1 << 64);
    KsAdd kad;
    memset(&kad, 0, sizeof kad);
    // Both addends fold into the inner product.  FHE_FOLD_ACC=0 leaves the rotate-and-add
    // addend (the input ciphertext, no automorphism) to the ModDown epilogue instead: measured
    // equal in kernel time (k_ks_inner -177 ms, k_rescale +178 ms per configs[2] chunk) and
    // 2.6 % slower overall.
    static int fold_acc = -1, fused_env = -1;
    if (fused_env < 0) { const char *e = getenv("FHE_FUSED_MODDOWN"); fused_env = e ? atoi(e) : 0; }
    if (fold_acc < 0) { const char *e = getenv("FHE_FOLD_ACC"); fold_acc = (e ? atoi(e) : 1) || fused_env; }   // k_moddown folds both
    if (fold) {
        for (int s = 0; s < S; s++) { kad.add[s] = ko.add[s]; kad.add_g[s] = ko.add_g[s]; kad.acc[s] = fold_acc ? ko.acc[s] : nullptr; }
        kad.add_pstride = ko.add_pstride;
        kad.acc_pstride = ko.acc_pstride;
        kad.add_pmask = ko.add_pmask;
        for (u32 i = 0; i < l; i++) kad.pr[i] = c->pmont[i];
    }
    // FHE_FUSED_MODDOWN=1: the q primes' inner product runs in k_moddown's epilogue instead
    // of a separate k_ks_inner pass (needs the addend fold).  Off by default: measured 3 %
    // slower (the epilogue serialises behind the NTT in each CTA)
    const bool fused = fold && fused_env != 0;
    if (!fused) {
        ProfScope ps_(c, "k_ks_inner");
        const unsigned nb = (unsigned)nblocks(tot);
#define KS_LAUNCH(LLV, GV, MB) k_ks_inner<LLV, GV, MB><<<nb, 256, 0, c->st>>>(c->w_Ext, dt, c->w_Acc, S, L, \
                                                        (int)c->logn, c->special_id, c->d_mods, kad)
#define KS_LAUNCH_SM(LLV, GV, MB, PFV) k_ks_inner<(LLV <= 12 ? LLV : 1), GV, MB, true, PFV><<<nb, 256, 0, c->st>>>(c->w_Ext, dt, c->w_Acc, S, L, \
                                                        (int)c->logn, c->special_id, c->d_mods, kad)
#define KS_CASE(LLV) case LLV:                                        \
        if (ksm && ksv == 7) KS_LAUNCH_SM(LLV, 8, 4, true);           \
        else if (ksm && ksv == 9) KS_LAUNCH_SM(LLV, 16, 4, true);     \
        else if (ksm) KS_LAUNCH_SM(LLV, 8, 5, false);                 \
        else if (ksv == 1) KS_LAUNCH(LLV, 2, 1);                      \
        else if (ksv == 3) KS_LAUNCH(LLV, 2, 4);                      \
        else if (ksv == 0) KS_LAUNCH(LLV, 4, 1);                      \
        else KS_LAUNCH(LLV, 4, 4);                                    \
        break;
        switch (l) {
            KS_CASE(1) KS_CASE(2) KS_CASE(3) KS_CASE(4) KS_CASE(5) KS_CASE(6) KS_CASE(7) KS_CASE(8)
            KS_CASE(9) KS_CASE(10) KS_CASE(11) KS_CASE(12) KS_CASE(13) KS_CASE(14) KS_CASE(15) KS_CASE(16)
            KS_CASE(17) KS_CASE(18) KS_CASE(19) KS_CASE(20) KS_CASE(21) KS_CASE(22) KS_CASE(23) KS_CASE(24)
            default: return fail(FHE_EINVAL, "level %u unsupported by k_ks_inner", l);
        }
#undef KS_CASE
#undef KS_LAUNCH
#undef KS_LAUNCH_SM
    }
    CHECK_LAUNCH();
    // the special prime's inner product + ModDown INTT of both accumulators (one row each)
    LOGN_SWITCH(c->logn, launch_row<LG, true>(c, "k_ks_special", k_ks_special<LG>, dim3(2 * S), c->st,
                                              (const u64 *)c->w_Ext, dt, c->w_Acc, (int)l, L, c->special_id, c->d_mods));
    CHECK_LAUNCH();
    RescaleArgs ra;
    memset(&ra, 0, sizeof ra);
    for (int s = 0; s < S; s++) {
        ra.coef[s] = c->w_Acc + ((size_t)s * 2 * (l + 1) + l) * n;
        ra.base[s] = c->w_Acc + (size_t)s * 2 * (l + 1) * n;
        ra.out[s] = ko.out[s];
        if (!fold) { ra.add[s] = ko.add[s]; ra.add_g[s] = ko.add_g[s]; }
        if (!fold || !fold_acc) ra.acc[s] = ko.acc[s];
    }
    ra.coef_pstride = (long long)(l + 1) * n;
    ra.base_pstride = (long long)(l + 1) * n;
    ra.out_pstride = ko.out_pstride;
    if (!fold) {
        ra.add_pstride = ko.add_pstride;
        ra.add_pmask = ko.add_pmask;
    }
    ra.acc_pstride = ko.acc_pstride;
    ra.src_id = c->special_id;
    for (u32 i = 0; i < l; i++) { ra.fac[i] = c->pinv[i]; ra.fac_sh[i] = c->pinv_sh[i]; }
    if (fused) {
        LOGN_SWITCH(c->logn, launch_row<LG, false, RescaleW<LG>::value>(c, "k_moddown", k_moddown<LG>, dim3(S, 2, l), c->st, ra,
                                                                        (const u64 *)c->w_Ext, dt, kad, (int)l, L, c->d_mods));
    } else {
        LOGN_SWITCH(c->logn, launch_row<LG, false, RescaleW<LG>::value>(c, "k_rescale(moddown)", k_rescale<LG>, dim3(S, 2, l), c->st, ra, c->d_mods));
    }
    CHECK_LAUNCH();
    return 0;
}

// ModUp fused into the key inner product (ks_fused.cuh): extended digits stay on
// chip, accumulators in TMEM; then the ModDown rescale.  Single-CTA rows of
// 2^9 .. 2^14 words, digits read in natural order (not the hoisted Ext path).
template <int LOGN>
static void launch_ks_fused(fhe_ctx *c, int S, u32 l, const DigitTab &dt, const KsAdd &kad) {
    using F = KsfCfg<LOGN>;
    using C = typename F::C;
    const size_t smem = (size_t)C::SMEM_WORDS * sizeof(u64);
    auto kern = k_ks_fused<LOGN>;
    {
        std::lock_guard<std::mutex> lk(g_attr_mu);
        if (!g_attr_done.count((const void *)kern)) {
            cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            g_attr_done.insert((const void *)kern);
        }
    }
    ProfScope ps_(c, "k_ks_fused");
    const unsigned items = (unsigned)(S * (l + 1));
    if constexpr (C::CR == 1) {
        kern<<<items, F::TH, smem, c->st>>>(dt, c->w_Acc, S, (int)l, (int)c->L, c->special_id, c->d_mods, kad);
    } else {
        // one thread-block cluster of CR CTAs per (ciphertext, prime): each CTA owns 2^14
        // words of the row and their accumulators in its TMEM
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(items * C::CR);
        cfg.blockDim = dim3(F::TH);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = c->st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C::CR;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, dt, c->w_Acc, S, (int)l, (int)c->L, c->special_id, (const ModInfo *)c->d_mods, kad);
    }
}

// FHE_KS_FUSED=1 selects the fused path.  Off by default: bit-exact, but measured slower
// at configs[1] (127 K vs 150 K rotations/s) -- the TMEM accumulators
// hold 64 bits per word, so every product needs its own Montgomery reduction, where
// k_ks_inner accumulates l products in 128 bits and reduces once.
static bool ks_fused_ok(const fhe_ctx *c) {
    const char *e = getenv("FHE_KS_FUSED");
    return e && atoi(e) && c->logn >= 9 && c->logn <= 16;
}

static int keyswitch_fused(fhe_ctx *c, int S, u32 l, const DigitTab &dt, const KsOut &ko) {
    const size_t n = c->n;
    KsAdd kad;
    memset(&kad, 0, sizeof kad);
    for (int s = 0; s < S; s++) { kad.add[s] = ko.add[s]; kad.add_g[s] = ko.add_g[s]; kad.acc[s] = ko.acc[s]; }
    kad.add_pstride = ko.add_pstride;
    kad.acc_pstride = ko.acc_pstride;
    kad.add_pmask = ko.add_pmask;
    for (u32 i = 0; i < l; i++) kad.pr[i] = c->pmont[i];
    // l^2 ModUp transforms + 2 special-prime inverses per ciphertext, key inner product + ModDown scaling
    c->alg_mm += (double)S * ((double)(l * l + 2) * (n / 2) * c->logn + (2.0 * l * (l + 1) + 2.0 * l) * n);
    switch (c->logn) {
        case 9: launch_ks_fused<9>(c, S, l, dt, kad); break;
        case 10: launch_ks_fused<10>(c, S, l, dt, kad); break;
        case 11: launch_ks_fused<11>(c, S, l, dt, kad); break;
        case 12: launch_ks_fused<12>(c, S, l, dt, kad); break;
        case 13: launch_ks_fused<13>(c, S, l, dt, kad); break;
        case 14: launch_ks_fused<14>(c, S, l, dt, kad); break;
        case 15: launch_ks_fused<15>(c, S, l, dt, kad); break;
        case 16: launch_ks_fused<16>(c, S, l, dt, kad); break;
        default: return fail(FHE_EINVAL, "fused key switching needs 2^9 <= n <= 2^16");
    }
    CHECK_LAUNCH();
    // the special prime's accumulators to coefficient form, in place: row r = (s, p)
    InttRowsArgs ia = iargs(c->w_Acc + (size_t)l * n, c->w_Acc + (size_t)l * n, 0);
    ia.rdiv = 2;
    ia.sA = ia.dA = (long long)2 * (l + 1) * n;
    ia.sB = ia.dB = (long long)(l + 1) * n;
    ia.map.id[0] = (unsigned char)c->special_id;
    c->alg_mm -= (double)2 * S * (n / 2) * c->logn;            // counted above
    TRY(intt_rows(c, 2 * S, ia, "k_intt_rows(ks_special)"));
    RescaleArgs ra;
    memset(&ra, 0, sizeof ra);
    for (int s = 0; s < S; s++) {
        ra.coef[s] = c->w_Acc + ((size_t)s * 2 * (l + 1) + l) * n;
        ra.base[s] = c->w_Acc + (size_t)s * 2 * (l + 1) * n;
        ra.out[s] = ko.out[s];
    }
    ra.coef_pstride = (long long)(l + 1) * n;
    ra.base_pstride = (long long)(l + 1) * n;
    ra.out_pstride = ko.out_pstride;
    ra.src_id = c->special_id;
    for (u32 i = 0; i < l; i++) { ra.fac[i] = c->pinv[i]; ra.fac_sh[i] = c->pinv_sh[i]; }
    LOGN_SWITCH(c->logn, launch_row<LG, false, RescaleW<LG>::value>(c, "k_rescale(moddown)", k_rescale<LG>, dim3(S, 2, l), c->st, ra, c->d_mods));
    CHECK_LAUNCH();
    return 0;
}

static int keyswitch_core(fhe_ctx *c, int S, u32 l, const DigitTab &dt, const KsOut &ko) {
    if (ks_fused_ok(c)) return keyswitch_fused(c, S, l, dt, ko);
    TRY(keyswitch_modup(c, S, l, dt));
    return keyswitch_tail(c, S, l, dt, ko);
}

// rotate a list of physical ciphertexts (each [2][l][n]) by Galois element g
static void use_lane(fhe_ctx *c, int k) {
    c->st = c->streams[k];
    c->w_D = c->ws_D[k]; c->w_Ext = c->ws_Ext[k]; c->w_Acc = c->ws_Acc[k];
}

// rotate a list of physical ciphertexts (each [2][l][n]), ciphertext i by
// Galois element g[i].  Sub-batches alternate between two streams with their
// own workspaces so the small-grid steps of one (ModDown INTT) overlap the
// next one's ModUp.
// addend: when non-null, addend[i] ([2][l][n], e.g. the input itself for a rotate-and-sum
// level, or the left block of a combine merge) is added to output i in the epilogue.
static int rotate_phys(fhe_ctx *c, const std::vector<const u64 *> &in, const std::vector<u64 *> &out, u32 l,
                       const std::vector<u32> &g, const std::vector<const u64 *> *addend = nullptr) {
    std::vector<const u64 *> keys(in.size());
    size_t n = c->n;
    // (profiling runs single-stream so every kernel is timed in isolation)
    // balanced sub-batches: ceil(count / ceil(count / S)) instead of S + remainder
    size_t Smax = c->S;
    if (ks_fused_ok(c) && !getenv("FHE_KS_BATCH")) {
        // fused path: one CTA per (ciphertext, prime), S (l + 1) CTAs per launch -- the
        // largest S whose launch fills whole waves of the SMs best
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->dev);
        double best = 0;
        for (int s = c->S; s >= std::max(1, c->S / 2); s--) {
            const int blocks = s * (int)(l + 1), waves = (blocks + sms - 1) / sms;
            const double eff = (double)blocks / ((double)waves * sms);
            if (eff > best + 0.02) { best = eff; Smax = (size_t)s; }
        }
    }
    const bool two = in.size() > Smax && !c->prof && c->lanes > 1;
    const size_t nsub = (in.size() + Smax - 1) / Smax;
    const size_t SB = (in.size() + nsub - 1) / nsub;
    if (two) {
        CU(cudaEventRecord(c->ev_fork, c->streams[0]));
        for (int k = 1; k < c->lanes; k++) CU(cudaStreamWaitEvent(c->streams[k], c->ev_fork, 0));
    }
    int rc = 0;
    int lane = 0;
    for (size_t b0 = 0; b0 < in.size() && !rc; b0 += SB, lane = (lane + 1) % c->lanes) {
        use_lane(c, two ? lane : 0);
        int S = (int)std::min<size_t>(SB, in.size() - b0);
        c->key_tick++;                       // keys of this sub-batch are pinned
        for (size_t i = b0; i < b0 + S && !rc; i++) {
            if (i > b0 && g[i] == g[i - 1]) { keys[i] = keys[i - 1]; continue; }
            rc = get_key(c, g[i], &keys[i]);
        }
        if (rc) break;
        PtrTab pt;
        memset(&pt, 0, sizeof pt);
        for (int s = 0; s < S; s++) { pt.in[s] = in[b0 + s]; pt.out[s] = out[b0 + s]; pt.g[s] = g[b0 + s]; }
        LOGN_SWITCH(c->logn, launch_row<LG, true>(c, "k_rot_gather_intt", k_rot_gather_intt<LG>, dim3(S, l), c->st,
                                                  pt, (int)l, c->w_D, c->d_mods));
        if (cudaGetLastError() != cudaSuccess) { rc = fail(FHE_EDEVICE, "k_rot_gather_intt launch failed"); break; }
        DigitTab dt;
        KsOut ko;
        memset(&dt, 0, sizeof dt);
        memset(&ko, 0, sizeof ko);
        for (int s = 0; s < S; s++) {
            dt.coef[s] = c->w_D + (size_t)s * l * n;
            dt.ntt[s] = in[b0 + s] + (size_t)l * n;      // c1 limbs, read through the automorphism
            dt.dperm[s] = g[b0 + s];
            dt.key[s] = keys[b0 + s];
            ko.out[s] = out[b0 + s];
            ko.add[s] = in[b0 + s];          // c0 limbs, read through the automorphism
            ko.add_g[s] = g[b0 + s];
            ko.acc[s] = addend ? (*addend)[b0 + s] : nullptr;
        }
        ko.acc_pstride = (long long)l * n;
        ko.out_pstride = (long long)l * n;
        ko.add_pstride = 0;
        ko.add_pmask = 1;
        rc = keyswitch_core(c, S, l, dt, ko);
    }
    use_lane(c, 0);
    if (two) {
        for (int k = 1; k < c->lanes; k++) {
            CU(cudaEventRecord(c->ev_join[k], c->streams[k]));
            CU(cudaStreamWaitEvent(c->streams[0], c->ev_join[k], 0));
        }
    }
    return rc;
}

static int check_rot(fhe_ctx *c, u32 k) {
    if (k == 0 || k >= c->N) return fail(FHE_EINVAL, "rotation step %u outside [1, %u)", k, c->N);
    return 0;
}

// Test access to the stages of a rotation's key switch: the product pipeline (gather + INTT,
// ModUp, inner products, special-row INTT) on one sub-batch, without the c0 addend, with the
// workspaces copied out (ffconv_he.h: fhe_debug_rotate_stages).
extern "C" int fhe_debug_rotate_stages(fhe_ctx *c, const fhe_ct *a, uint32_t k, uint64_t *digits, uint64_t *ext,
                                       uint64_t *acc) {
    TRY(check_rot(c, k));
    if (ks_fused_ok(c)) return fail(FHE_EINVAL, "debug_rotate_stages: the fused key switch keeps no stages");
    const int S = (int)a->count;
    if (S > c->S) return fail(FHE_EINVAL, "debug_rotate_stages: at most %d physical ciphertexts", c->S);
    const u32 l = a->level, g = galois_elt(c, k);
    const size_t n = c->n, stride = 2ull * l * n;
    use_lane(c, 0);
    const u64 *key;
    c->key_tick++;
    TRY(get_key(c, g, &key));
    fhe_ct *scratch = nullptr;
    TRY(fhe_ct_create(c, a->R, l, &scratch));
    PtrTab pt;
    memset(&pt, 0, sizeof pt);
    for (int s = 0; s < S; s++) { pt.in[s] = a->d + s * stride; pt.out[s] = scratch->d + s * stride; pt.g[s] = g; }
    LOGN_SWITCH(c->logn, launch_row<LG, true>(c, "k_rot_gather_intt", k_rot_gather_intt<LG>, dim3(S, l), c->st,
                                              pt, (int)l, c->w_D, c->d_mods));
    DigitTab dt;
    KsOut ko;
    memset(&dt, 0, sizeof dt);
    memset(&ko, 0, sizeof ko);
    for (int s = 0; s < S; s++) {
        dt.coef[s] = c->w_D + (size_t)s * l * n;
        dt.ntt[s] = a->d + s * stride + (size_t)l * n;
        dt.dperm[s] = g;
        dt.key[s] = key;
        ko.out[s] = scratch->d + s * stride;
    }
    ko.out_pstride = (long long)l * n;
    ko.add_pmask = 0;
    cudaMemsetAsync(c->w_Ext, 0, (size_t)S * l * (l + 1) * n * 8, c->st);      // the diagonal stays zero
    int rc = keyswitch_modup(c, S, l, dt);
    if (!rc) rc = keyswitch_tail(c, S, l, dt, ko);
    if (!rc) {
        cudaMemcpyAsync(digits, c->w_D, (size_t)S * l * n * 8, cudaMemcpyDeviceToHost, c->st);
        cudaMemcpyAsync(ext, c->w_Ext, (size_t)S * l * (l + 1) * n * 8, cudaMemcpyDeviceToHost, c->st);
        cudaMemcpyAsync(acc, c->w_Acc, (size_t)S * 2 * (l + 1) * n * 8, cudaMemcpyDeviceToHost, c->st);
        if (cudaStreamSynchronize(c->st) != cudaSuccess) rc = fail(FHE_EDEVICE, "debug_rotate_stages: copy failed");
    }
    fhe_ct_destroy(scratch);
    if (rc) return rc;
    // ModUp leaves lazy representatives (< B q): canonical form for the comparison
    for (int s = 0; s < S; s++)
        for (u32 j = 0; j < l; j++)
            for (u32 i = 0; i <= l; i++) {
                const u64 q = i == l ? c->P.p[0] : c->P.q[i];
                u64 *row = ext + (((size_t)s * l + j) * (l + 1) + i) * n;
                for (size_t x = 0; x < n; x++) row[x] %= q;
            }
    return 0;
}

extern "C" int fhe_rotate(fhe_ctx *c, const fhe_ct *a, uint32_t k, fhe_ct *out) {
    TRY(check_rot(c, k));
    if (!same_shape(a, out)) return fail(FHE_ELEVEL, "rotate: shape/level mismatch");
    if (a == out || a->d == out->d) return fail(FHE_EINVAL, "rotate: out must not alias the input");
    std::vector<const u64 *> in;
    std::vector<u64 *> o;
    size_t stride = 2ull * a->level * c->n;
    for (u32 ci = 0; ci < a->count; ci++) { in.push_back(a->d + ci * stride); o.push_back(out->d + ci * stride); }
    return rotate_phys(c, in, o, a->level, std::vector<u32>(in.size(), galois_elt(c, k)));
}

extern "C" int fhe_rotate_many(fhe_ctx *c, fhe_ct *const *a, fhe_ct *const *out, uint32_t m, uint32_t k) {
    TRY(check_rot(c, k));
    if (!m) return 0;
    u32 l = a[0]->level;
    std::vector<const u64 *> in;
    std::vector<u64 *> o;
    for (u32 h = 0; h < m; h++) {
        if (a[h]->level != l || !same_shape(a[h], out[h])) return fail(FHE_ELEVEL, "rotate_many: shape/level mismatch");
        if (a[h]->d == out[h]->d) return fail(FHE_EINVAL, "rotate_many: out must not alias the input");
        size_t stride = 2ull * l * c->n;
        for (u32 ci = 0; ci < a[h]->count; ci++) { in.push_back(a[h]->d + ci * stride); o.push_back(out[h]->d + ci * stride); }
    }
    return rotate_phys(c, in, o, l, std::vector<u32>(in.size(), galois_elt(c, k)));
}

extern "C" int fhe_rotate_add_many(fhe_ctx *c, fhe_ct *const *a, fhe_ct *const *out, uint32_t m, uint32_t k) {
    TRY(check_rot(c, k));
    if (!m) return 0;
    u32 l = a[0]->level;
    std::vector<const u64 *> in;
    std::vector<u64 *> o;
    for (u32 h = 0; h < m; h++) {
        if (a[h]->level != l || !same_shape(a[h], out[h])) return fail(FHE_ELEVEL, "rotate_add_many: shape/level mismatch");
        if (a[h]->d == out[h]->d) return fail(FHE_EINVAL, "rotate_add_many: out must not alias the input");
        size_t stride = 2ull * l * c->n;
        for (u32 ci = 0; ci < a[h]->count; ci++) { in.push_back(a[h]->d + ci * stride); o.push_back(out[h]->d + ci * stride); }
    }
    return rotate_phys(c, in, o, l, std::vector<u32>(in.size(), galois_elt(c, k)), &in);
}

extern "C" int fhe_rotate_multi(fhe_ctx *c, fhe_ct *const *a, fhe_ct *const *out, const uint32_t *k, uint32_t m) {
    if (!m) return 0;
    u32 l = a[0]->level;
    std::vector<const u64 *> in;
    std::vector<u64 *> o;
    std::vector<u32> g;
    for (u32 h = 0; h < m; h++) {
        TRY(check_rot(c, k[h]));
        if (a[h]->level != l || !same_shape(a[h], out[h])) return fail(FHE_ELEVEL, "rotate_multi: shape/level mismatch");
        if (a[h]->d == out[h]->d) return fail(FHE_EINVAL, "rotate_multi: out must not alias the input");
        size_t stride = 2ull * l * c->n;
        u32 gh = galois_elt(c, k[h]);
        for (u32 ci = 0; ci < a[h]->count; ci++) {
            in.push_back(a[h]->d + ci * stride);
            o.push_back(out[h]->d + ci * stride);
            g.push_back(gh);
        }
    }
    return rotate_phys(c, in, o, l, g);
}

// Rotations of one ciphertext by m steps sharing one ModUp (Halevi-Shoup hoisting).
// Per physical ct: digits + ModUp once; per step: the inner product reads the extended
// digits through the NTT-domain automorphism (Ext(tau_g(c1)) = perm_g(Ext(c1)): the
// automorphism commutes with the digit lift and permutes NTT slots identically for
// every prime), then ModDown with tau_g(c0).  Words equal m separate fhe_rotate calls.
extern "C" int fhe_rotate_hoisted(fhe_ctx *c, const fhe_ct *a, const uint32_t *k, uint32_t m, fhe_ct *const *out) {
    if (!m) return 0;
    const u32 l = a->level;
    std::vector<u32> g(m);
    for (u32 j = 0; j < m; j++) {
        TRY(check_rot(c, k[j]));
        if (!same_shape(a, out[j])) return fail(FHE_ELEVEL, "rotate_hoisted: shape/level mismatch");
        if (a->d == out[j]->d) return fail(FHE_EINVAL, "rotate_hoisted: out must not alias the input");
        g[j] = galois_elt(c, k[j]);
    }
    const size_t n = c->n, stride = 2ull * l * n;
    use_lane(c, 0);
    const int SI = std::max(1, std::min<int>(c->S, (int)a->count));    // source cts per ModUp batch
    for (u32 b0 = 0; b0 < a->count; b0 += SI) {
        const int si = (int)std::min<u32>(SI, a->count - b0);
        // digits of c1 (identity gather) and ModUp, once per source ct
        PtrTab pt;
        memset(&pt, 0, sizeof pt);
        for (int s = 0; s < si; s++) { pt.in[s] = a->d + (b0 + s) * stride; pt.out[s] = nullptr; pt.g[s] = 1; }
        LOGN_SWITCH(c->logn, launch_row<LG, true>(c, "k_rot_gather_intt", k_rot_gather_intt<LG>, dim3(si, l), c->st,
                                                  pt, (int)l, c->w_D, c->d_mods));
        CHECK_LAUNCH();
        DigitTab dm;
        memset(&dm, 0, sizeof dm);
        for (int s = 0; s < si; s++) dm.coef[s] = c->w_D + (size_t)s * l * n;
        TRY(keyswitch_modup(c, si, l, dm));
        // items (source s, step j), at most S per inner-product / ModDown launch
        const size_t items = (size_t)si * m;
        for (size_t i0 = 0; i0 < items; i0 += c->S) {
            const int S = (int)std::min<size_t>(c->S, items - i0);
            c->key_tick++;
            DigitTab dt;
            KsOut ko;
            memset(&dt, 0, sizeof dt);
            memset(&ko, 0, sizeof ko);
            for (int it = 0; it < S; it++) {
                const size_t item = i0 + it;
                const u32 j = (u32)(item / si), s = (u32)(item % si);
                const u64 *src = a->d + (b0 + s) * stride;
                const u64 *key;
                TRY(get_key(c, g[j], &key));
                dt.ntt[it] = src + (size_t)l * n;      // c1 limbs, natural NTT order (diagonal digits)
                dt.key[it] = key;
                dt.perm[it] = g[j];
                dt.dperm[it] = g[j];
                dt.esrc[it] = s;
                ko.out[it] = out[j]->d + (b0 + s) * stride;
                ko.add[it] = src;                      // c0 limbs, read through the automorphism
                ko.add_g[it] = g[j];
            }
            ko.out_pstride = (long long)l * n;
            ko.add_pstride = 0;
            ko.add_pmask = 1;
            TRY(keyswitch_tail(c, S, l, dt, ko));
        }
    }
    return 0;
}

extern "C" int fhe_hoisted_dot(fhe_ctx *c, fhe_ct *const *R, const uint32_t *g, uint32_t K, fhe_pt *const *pt,
                               uint32_t S, fhe_ct *const *out) {
    if (K < 1 || K > HMAXK) return fail(FHE_EINVAL, "hoisted_dot: K must be in [1, %d]", HMAXK);
    for (u32 k = 0; k < K; k++)
        if (!same_shape(R[k], R[0]) || !(g[k] & 1) || g[k] >= 2 * c->n) return fail(FHE_EINVAL, "hoisted_dot: bad operand %u", k);
    const u32 l = R[0]->level;
    for (u32 s0 = 0; s0 < S; s0 += HTILE) {
        const u32 St = std::min<u32>(HTILE, S - s0);
        HoistArgs a;
        memset(&a, 0, sizeof a);
        for (u32 k = 0; k < K; k++) { a.R[k] = R[k]->d; a.g[k] = g[k]; }
        for (u32 s = 0; s < St; s++) {
            if (!same_shape(out[s0 + s], R[0])) return fail(FHE_ELEVEL, "hoisted_dot: output shape mismatch");
            if (!pt[s0 + s]->encoded) return fail(FHE_EINVAL, "hoisted_dot: plaintext was never encoded");
            a.pt[s] = pt[s0 + s]->ntt_m;
            a.out[s] = out[s0 + s]->d;
        }
        a.K = (int)K; a.S = (int)St; a.Rr = (int)R[0]->R; a.l = (int)l; a.L = (int)c->L; a.logn = (int)c->logn;
        dim3 grid((unsigned)(c->n / 32 > 0 ? c->n / 32 : 1), c->T * l, (St + 7) / 8);
        if (c->n < 32) return fail(FHE_EINVAL, "hoisted_dot needs n >= 32");
        c->alg_mm += (double)St * K * c->T * R[0]->R * 2.0 * l * c->n;
        ProfScope ps_(c, "k_hoisted_dot");
        k_hoisted_dot<<<grid, 256, 0, c->st>>>(a, c->d_mods);
        CHECK_LAUNCH();
    }
    return 0;
}

// one launch per MANY same-shape items (item = blockIdx.z); a list of mixed shapes is
// split at every shape change
extern "C" int fhe_mul_plain_many(fhe_ctx *c, fhe_ct *const *a, fhe_pt *const *pt, fhe_ct *const *out, uint32_t m) {
    for (u32 i = 0; i < m; i++) {
        if (!same_shape(a[i], out[i])) return fail(FHE_ELEVEL, "mul_plain_many: shape/level mismatch at %u", i);
        if (!pt[i]->encoded) return fail(FHE_EINVAL, "mul_plain_many: plaintext %u was never encoded", i);
    }
    for (u32 i0 = 0; i0 < m;) {
        u32 i1 = i0 + 1;
        while (i1 < m && i1 - i0 < MANY && same_shape(a[i1], a[i0])) i1++;
        ManyTab t;
        memset(&t, 0, sizeof t);
        for (u32 i = i0; i < i1; i++) { t.a[i - i0] = a[i]->d; t.b[i - i0] = pt[i]->ntt_m; t.out[i - i0] = out[i]->d; }
        const int rows = (int)(a[i0]->count * 2 * a[i0]->level);
        const unsigned bx = (unsigned)std::max<size_t>(1, (c->n / 2 + 255) / 256);
        dim3 grid(bx, (unsigned)std::min(rows, 65535), i1 - i0);
        ProfScope ps_(c, "k_mul_plain");
        k_mul_plain_many<<<grid, 256, 0, c->st>>>(t, rows, (int)a[i0]->level, (int)c->L, (int)a[i0]->R, (int)c->logn,
                                                  c->d_mods);
        CHECK_LAUNCH();
        i0 = i1;
    }
    return 0;
}
extern "C" int fhe_add_many(fhe_ctx *c, fhe_ct *const *a, fhe_ct *const *b, fhe_ct *const *out, uint32_t m) {
    for (u32 i = 0; i < m; i++)
        if (!same_shape(a[i], b[i]) || !same_shape(a[i], out[i])) return fail(FHE_ELEVEL, "add_many: shape/level mismatch at %u", i);
    for (u32 i0 = 0; i0 < m;) {
        u32 i1 = i0 + 1;
        while (i1 < m && i1 - i0 < MANY && same_shape(a[i1], a[i0])) i1++;
        ManyTab t;
        memset(&t, 0, sizeof t);
        for (u32 i = i0; i < i1; i++) { t.a[i - i0] = a[i]->d; t.b[i - i0] = b[i]->d; t.out[i - i0] = out[i]->d; }
        const long long total = (long long)ct_words(a[i0]);
        const unsigned bx = (unsigned)std::max<long long>(1, std::min<long long>((total / 2 + 255) / 256, 148 * 8));
        ProfScope ps_(c, "k_add");
        k_add_many<<<dim3(bx, 1, i1 - i0), 256, 0, c->st>>>(t, total, (int)a[i0]->level, (int)c->logn, c->d_mods);
        CHECK_LAUNCH();
        i0 = i1;
    }
    return 0;
}

// ------------------------------------------------------ composite operators
// rotate_and_sum of m objects: every tree level is one fused rotate-and-add launch
// sequence over all physical ciphertexts (reference hesim.py:347-366)
extern "C" int fhe_rotate_and_sum(fhe_ctx *c, fhe_ct *const *a, fhe_ct *const *out, uint32_t m, uint32_t span) {
    if (span < 1 || span > c->N) return fail(FHE_EINVAL, "rotate_and_sum: span %u outside [1, %u]", span, c->N);
    if (!m) return 0;
    const u32 l = a[0]->level;
    for (u32 h = 0; h < m; h++) {
        if (a[h]->level != l || !same_shape(a[h], out[h])) return fail(FHE_ELEVEL, "rotate_and_sum: shape/level mismatch");
        if (a[h]->d == out[h]->d) return fail(FHE_EINVAL, "rotate_and_sum: out must not alias the input");
    }
    u32 rounds = 0;
    while ((1u << rounds) < span) rounds++;
    if (!rounds) {
        for (u32 h = 0; h < m; h++) TRY(fhe_ct_copy(c, a[h], out[h]));
        return 0;
    }
    // levels alternate between out and one set of temporaries so the last one lands in out
    std::vector<fhe_ct *> tmp(rounds > 1 ? m : 0, nullptr);
    int rc = 0;
    for (u32 h = 0; h < tmp.size() && !rc; h++) rc = fhe_ct_create(c, a[h]->R, l, &tmp[h]);
    const size_t stride = 2ull * l * c->n;
    for (u32 r = 0; r < rounds && !rc; r++) {
        const bool to_out = (rounds - r) & 1;
        std::vector<const u64 *> in;
        std::vector<u64 *> o;
        for (u32 h = 0; h < m; h++) {
            const u64 *src = r == 0 ? a[h]->d : (to_out ? tmp[h]->d : out[h]->d);
            u64 *dst = to_out ? out[h]->d : tmp[h]->d;
            for (u32 ci = 0; ci < a[h]->count; ci++) { in.push_back(src + ci * stride); o.push_back(dst + ci * stride); }
        }
        rc = rotate_phys(c, in, o, l, std::vector<u32>(in.size(), galois_elt(c, 1u << (rounds - 1 - r))), &in);
    }
    for (fhe_ct *t : tmp) fhe_ct_destroy(t);
    return rc;
}

// Tree concatenation of slot-0-anchored payloads (reference packing.py:350-368): every
// level merges adjacent blocks as left + rotate(right, N - len(left)), all merges of a
// level in one key-switching launch sequence with the addition in its epilogue.
extern "C" int fhe_combine(fhe_ctx *c, fhe_ct *const *cts, const uint32_t *lengths, uint32_t m, fhe_ct *out) {
    if (m < 1) return fail(FHE_EINVAL, "combine: no ciphertexts");
    u64 total = 0;
    for (u32 i = 0; i < m; i++) {
        if (!same_shape(cts[i], out)) return fail(FHE_ELEVEL, "combine: shape/level mismatch");
        if (cts[i]->d == out->d) return fail(FHE_EINVAL, "combine: out must not alias an input");
        if (lengths[i] < 1) return fail(FHE_EINVAL, "combine: payload %u is empty", i);
        total += lengths[i];
    }
    if (total > c->N) return fail(FHE_EINVAL, "combine: payload of %llu slots exceeds %u", (unsigned long long)total, c->N);
    if (m == 1) return fhe_ct_copy(c, cts[0], out);
    struct Item { fhe_ct *ct; u32 len; bool own; };
    std::vector<Item> cur;
    for (u32 i = 0; i < m; i++) cur.push_back({cts[i], lengths[i], false});
    const u32 l = out->level;
    const size_t stride = 2ull * l * c->n;
    int rc = 0;
    while (cur.size() > 1 && !rc) {
        std::vector<Item> next;
        std::vector<const u64 *> in, left;
        std::vector<u64 *> o;
        std::vector<u32> g;
        for (size_t k = 0; k + 1 < cur.size() && !rc; k += 2) {
            fhe_ct *dst = out;
            if (cur.size() > 2) rc = fhe_ct_create(c, out->R, l, &dst);
            if (rc) break;
            const u32 ge = galois_elt(c, c->N - cur[k].len);
            for (u32 ci = 0; ci < out->count; ci++) {
                in.push_back(cur[k + 1].ct->d + ci * stride);
                left.push_back(cur[k].ct->d + ci * stride);
                o.push_back(dst->d + ci * stride);
                g.push_back(ge);
            }
            next.push_back({dst, cur[k].len + cur[k + 1].len, dst != out});
        }
        if (!rc) rc = rotate_phys(c, in, o, l, g, &left);
        if (rc)
            for (auto &it : next)
                if (it.own) fhe_ct_destroy(it.ct);
        const size_t paired = cur.size() & ~(size_t)1;
        for (size_t k = 0; k < paired; k++)
            if (cur[k].own) fhe_ct_destroy(cur[k].ct);        // stream-ordered: the level above was enqueued
        if (rc) {
            if ((cur.size() & 1) && cur.back().own) fhe_ct_destroy(cur.back().ct);
            break;
        }
        if (cur.size() & 1) next.push_back(cur.back());
        cur.swap(next);
    }
    return rc;
}

// ct-GEMM (reference engine.py:178-197): out[o] = sum_k w[k O + o] a[k]
static int gemm_table(fhe_ctx *c, const int64_t *w, u32 K, u32 O, const u64 **tab) {
    u64 h = 1469598103934665603ull;
    auto mix = [&](u64 v) { for (int b = 0; b < 8; b++) { h ^= (v >> (8 * b)) & 0xFF; h *= 1099511628211ull; } };
    mix(K); mix(O);
    for (size_t e = 0; e < (size_t)K * O; e++) mix((u64)w[e]);
    auto it = c->gemm_tabs.find(h);
    if (it != c->gemm_tabs.end()) { *tab = it->second; return 0; }
    if (c->cap_arena) return fail(FHE_EINVAL, "ct_gemm weight table created inside a capture (warm the walk up first)");
    const u32 L = c->L;
    std::vector<u64> host((size_t)L * K * O);
    for (u32 i = 0; i < L; i++) {
        const u64 q = c->P.q[i];
        for (size_t e = 0; e < (size_t)K * O; e++) {
            const int64_t v = w[e];
            const u64 r = v >= 0 ? (u64)v % q : hm::neg((u64)(-(v + 1)) % q + 1, q);
            host[(size_t)i * K * O + e] = hm::mont(r, q);
        }
    }
    u64 *d = nullptr;
    if (cudaMalloc((void **)&d, host.size() * 8) != cudaSuccess) return fail(FHE_ENOMEM, "ct_gemm weight table");
    CU(cudaMemcpyAsync(d, host.data(), host.size() * 8, cudaMemcpyHostToDevice, c->st));
    CU(cudaStreamSynchronize(c->st));          // host staging goes out of scope
    c->gemm_tabs[h] = d;
    *tab = d;
    return 0;
}

extern "C" int fhe_ct_gemm(fhe_ctx *c, fhe_ct *const *a, uint32_t K, const int64_t *w, uint32_t O, fhe_ct *const *out) {
    if (K < 1 || O < 1) return fail(FHE_EINVAL, "ct_gemm: empty operand list");
    for (u32 k = 0; k < K; k++)
        if (!same_shape(a[k], a[0])) return fail(FHE_ELEVEL, "ct_gemm: shape/level mismatch");
    for (u32 o = 0; o < O; o++) {
        if (!same_shape(out[o], a[0])) return fail(FHE_ELEVEL, "ct_gemm: shape/level mismatch");
        for (u32 k = 0; k < K; k++)
            if (out[o]->d == a[k]->d) return fail(FHE_EINVAL, "ct_gemm: out must not alias an input");
    }
    const u64 *tab = nullptr;
    TRY(gemm_table(c, w, K, O, &tab));
    const u32 l = a[0]->level;
    u64 maxq = 0;
    for (u32 i = 0; i < l; i++) maxq = std::max<u64>(maxq, c->P.q[i]);
    const int kc = (int)std::min<u64>(GEMM_MAXK, ~0ull / maxq);          // kc q < 2^64
    const int rows = (int)(a[0]->count * 2 * l);
    const unsigned bx = (unsigned)std::max<size_t>(1, (c->n / 2 + 255) / 256);
    c->alg_mm += (double)rows * c->n * K * O;
    for (u32 o0 = 0; o0 < O; o0 += GEMM_OT) {
        const int ot = (int)std::min<u32>(GEMM_OT, O - o0);
        for (u32 k0 = 0; k0 < K; k0 += GEMM_MAXK) {
            const int kk = (int)std::min<u32>(GEMM_MAXK, K - k0);
            GemmTab t;
            memset(&t, 0, sizeof t);
            for (int k = 0; k < kk; k++) t.in[k] = a[k0 + k]->d;
            for (int o = 0; o < ot; o++) t.out[o] = out[o0 + o]->d;
            ProfScope ps_(c, "k_ct_gemm");
            if (k0 == 0)
                k_ct_gemm<false><<<dim3(bx, rows), 256, 0, c->st>>>(t, tab, kk, (int)K, (int)k0, (int)O, (int)o0, ot, kc,
                                                                   (int)l, (int)c->logn, c->d_mods);
            else
                k_ct_gemm<true><<<dim3(bx, rows), 256, 0, c->st>>>(t, tab, kk, (int)K, (int)k0, (int)O, (int)o0, ot, kc,
                                                                  (int)l, (int)c->logn, c->d_mods);
            CHECK_LAUNCH();
        }
    }
    return 0;
}

// ------------------------------------------------------------ mod switch
extern "C" int fhe_mod_switch(fhe_ctx *c, const fhe_ct *a, fhe_ct *out) {
    u32 l = a->level;
    size_t n = c->n;
    if (l < 2) return fail(FHE_ELEVEL, "mod_switch: already at level 1");
    if (out->level != l - 1 || out->R != a->R) return fail(FHE_ELEVEL, "mod_switch: out must have level %u", l - 1);
    size_t cnt = a->count;
    TRY(ensure_tmp(c, cnt * 2 * n));
    // INTT of the dropped limb of both polynomials: row r = ci*2 + p
    InttRowsArgs ia = iargs(a->d + (l - 1) * n, c->w_tmp, (long long)l * n);
    ia.dA = n;
    ia.map.id[0] = (unsigned char)(l - 1);
    TRY(intt_rows(c, (int)(cnt * 2), ia, "k_intt_rows(modswitch)"));
    const LevelDev &T = c->hlv[l];
    for (size_t b0 = 0; b0 < cnt; b0 += MAXS) {
        int S = (int)std::min<size_t>(MAXS, cnt - b0);
        RescaleArgs ra;
        memset(&ra, 0, sizeof ra);
        for (int s = 0; s < S; s++) {
            size_t ci = b0 + s;
            ra.coef[s] = c->w_tmp + ci * 2 * n;
            ra.base[s] = a->d + ci * 2 * l * n;
            ra.out[s] = out->d + ci * 2 * (l - 1) * n;
        }
        ra.coef_pstride = n;
        ra.base_pstride = (long long)l * n;
        ra.out_pstride = (long long)(l - 1) * n;
        ra.src_id = (int)(l - 1);
        for (u32 i = 0; i + 1 < l; i++) { ra.fac[i] = T.msinv[i]; ra.fac_sh[i] = T.msinv_sh[i]; }
        LOGN_SWITCH(c->logn, launch_row<LG, false, RescaleW<LG>::value>(c, "k_rescale(modswitch)", k_rescale<LG>, dim3(S, 2, l - 1), c->st, ra, c->d_mods));
        CHECK_LAUNCH();
    }
    return 0;
}

// --------------------------------------------------------------- squaring
extern "C" int fhe_square(fhe_ctx *c, const fhe_ct *a, fhe_ct *out) {
    if (!c->nb) return fail(FHE_EINVAL, "square: context created without an auxiliary base");
    if (!same_shape(a, out)) return fail(FHE_ELEVEL, "square: shape/level mismatch");
    if (a == out || a->d == out->d) return fail(FHE_EINVAL, "square: out must not alias the input");
    const u64 *rk;
    TRY(get_key(c, 0, &rk));
    size_t n = c->n, l = a->level, nb = c->nb, nt = l + nb;
    const size_t per = n * (2 * l + 2 * nb + 3 * nt + 3 * l + 3 * l);
    int Smax = (int)std::min<size_t>(c->S, c->w_sq_words / per);
    if (Smax < 1) return fail(FHE_ENOMEM, "square workspace too small");
    for (size_t b0 = 0; b0 < a->count; b0 += Smax) {
        int S = (int)std::min<size_t>(Smax, a->count - b0);
        const u64 *in = a->d + b0 * 2 * l * n;
        u64 *X = c->w_sq, *Xb = X + S * 2 * l * n, *D = Xb + S * 2 * nb * n, *E = D + S * 3 * nt * n,
            *En = E + S * 3 * l * n;
        // 1. coefficient form of c0, c1 over Q_l
        InttRowsArgs ia = iargs(in, X, n);
        ia.period = l;
        map_q(ia.map, l);
        TRY(intt_rows(c, S * 2 * (int)l, ia));
        // 2. centered lift to B, NTT over B
        long long tot = (long long)S * 2 * n;
        EW(k_sq_lift, tot, X, Xb, tot, (int)l, (int)nb, (int)c->logn, c->d_lv + l, c->b_id0, c->d_mods);
        CHECK_LAUNCH();
        NttRowsArgs na = nargs(Xb, Xb, n);
        na.period = nb;
        map_range(na.map, nb, c->b_id0);
        TRY(ntt_rows(c, S * 2 * (int)nb, na));
        // 3. tensor over Q_l u B, back to coefficients
        tot = (long long)S * nt * n;
        EW(k_sq_tensor, tot, in, Xb, D, tot, (int)l, (int)nb, (int)c->logn, c->b_id0, c->d_mods);
        CHECK_LAUNCH();
        ia = iargs(D, D, n);
        ia.period = nt;
        for (size_t ii = 0; ii < nt; ii++) ia.map.id[ii] = (unsigned char)(ii < l ? ii : c->b_id0 + ii - l);
        TRY(intt_rows(c, S * 3 * (int)nt, ia));
        // 4. scale by t/Q_l into B, back to Q_l
        tot = (long long)S * 3 * n;
        EW(k_sq_scale, tot, D, E, tot, (int)l, (int)nb, (int)a->R, (int)b0, (int)c->logn, c->d_lv + l, c->d_ax,
           c->b_id0, c->d_mods);
        CHECK_LAUNCH();
        na = nargs(E, En, n);
        na.period = l;
        map_q(na.map, l);
        TRY(ntt_rows(c, S * 3 * (int)l, na));
        // 5. relinearize e2, add e0/e1
        DigitTab dt;
        KsOut ko;
        memset(&dt, 0, sizeof dt);
        memset(&ko, 0, sizeof ko);
        for (int s = 0; s < S; s++) {
            dt.coef[s] = E + ((size_t)s * 3 + 2) * l * n;
            dt.ntt[s] = En + ((size_t)s * 3 + 2) * l * n;
            dt.key[s] = rk;
            ko.out[s] = out->d + (b0 + s) * 2 * l * n;
            ko.add[s] = En + (size_t)s * 3 * l * n;
        }
        ko.out_pstride = (long long)l * n;
        ko.add_pstride = (long long)l * n;
        ko.add_pmask = 3;
        TRY(keyswitch_core(c, S, (u32)l, dt, ko));
    }
    return 0;
}
