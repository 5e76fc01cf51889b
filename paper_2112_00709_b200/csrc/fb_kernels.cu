// fb_kernels.cu — sm_100a kernels and C-ABI entry points of libfb.
//
// One CTA per sequence runs the whole time recursion of one direction with the
// sequence's graph schedule resident in shared memory (P:173-191 in the log
// semifield, P:193-227 batched).  Per frame n one CTA does:
//
//   phase A  every lane walks its slot column of the nnz-balanced schedule and
//            reduces its row segments: factored mode  Σ p_src·e^{T} with
//            p = 2^{u} (one FMA per arc, exact max-then-sum fallback when the
//            sum leaves [2^-80, 2^120]); exact mode online max-then-sum (one
//            ex2 per arc).  Segment results (log2) go to smem `part`.
//   barrier
//   phase B1 per owned state: combine its segments, add the emission
//            (forward: v_n after the product, Eq. (13); backward: v_n on the
//            new β̂_n, Eq. (14) with ledger L2), apply the exact viability mask,
//            warp max of the new vector.
//   barrier
//   phase B2 normalise by the block max (exact, so the largest viable entry is
//            0 — SURVEY §8(c4)), accumulate the float64 scale, write α̂/β̂ to
//            HBM, refresh u (log2) and p = 2^{u} in smem; backward also forms
//            x = α̂_n + β̂_n and its warp log-sum-exp for the fused posterior
//            epilogue, which is completed one frame later (no extra barrier).
//   barrier
//
// All log quantities are carried in base 2 inside the kernels (ex2/lg2 are the
// native MUFU ops) and converted to natural logs at the HBM boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "fb_internal.h"

namespace fbx {

static const float kL2E = 1.4426950408889634f;
static const double kLN2 = 0.6931471805599453;

// ------------------------------------------------------------------ error / profiling

static std::mutex g_err_mu;
static std::string g_err = "";

void set_cuda_error(const char *what, int code) {
    std::lock_guard<std::mutex> lk(g_err_mu);
    g_err = std::string(what) + ": " + cudaGetErrorString((cudaError_t)code);
}

struct ProfRec {
    const char *name;
    cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_event_pool;

static cudaEvent_t pool_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

struct ProfScope {
    bool on;
    ProfRec r;
    cudaStream_t s;
    ProfScope(const char *name, cudaStream_t st) : on(false), s(st) {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        if (!g_prof_on) return;
        on = true;
        r.name = name;
        r.a = pool_event();
        r.b = pool_event();
        cudaEventRecord(r.a, s);
    }
    ~ProfScope() {
        if (!on) return;
        cudaEventRecord(r.b, s);
        std::lock_guard<std::mutex> lk(g_prof_mu);
        g_prof.push_back(r);
    }
};

// ------------------------------------------------------------------ device helpers

#define NEG_INF (-__int_as_float(0x7f800000))
#define NEG_INF_D (-__longlong_as_double(0x7ff0000000000000ll))

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <class V>
__device__ __forceinline__ V ninf() { return (V)NEG_INF_D; }
template <class V>
__device__ __forceinline__ V vmax(V a, V b) { return a > b ? a : (b > a ? b : a); }
template <class V>
__device__ __forceinline__ V vmin(V a, V b) { return a < b ? a : (b < a ? b : a); }
template <class V>
__device__ __forceinline__ V warp_max(V v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = vmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
// Warp max of a float via one REDUX on order-preserving integer keys
// (doubles use shuffles); warp sum via shuffles.
__device__ __forceinline__ int f2key(float f) {
    const int i = __float_as_int(f);
    return i ^ ((i >> 31) & 0x7FFFFFFF);
}
__device__ __forceinline__ float key2f(int k) { return __int_as_float(k ^ ((k >> 31) & 0x7FFFFFFF)); }
__device__ __forceinline__ float warp_max_fast(float v) { return key2f(__reduce_max_sync(0xffffffffu, f2key(v))); }
__device__ __forceinline__ double warp_max_fast(double v) { return warp_max(v); }
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// Block log-sum-exp (log2) from per-warp (max, Σ 2^{x-max}) pairs held by lanes < W.
template <class V>
__device__ __forceinline__ V block_lse_pairs(V m, float s) {
    const V M = warp_max_fast(m);
    const V Ms = (M == ninf<V>()) ? (V)0 : M;
    const float t = (m == ninf<V>()) ? 0.f : s * ex2((float)(m - Ms));
    const float S = warp_sum(t);
    return (M == ninf<V>()) ? M : M + (V)lg2(S);
}
// This thread's (max, Σ) over its SPT values reduced over the warp.
template <class V, int SPT>
__device__ __forceinline__ void warp_lse_vals(const V *x, V &wm, float &ws) {
    V m = ninf<V>();
#pragma unroll
    for (int k = 0; k < SPT; ++k) m = vmax(m, x[k]);
    m = warp_max_fast(m);
    const V ms = (m == ninf<V>()) ? (V)0 : m;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < SPT; ++k) s += ex2((float)(x[k] - ms));
    wm = m;
    ws = warp_sum(s);
}

// (m, s) log-sum-exp pair (value = m + log2 s), m in V, s in float (s ∈ [1, n])
template <class V>
__device__ __forceinline__ void lse_push(V &m, float &s, V x) {
    if (x > m) { s = (m == ninf<V>() ? 0.f : s * ex2((float)(m - x))) + 1.f; m = x; }
    else if (x != ninf<V>()) s += ex2((float)(x - m));
}
template <class V>
__device__ __forceinline__ void lse_combine(V &m, float &s, V m2, float s2) {
    V M = vmax(m, m2);
    if (M == ninf<V>()) { m = ninf<V>(); s = 0.f; return; }
    s = (m == ninf<V>() ? 0.f : s * ex2((float)(m - M))) + (m2 == ninf<V>() ? 0.f : s2 * ex2((float)(m2 - M)));
    m = M;
}
template <class V>
__device__ __forceinline__ void warp_lse(V &m, float &s) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        V m2 = __shfl_xor_sync(0xffffffffu, m, o);
        float s2 = __shfl_xor_sync(0xffffffffu, s, o);
        lse_combine(m, s, m2, s2);
    }
}

// Shared-memory access through 32-bit shared-window addresses (explicit PTX so
// the hot loops carry no generic-address arithmetic).
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return (uint32_t)v;
}
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds_v(uint32_t a, float) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_v(uint32_t a, double) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_v(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v)); }
__device__ __forceinline__ void sts_v(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
__device__ __forceinline__ void sts_i(uint32_t a, int v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v)); }
__device__ __forceinline__ int lds_i(uint32_t a) { return (int)lds_u32(a); }

// TMA bulk copy global → shared with mbarrier completion (Hopper+/Blackwell).
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P1;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAIT_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}

// Block log-sum-exp from per-warp (m, s) pairs in (generic) shared memory.
template <class V>
__device__ __forceinline__ V block_lse_from(const double *wz, int W, int lane) {
    V m = lane < W ? (V)wz[2 * lane] : ninf<V>();
    float s = lane < W ? (float)wz[2 * lane + 1] : 0.f;
    warp_lse(m, s);
    return m == ninf<V>() ? ninf<V>() : m + (V)lg2(s);
}


struct FBArgs {
    Graph g;
    const float *emis;
    const int *lengths;
    int B, N_max, D;
    float *lat;         // α̂ (fwd) / β̂ (bwd) out, may be null
    double *scale;      // [B][N_max] out, may be null
    double *logZ;       // fwd: logZ; bwd: logZ_beta (may be null)
    int *status;        // fwd: out; bwd: in/out
    const int *status2; // bwd (lfmmi): numerator status, OR-ed in (may be null)
    // backward epilogue
    const float *alpha; // α̂ from the forward (natural log), may be null
    int post_kind;
    float *post;        // state / dense pdf / compact pdf / grad
    // lfmmi gradient (POST_GRAD): Γ_num compact and the numerator pdf map
    const float *gnum;
    const int *num_slot_off;
    const int *num_pdf_slot; // [B*D]
    int num_U_max;           // largest numerator slot count (gnbuf size)
    int tma;                 // stage φ rows in shared memory with TMA bulk copies
    // MODE_RAW (lfmmi numerator): float64 log2 lattices, posteriors normalised by logZ_in
    double *lat64;
    const double *alpha64;
    const double *logZ_in;
};

// Exact max-then-sum over one row held by g lanes (fallback of factored mode,
// where weights are stored as e^{T}); `cur` is the slice, `lane` the group
// leader.  Accurate libm ops; rare.
__device__ __noinline__ float exact_row(uint32_t cur, int L2, int g, int lane, uint32_t a_u) {
    float m = NEG_INF, sum = 0.f;
    for (int t = 0; t < g; ++t)
        for (int s = 0; s < 2 * L2; ++s) {
            uint32_t ix = lds_u32(cur + 128 + (s >> 1) * 128 + (lane + t) * 4);
            uint32_t o = (s & 1) ? (ix >> 16) : (ix & 0xFFFFu);
            float w = lds_v(cur + 128 + L2 * 128 + (s >> 1) * 256 + (lane + t) * 8 + (s & 1) * 4, 0.f);
            float x = lds_v(a_u + o, 0.f) + log2f(w);
            if (x == NEG_INF) continue;
            if (x > m) { sum = sum * exp2f(m - x) + 1.f; m = x; }
            else sum += exp2f(x - m);
        }
    return m == NEG_INF ? NEG_INF : m + log2f(sum);
}

// Phase A: walk this warp's slices (layout: fb_internal.h, Sched).  Lane l
// reduces one row segment per slice; the g lanes of a split row are combined
// with a uniform xor-shuffle and the group leader writes the row's log2 value
// into part[row].
//  factored: Σ p_src · e^{T} (one FMA per arc, two accumulators), exact
//            fallback when the sum leaves [2^-80, 2^120];
//  exact:    online max-then-sum in V (double) with one ex2 per arc (two chains).
template <int MODE, class V>
__device__ __forceinline__ void phase_a(uint32_t cur, int nsl, int lane, uint32_t a_u, uint32_t a_p,
                                        uint32_t a_part) {
    constexpr float kTiny = 8.271806125530277e-25f;  // 2^-80
    constexpr float kHuge = 1.329227995784916e+36f;  // 2^120
    constexpr uint32_t VS = sizeof(V);
    for (int q = 0; q < nsl; ++q) {
        const uint32_t h = lds_u32(cur + lane * 4);
        const int row = (int)(h & 0xFFFFu) - 1, lg = (int)((h >> 16) & 7u), L2 = (int)(h >> 19);
        uint32_t ia = cur + 128 + lane * 4;
        uint32_t wa = cur + 128 + (uint32_t)L2 * 128 + lane * 8;
        if (MODE == MODE_FACTORED) {
            float a0 = 0.f, a1 = 0.f;
#pragma unroll 2
            for (int s = 0; s < L2; ++s) {
                const uint32_t ix = lds_u32(ia);
                const float2 w2 = lds_f2(wa);
                const float p0 = lds_v(a_p + (ix & 0xFFFFu), 0.f), p1 = lds_v(a_p + (ix >> 16), 0.f);
                a0 = fmaf(p0, w2.x, a0);
                a1 = fmaf(p1, w2.y, a1);
                ia += 128;
                wa += 256;
            }
            float acc = a0 + a1;
            if (lg) {
                for (int o = 1; o < (1 << lg); o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            }
            if (row >= 0)
                sts_v(a_part + (uint32_t)row * VS,
                      (V)((acc >= kTiny && acc <= kHuge) ? lg2(acc) : exact_row(cur, L2, 1 << lg, lane, a_u)));
        } else {
            V m0 = ninf<V>(), m1 = ninf<V>();
            float s0 = 0.f, s1 = 0.f;
            auto push = [&](V &m, float &sm, uint32_t off, float w) {
                V x = lds_v(a_u + off, (V)0) + (V)w;
                V hi = vmax(m, x), lo = vmin(m, x);
                float e = (lo == ninf<V>()) ? 0.f : ex2((float)(lo - hi));
                sm = (x > m) ? fmaf(sm, e, 1.f) : sm + e;
                m = hi;
            };
            for (int s = 0; s < L2; ++s) {
                const uint32_t ix = lds_u32(ia);
                const float2 w2 = lds_f2(wa);
                push(m0, s0, ix & 0xFFFFu, w2.x);
                push(m1, s1, ix >> 16, w2.y);
                ia += 128;
                wa += 256;
            }
            lse_combine(m0, s0, m1, s1);
            for (int o = 1; o < (1 << lg); o <<= 1) {
                V m2 = __shfl_xor_sync(0xffffffffu, m0, o);
                float s2 = __shfl_xor_sync(0xffffffffu, s0, o);
                lse_combine(m0, s0, m2, s2);
            }
            if (row >= 0) sts_v(a_part + (uint32_t)row * VS, (m0 == ninf<V>()) ? m0 : m0 + (V)lg2(s0));
        }
        cur += 128 + (uint32_t)L2 * 384;
    }
}

// Write one frame's pdf-level posterior (or gradient) row.  gbuf holds γ in the
// member's slot order, so pdf slot s sums gbuf[ssp[s] .. ssp[s+1]) (ascending
// state order, ledger L9); maps staged in shared memory (PdfRegion), addressed
// through the 32-bit shared window.
__device__ __forceinline__ int lds_s16(uint32_t a) {
    short v;
    asm volatile("ld.shared.s16 %0, [%1];" : "=h"(v) : "r"(a));
    return (int)v;
}
__device__ __forceinline__ void pdf_row(const FBArgs &a, uint32_t a_gbuf, uint32_t a_ssp, uint32_t a_pslot, int gi,
                                        int b, int n, int tid, int T) {
    const Graph &G = a.g;
    const PdfMap &pm = G.pm;
    if (a.post_kind == POST_PDF_COMPACT) {
        const int so = pm.slot_off[gi], U = pm.slot_off[gi + 1] - so;
        float *row = a.post + (size_t)a.N_max * so + (size_t)n * U;
        for (int sl = tid; sl < U; sl += T) {
            const int q0 = (int)lds_u16(a_ssp + 2 * sl), q1 = (int)lds_u16(a_ssp + 2 * sl + 2);
            float acc = 0.f;
            for (int q = q0; q < q1; ++q) acc += lds_v(a_gbuf + 4 * q, 0.f);
            row[sl] = acc;
        }
        return;
    }
    const int D = a.D;
    float *row = a.post + ((size_t)b * a.N_max + n) * D;
    const float sgn = a.post_kind == POST_GRAD ? -1.f : 1.f;  // grad: −Γ_den; Γ_num added by k_add_num
    for (int d = tid; d < D; d += T) {
        const int sl = lds_s16(a_pslot + 2 * d);
        float acc = 0.f;
        if (sl >= 0) {
            const int q0 = (int)lds_u16(a_ssp + 2 * sl), q1 = (int)lds_u16(a_ssp + 2 * sl + 2);
            acc = lds_v(a_gbuf + 4 * q0, 0.f);
            for (int q = q0 + 1; q < q1; ++q) acc += lds_v(a_gbuf + 4 * q, 0.f);
        }
        row[d] = sgn * acc;
    }
}

// Zero (posterior) / −∞ (lattice) rows for frames [n0, n1).
__device__ void write_pad_rows(const FBArgs &a, int gi, int b, int K, int s0, int n0, int n1, int tid, int T,
                               bool lattice, bool bwd) {
    const Graph &G = a.g;
    const size_t lat_base = (size_t)a.N_max * (G.G == 1 ? (size_t)b * K : (size_t)s0);
    for (int n = n0; n < n1; ++n) {
        if (lattice && a.lat)
            for (int j = tid; j < K; j += T) a.lat[lat_base + (size_t)n * K + j] = NEG_INF;
        if (lattice && a.scale && tid == 0) a.scale[(size_t)b * a.N_max + n] = 0.0;
        if (!bwd || a.post_kind == POST_NONE) continue;
        if (a.post_kind == POST_STATE) {
            for (int j = tid; j < K; j += T) a.post[lat_base + (size_t)n * K + j] = 0.f;
        } else if (a.post_kind == POST_PDF_COMPACT) {
            const int so = G.pm.slot_off[gi], U = G.pm.slot_off[gi + 1] - so;
            for (int j = tid; j < U; j += T) a.post[(size_t)a.N_max * so + (size_t)n * U + j] = 0.f;
        } else {
            for (int d = tid; d < a.D; d += T) a.post[((size_t)b * a.N_max + n) * a.D + d] = 0.f;
        }
    }
}

// ------------------------------------------------------------------ forward / backward kernel

// One CTA runs the whole recursion of one sequence in one direction.  Per frame:
//   phase A (arcs) → barrier → phase B (states) → barrier.
// Phase B normalises with the lagged constant c_n = max of the previous
// frame's vector (known after the barrier, no extra reduction pass); the
// float64 offset accumulates c_n exactly, and the largest entry of each stored
// frame is the one-frame change of the recursion, so exp2 of the vector stays
// in range (exact fallback otherwise).
// MODEX: MODE_FACTORED / MODE_EXACT / MODE_RAW, or kModeFactoredTma (factored
// arithmetic with φ rows staged through TMA).
constexpr int kModeFactoredTma = 4;
template <bool BWD, int MODEX, int SPT>
__device__ __forceinline__ void fb_sequence(const FBArgs &a, const int b) {
    constexpr bool TMA = MODEX == kModeFactoredTma;
    constexpr int MODE = TMA ? (int)MODE_FACTORED : MODEX;
    using V = typename std::conditional<MODE == MODE_FACTORED, float, double>::type;
    constexpr uint32_t VS = sizeof(V);
    constexpr bool RAW = MODE == MODE_RAW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Graph &G = a.g;
    const int gi = (G.G == 1) ? 0 : b;
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, W = T >> 5;
    const int s0 = G.state_off[gi];
    const int K = G.state_off[gi + 1] - s0;
    const int N = a.lengths[b];
    const Sched &S = BWD ? G.bwd : G.fwd;
    const bool want_post = BWD && a.post_kind != POST_NONE;
    const bool pdf_post = want_post && a.post_kind != POST_STATE;
    const SmemLayout SL = smem_layout(S.bytes_max, T * SPT, MODE != MODE_FACTORED, want_post && pdf_post);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t a_u = sb + (uint32_t)SL.u, a_p = sb + (uint32_t)SL.p, a_part = sb + (uint32_t)SL.part;
    const uint32_t a_wmax = sb + (uint32_t)SL.red, a_wz = a_wmax + 64 * 8, a_flag = a_wmax + 192 * 8;
    float *gbuf = (float *)(smem_raw + SL.gbuf);
    const PdfRegion PR = pdf_region(a.post_kind, G.pm.U_max, a.D);
    unsigned short *ssp = (unsigned short *)(smem_raw + SL.total + PR.ssp);
    short *pslot = (short *)(smem_raw + SL.total + PR.pslot);
    const uint32_t a_gbuf = sb + (uint32_t)SL.gbuf;
    // φ row staging (TMA): two row buffers + two mbarriers after the pdf region
    constexpr bool use_tma = TMA;
    const uint32_t rowbytes = (uint32_t)a.D * 4;
    const uint32_t a_ebuf = sb + (uint32_t)(SL.total + PR.bytes);
    const uint32_t a_mbar = a_ebuf + (uint32_t)fbx_a16(2 * (size_t)rowbytes);
    const uint32_t a_ssp = sb + (uint32_t)(SL.total + PR.ssp), a_pslot = sb + (uint32_t)(SL.total + PR.pslot);
    const V L2E = (V)1.4426950408889634;
    const V LN2 = (V)0.6931471805599453;
    const V NINF = ninf<V>();

    int st = 0;
    if (BWD) {
        st = a.status[b];
        if (a.status2) st |= a.status2[b];
    }
    if (N < 1 || N > a.N_max) st |= FB_SEQ_BAD_LENGTH;
    // Frames past the end (and whole flagged sequences in the backward) are written up front.
    const bool skip = (st & FB_SEQ_BAD_LENGTH) || (BWD && st != 0);
    write_pad_rows(a, gi, b, K, s0, skip ? 0 : N, a.N_max, tid, T, !(st & FB_SEQ_BAD_LENGTH), BWD);
    if (skip) {
        if (tid == 0) {
            if (a.logZ) a.logZ[b] = -INFINITY;
            a.status[b] = st;
        }
        return;
    }

    // schedule → shared memory (16-byte vector copy)
    {
        const uint4 *src = (const uint4 *)(S.rec + S.rec_off[gi]);
        uint4 *dst = (uint4 *)(smem_raw + SL.rec);
        const int n16 = S.rec_bytes[gi] >> 4;
        for (int x = tid; x < n16; x += T) dst[x] = src[x];
    }
    if (tid == 0) sts_i(a_flag, 0);
    // pdf-level epilogue maps → shared memory
    if (pdf_post) {
        const int so = G.pm.slot_off[gi], U = G.pm.slot_off[gi + 1] - so;
        const int base = G.pm.slot_sptr[so];
        for (int x = tid; x <= U; x += T) ssp[x] = (unsigned short)(G.pm.slot_sptr[so + x] - base);
        if (a.post_kind != POST_PDF_COMPACT)
            for (int d = tid; d < a.D; d += T) pslot[d] = (short)G.pm.pdf_slot[(size_t)gi * a.D + d];
    }
    const int nsl = S.warp_nsl[gi * W + warp];
    const uint32_t mysl = sb + (uint32_t)SL.rec + (uint32_t)S.warp_off[gi * W + warp];
    const bool use_mask = BWD ? G.mask_bwd : G.mask_fwd;

    // Owned states j = tid + k*T (k < SPT).  Slots with j ≥ K are inert: their
    // partial stays 0̄, pdf 0, never stored to HBM.
    int pdfk[SPT];   // emission column
    int distk[SPT];  // viability distance
    int posk[SPT];   // position in the slot-ordered γ buffer (pdf-level epilogue)
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const int j = tid + k * T;
        pdfk[k] = 0;
        distk[k] = 0;
        posk[k] = 0;
        if (j < K) {
            pdfk[k] = G.pdf[s0 + j];
            distk[k] = BWD ? G.dist_start[s0 + j] : G.dist_fin[s0 + j];
            if (pdf_post) posk[k] = G.pm.slot_pos[s0 + j];
        }
        sts_v(a_part + (uint32_t)j * VS, NINF);  // rows without arcs are never written by phase A
    }
    const float *em = a.emis + (size_t)b * a.N_max * a.D;
    const size_t lat_base = (size_t)a.N_max * (G.G == 1 ? (size_t)b * K : (size_t)s0);
    auto load_v = [&](int n, float *v) {
        if (use_tma) return;  // rows arrive in shared memory instead
        const float *row = em + (size_t)min(max(n, 0), N - 1) * a.D;
#pragma unroll
        for (int k = 0; k < SPT; ++k) v[k] = __ldg(row + pdfk[k]);
    };
    // TMA: step t (t-th frame processed) uses buffer t & 1, whose (t >> 1)-th
    // completion has parity (t >> 1) & 1.  Issued by one thread one step ahead.
    auto tma_issue = [&](int t, int n) {
        if (!use_tma || tid != 0) return;
        if (n < 0 || n >= N) return;
        const uint32_t mb = a_mbar + 8u * (uint32_t)(t & 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_tx(mb, rowbytes);
        tma_g2s(a_ebuf + (uint32_t)(t & 1) * rowbytes, em + (size_t)n * a.D, rowbytes, mb);
    };
    // this thread's emissions of the frame processed at step t
    auto fetch_v = [&](int t, const float *vreg, float *v) {
        if (!use_tma) {
#pragma unroll
            for (int k = 0; k < SPT; ++k) v[k] = vreg[k];
            return;
        }
        mbar_wait(a_mbar + 8u * (uint32_t)(t & 1), (uint32_t)((t >> 1) & 1));
        const uint32_t base = a_ebuf + (uint32_t)(t & 1) * rowbytes;
#pragma unroll
        for (int k = 0; k < SPT; ++k) v[k] = lds_v(base + 4u * (uint32_t)pdfk[k], 0.f);
    };
    if (use_tma && tid == 0) {
        mbar_init(a_mbar, 1);
        mbar_init(a_mbar + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (use_tma) __syncthreads();  // barriers initialised before anyone waits on them
    // α̂ of frame n as stored (float natural log, or the raw float64 log2 lattice);
    // converted to log2 at use so the load is not waited on at issue
    auto load_alpha = [&](int n, V *v) {
        const size_t ro = lat_base + (size_t)min(max(n, 0), N - 1) * K;
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const int j = min(tid + k * T, K - 1);
            if (RAW) v[k] = (V)__ldg(a.alpha64 + ro + j);
            else v[k] = (V)__ldg(a.alpha + ro + j);
        }
    };
    // viable(k, n): forward — a final state is reachable in the N-1-n remaining
    // transitions; backward — the state is reachable from an initial state in n.
    auto viable = [&](int k, int n) { return !use_mask || (BWD ? (distk[k] <= n) : (distk[k] <= N - 1 - n)); };

    // Ping-pong prefetch buffers (A: even steps, B: odd steps): a buffer is
    // consumed by its frame's phase B and immediately refilled with the frame
    // two steps ahead, so loads have a whole frame of slack and no register moves.
    float vA[SPT], vB[SPT];  // emissions
    V aA[SPT], aB[SPT];      // α̂ (backward epilogue), log2 units
    V uk[SPT];               // this thread's entries of the current vector u (log2)
    V xpost[SPT];            // α̂_n + β̂_n of the frame whose posterior is pending
    const int dir = BWD ? -1 : 1;
    const int n_first = BWD ? N - 1 : 0;
    load_v(n_first, vA);
    load_v(n_first + dir, vB);
    tma_issue(0, n_first);
    tma_issue(1, n_first + dir);
    int tstep = 0;  // index of the frame being produced (t in tma_issue / fetch_v)
    if (want_post) { load_alpha(n_first, aA); load_alpha(n_first + dir, aB); }
    double scale = 0.0;  // C_n (fwd) / D_n (bwd), log2 units
    float vsum = 0.f;    // Σ of every emission read: NaN / +∞ ⇒ non-finite input
    int par = 0;         // parity of the reduction buffers of the current frame

    // Store frame n's normalised values h (α̂_n or β̂_n) and u; reduce max(u) and,
    // in the backward, the log-sum-exp of x = α̂_n + β̂_n into buffers [par].
    auto emit = [&](int n, const V *h, const V *acur) {
        float *latn = (!RAW && a.lat) ? a.lat + lat_base + (size_t)n * K : nullptr;
        double *latn64 = (RAW && a.lat64) ? a.lat64 + lat_base + (size_t)n * K : nullptr;
        V lmax = NINF;
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const int j = tid + k * T;
            if (j < K && latn) latn[j] = (float)(h[k] * LN2);
            if (j < K && latn64) latn64[j] = (double)h[k];
            sts_v(a_u + (uint32_t)j * VS, uk[k]);
            if (MODE == MODE_FACTORED) sts_v(a_p + (uint32_t)j * 4, ex2((float)uk[k]));
            lmax = vmax(lmax, uk[k]);
        }
        if (!RAW) {
            lmax = warp_max_fast(lmax);
            if (lane == 0) sts_v(a_wmax + (uint32_t)(par * 32 + warp) * 8, lmax);
        }
        if (want_post) {
#pragma unroll
            for (int k = 0; k < SPT; ++k)
                xpost[k] = (tid + k * T < K) ? (RAW ? acur[k] : acur[k] * L2E) + h[k] : NINF;
        }
        if (want_post && !RAW) {
            V zm;
            float zs;
            warp_lse_vals<V, SPT>(xpost, zm, zs);
            if (lane == 0) {
                sts_v(a_wz + (uint32_t)(par * 64 + 2 * warp) * 8, zm);
                sts_v(a_wz + (uint32_t)(par * 64 + 2 * warp + 1) * 8, zs);
            }
        }
    };
    // γ of the frame whose x and Z (buffers [pp]) were produced one frame ago.
    auto posterior = [&](int pn, int pp) {
        V Z;
        if (RAW) {  // unnormalised float64 lattices: Eq. (15) with the forward's logZ
            const double z = a.logZ_in[b];
            Z = (z > -INFINITY) ? (V)(z * 1.4426950408889634) : NINF;
        } else {
            const V m = lane < W ? lds_v(a_wz + (uint32_t)(pp * 64 + 2 * lane) * 8, (V)0) : NINF;
            const float s = lane < W ? lds_v(a_wz + (uint32_t)(pp * 64 + 2 * lane + 1) * 8, 0.f) : 0.f;
            Z = block_lse_pairs<V>(m, s);
        }
        const V Zs = (Z == NINF) ? (V)0 : Z;
        if (a.post_kind == POST_STATE) {
            float *prow = a.post + lat_base + (size_t)pn * K;
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                const int j = tid + k * T;
                const float gam = (Z == NINF) ? 0.f : ex2((float)(xpost[k] - Zs));
                if (j < K) prow[j] = gam;
            }
        } else {
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                const float gam = (Z == NINF) ? 0.f : ex2((float)(xpost[k] - Zs));
                if (tid + k * T < K) sts_v(a_gbuf + 4 * (uint32_t)posk[k], gam);
            }
        }
    };
    auto block_max_prev = [&](int pp) {
        const V v = lane < W ? lds_v(a_wmax + (uint32_t)(pp * 32 + lane) * 8, (V)0) : NINF;
        return warp_max_fast(v);
    };

    // ---- first frame: π ⊗ v_0 (fwd, L6) / β̂_{N-1} = ω (bwd, L7), exact max
    {
        V h[SPT];
        V lmax = NINF;
        float vv[SPT];
        fetch_v(0, vA, vv);
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const int j = tid + k * T;
            const bool ok = j < K && viable(k, n_first);
            const float v = vv[k];
            vsum += v;
            const V v2 = (V)v * L2E;
            if (!BWD) {
                h[k] = ok ? (V)G.init2[s0 + min(j, K - 1)] + v2 : NINF;
                uk[k] = h[k];
            } else {
                h[k] = ok ? (V)G.final2[s0 + min(j, K - 1)] : NINF;
                uk[k] = h[k] + v2;
            }
            lmax = vmax(lmax, uk[k]);
        }
        if (!RAW) {
            lmax = warp_max_fast(lmax);
            if (lane == 0) sts_v(a_wmax + (uint32_t)(32 + warp) * 8, lmax);
        }
        __syncthreads();  // schedule, flag, wmax[1] visible
        V c = RAW ? (V)0 : block_max_prev(1);
        if (c == NINF) c = (V)0;
        scale = (double)c;
#pragma unroll
        for (int k = 0; k < SPT; ++k) { h[k] -= c; uk[k] -= c; }
        if (tid == 0 && a.scale) a.scale[(size_t)b * a.N_max + n_first] = scale * kLN2;
        emit(n_first, h, aA);
        load_v(n_first + 2 * dir, vA);
        if (want_post) load_alpha(n_first + 2 * dir, aA);
    }
    int n = n_first;
    int pend_n = n_first;  // frame whose posterior is pending
    auto step = [&](float (&vb)[SPT], V (&ab)[SPT]) -> bool {
        const int n_next = n + dir;
        if (BWD ? (n_next < 0) : (n_next >= N)) return false;
        __syncthreads();  // u, p, wmax[par], wz[par] of frame n visible
        ++tstep;
        tma_issue(tstep + 1, n_next + dir);  // buffer of step tstep-1 is free now
        // ---- phase A of frame n_next (+ pdf-level row of the frame finished two frames ago)
        if (pdf_post && pend_n != n) pdf_row(a, a_gbuf, a_ssp, a_pslot, gi, b, pend_n, tid, T);
        phase_a<MODE, V>(mysl, nsl, lane, a_u, a_p, a_part);
        __syncthreads();
        // ---- phase B of frame n_next
        const int pp = par;
        par ^= 1;
        if (want_post) posterior(n, pp);  // γ_n (its x is in registers, Z in wz[pp])
        pend_n = n;
        n = n_next;
        V c = RAW ? (V)0 : block_max_prev(pp);  // lagged normaliser: max of the previous u
        if (c == NINF) c = (V)0;                // no viable state: keep 0̄ everywhere
        scale += (double)c;
        if (tid == 0 && a.scale) a.scale[(size_t)b * a.N_max + n] = scale * kLN2;
        V h[SPT];
        float vv[SPT];
        fetch_v(tstep, vb, vv);
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const V y = lds_v(a_part + (uint32_t)(tid + k * T) * VS, (V)0);
            const bool ok = viable(k, n);
            const float v = vv[k];
            vsum += v;
            const V v2 = (V)v * L2E;
            if (!BWD) {
                h[k] = ok ? y + v2 - c : NINF;
                uk[k] = h[k];
            } else {
                h[k] = ok ? y - c : NINF;
                uk[k] = h[k] + v2;
            }
        }
        emit(n, h, ab);
        load_v(n + 2 * dir, vb);  // refill with the frame two steps ahead
        if (want_post) load_alpha(n + 2 * dir, ab);
        return true;
    };
    for (;;) {
        if (!step(vB, aB)) break;
        if (!step(vA, aA)) break;
    }
    // ---- flush the pending posterior rows
    if (want_post) {
        __syncthreads();  // wz[par] of the last frame visible; gbuf of pend_n complete
        if (pdf_post && pend_n != n) pdf_row(a, a_gbuf, a_ssp, a_pslot, gi, b, pend_n, tid, T);
        if (pdf_post) __syncthreads();  // gbuf free again
        posterior(n, par);
        if (pdf_post) {
            __syncthreads();
            pdf_row(a, a_gbuf, a_ssp, a_pslot, gi, b, n, tid, T);
        }
    }
    // ---- termination: logZ = C + ⊕_k α̂(k) ⊗ ω(k)  /  logZ_β = D_0 + ⊕_k π(k) ⊗ u_0(k)
    {
        V xt[SPT];
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const int j = tid + k * T;
            xt[k] = (j < K) ? uk[k] + (V)(BWD ? G.init2[s0 + j] : G.final2[s0 + j]) : NINF;
        }
        V zm;
        float zs;
        warp_lse_vals<V, SPT>(xt, zm, zs);
        if (!(vsum < INFINITY)) sts_i(a_flag, 1);
        __syncthreads();  // every reader of the reduction buffers is done
        if (lane == 0) {
            sts_v(a_wz + (uint32_t)(2 * warp) * 8, zm);
            sts_v(a_wz + (uint32_t)(2 * warp + 1) * 8, zs);
        }
        __syncthreads();
        if (warp == 0) {
            const V m = lane < W ? lds_v(a_wz + (uint32_t)(2 * lane) * 8, (V)0) : NINF;
            const float sx = lane < W ? lds_v(a_wz + (uint32_t)(2 * lane + 1) * 8, 0.f) : 0.f;
            // float64 final combine of the per-warp pairs (logZ is assembled in fp64)
            const V M = warp_max_fast(m);
            const double Md = (M == NINF) ? 0.0 : (double)M;
            double t = (m == NINF) ? 0.0 : (double)sx * exp2((double)m - Md);
#pragma unroll
            for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) {
                double z = (M == NINF) ? -INFINITY : (scale + Md + log2(t)) * kLN2;
                int stt = st;
                if (lds_i(a_flag) == 1) stt |= FB_SEQ_NONFINITE_INPUT;
                if (!(z > -INFINITY)) stt |= FB_SEQ_EMPTY_LATTICE;
                if (stt) z = -INFINITY;
                if (a.logZ) a.logZ[b] = z;
                a.status[b] = stt;
            }
        }
    }
    if (use_tma && tid == 0) {  // all TMA rows were consumed; the next sequence re-initialises
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(a_mbar) : "memory");
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(a_mbar + 8) : "memory");
    }
}

// Sequences b = blockIdx.x, blockIdx.x + gridDim.x, …  (gridDim.x = B normally;
// fewer, persistent CTAs confine the numerator pass of lfmmi_loss_grad to the
// SMs the denominator leaves idle).
template <bool BWD, int MODEX, int SPT, int MAXT>
__global__ void __launch_bounds__(MAXT, (MAXT >= 512 ? 1 : (MAXT == 256 ? 2 : 7))) k_fb(const FBArgs a) {
    for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
        fb_sequence<BWD, MODEX, SPT>(a, b);
        __syncthreads();  // shared memory is reused by the next sequence
    }
}

// ------------------------------------------------------------------ Viterbi (tropical semiring, N1)

// Max-plus phase A over the Viterbi schedule (natural-log weights, float64
// gathers): per row, the best predecessor score and its source (lowest index
// on ties, the oracle's rule).
__device__ __forceinline__ void vit_consider(double &best, int &arg, double x, int src) {
    if (x > best || (x == best && src < arg)) { best = x; arg = src; }
}

__device__ __forceinline__ void phase_a_max(uint32_t cur, int nsl, int lane, uint32_t a_u, uint32_t a_best,
                                            uint32_t a_arg) {
    for (int q = 0; q < nsl; ++q) {
        const uint32_t h = lds_u32(cur + lane * 4);
        const int row = (int)(h & 0xFFFFu) - 1, lg = (int)((h >> 16) & 7u), L2 = (int)(h >> 19);
        uint32_t ia = cur + 128 + lane * 4;
        uint32_t wa = cur + 128 + (uint32_t)L2 * 128 + lane * 8;
        double b0 = NEG_INF_D, b1 = NEG_INF_D;
        int g0 = 0x7fffffff, g1 = 0x7fffffff;
        for (int s = 0; s < L2; ++s) {
            const uint32_t ix = lds_u32(ia);
            const float2 w2 = lds_f2(wa);
            const uint32_t o0 = ix & 0xFFFFu, o1 = ix >> 16;
            vit_consider(b0, g0, lds_v(a_u + o0, 0.0) + (double)w2.x, (int)(o0 >> 3));
            vit_consider(b1, g1, lds_v(a_u + o1, 0.0) + (double)w2.y, (int)(o1 >> 3));
            ia += 128;
            wa += 256;
        }
        vit_consider(b0, g0, b1, g1);
        for (int o = 1; o < (1 << lg); o <<= 1) {
            const double bo = __shfl_xor_sync(0xffffffffu, b0, o);
            const int go = __shfl_xor_sync(0xffffffffu, g0, o);
            vit_consider(b0, g0, bo, go);
        }
        if (row >= 0) {
            sts_v(a_best + (uint32_t)row * 8, b0);
            sts_i(a_arg + (uint32_t)row * 4, b0 == NEG_INF_D ? -1 : g0);
        }
        cur += 128 + (uint32_t)L2 * 384;
    }
}

struct VitArgs {
    Graph g;
    const float *emis;
    const int *lengths;
    int B, N_max, D;
    double *score;  // [B]
    int *path;      // [B][N_max]
    int *status;    // [B]
    void *bp;       // backpointers [B][N_max][K] (int16 if K ≤ 32767 else int32)
    int bp16;
};

// One CTA per sequence: δ_0 = π ⊗ v_0; δ_n(j) = v_n(j) ⊗ max_{i→j} δ_{n-1}(i) ⊗ T_ij
// (Eq. (13) with ⊕ = max), backpointers to HBM, argmax of δ_{N-1} ⊗ ω,
// backtrace by one thread.  Float64 values, no normalisation: scores are the
// same float64 sums the oracle forms, so the tie-broken path agrees exactly.
template <int SPT, int MAXT>
__global__ void __launch_bounds__(MAXT, (MAXT == 1024 ? 1 : 2)) k_viterbi(const VitArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Graph &G = a.g;
    const Sched &S = G.vit;
    const int b = blockIdx.x;
    const int gi = (G.G == 1) ? 0 : b;
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, W = T >> 5;
    const int s0 = G.state_off[gi];
    const int K = G.state_off[gi + 1] - s0;
    const int N = a.lengths[b];
    const SmemLayout SL = smem_layout(S.bytes_max, T * SPT, true, false);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t a_u = sb + (uint32_t)SL.u, a_best = sb + (uint32_t)SL.part;
    const uint32_t a_red = sb + (uint32_t)SL.red, a_arg = sb + (uint32_t)SL.total;
    int *path = a.path + (size_t)b * a.N_max;
    for (int n = max(0, min(N, a.N_max)) + tid; n < a.N_max; n += T) path[n] = -1;
    if (N < 1 || N > a.N_max) {
        for (int n = tid; n < a.N_max; n += T) path[n] = -1;
        if (tid == 0) { a.score[b] = -INFINITY; a.status[b] = FB_SEQ_BAD_LENGTH; }
        return;
    }
    {
        const uint4 *src = (const uint4 *)(S.rec + S.rec_off[gi]);
        uint4 *dst = (uint4 *)(smem_raw + SL.rec);
        const int n16 = S.rec_bytes[gi] >> 4;
        for (int x = tid; x < n16; x += T) dst[x] = src[x];
    }
    const int nsl = S.warp_nsl[gi * W + warp];
    const uint32_t mysl = sb + (uint32_t)SL.rec + (uint32_t)S.warp_off[gi * W + warp];
    int pdfk[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const int j = tid + k * T;
        pdfk[k] = j < K ? G.pdf[s0 + j] : 0;
        sts_v(a_best + (uint32_t)j * 8, NEG_INF_D);
    }
    const float *em = a.emis + (size_t)b * a.N_max * a.D;
    const size_t bp_base = (size_t)b * a.N_max * G.K_max;  // [B][N_max][K_max]
    float vsum = 0.f;
    double dk[SPT];
    // frame 0 (natural log, float64: the same sums the oracle forms)
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const int j = tid + k * T;
        const float v = __ldg(em + pdfk[k]);
        vsum += j < K ? v : 0.f;
        dk[k] = j < K ? (double)G.init_nat[s0 + j] + (double)v : NEG_INF_D;
        sts_v(a_u + (uint32_t)j * 8, dk[k]);
    }
    for (int n = 1; n < N; ++n) {
        __syncthreads();
        phase_a_max(mysl, nsl, lane, a_u, a_best, a_arg);
        __syncthreads();
        const float *row = em + (size_t)n * a.D;
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const int j = tid + k * T;
            const double best = lds_v(a_best + (uint32_t)j * 8, 0.0);
            const float v = __ldg(row + pdfk[k]);
            vsum += j < K ? v : 0.f;
            dk[k] = (best == NEG_INF_D) ? NEG_INF_D : best + (double)v;
            sts_v(a_u + (uint32_t)j * 8, dk[k]);
            if (j < K) {
                const int arg = lds_i(a_arg + (uint32_t)j * 4);
                if (a.bp16) ((short *)a.bp)[bp_base + (size_t)n * K + j] = (short)arg;
                else ((int *)a.bp)[bp_base + (size_t)n * K + j] = arg;
            }
        }
    }
    // argmax_j δ_{N-1}(j) ⊗ ω(j), lowest index on ties
    double best = NEG_INF_D;
    int arg = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const int j = tid + k * T;
        if (j < K) vit_consider(best, arg, dk[k] + (double)G.final_nat[s0 + j], j);
    }
    for (int o = 16; o; o >>= 1) {
        const double bo = __shfl_xor_sync(0xffffffffu, best, o);
        const int go = __shfl_xor_sync(0xffffffffu, arg, o);
        vit_consider(best, arg, bo, go);
    }
    // barrier (phase-A buffers free, this CTA's backpointers visible) + non-finite vote
    const int bad = __syncthreads_or(!(vsum < INFINITY));
    if (lane == 0) {
        sts_v(a_red + (uint32_t)warp * 16, best);
        sts_i(a_red + (uint32_t)warp * 16 + 8, arg);
    }
    __syncthreads();
    if (warp == 0) {
        best = lane < W ? lds_v(a_red + (uint32_t)lane * 16, 0.0) : NEG_INF_D;
        arg = lane < W ? lds_i(a_red + (uint32_t)lane * 16 + 8) : 0x7fffffff;
        for (int o = 16; o; o >>= 1) {
            const double bo = __shfl_xor_sync(0xffffffffu, best, o);
            const int go = __shfl_xor_sync(0xffffffffu, arg, o);
            vit_consider(best, arg, bo, go);
        }
        if (lane == 0) {
            int st = 0;
            if (bad) st |= FB_SEQ_NONFINITE_INPUT;
            if (best == NEG_INF_D) st |= FB_SEQ_EMPTY_LATTICE;
            a.score[b] = st ? -INFINITY : best;
            a.status[b] = st;
            int s = st ? -1 : arg;
            for (int n = N - 1; n >= 0; --n) {
                path[n] = s;
                if (s < 0 || n == 0) continue;
                s = a.bp16 ? (int)((const short *)a.bp)[bp_base + (size_t)n * K + s]
                           : ((const int *)a.bp)[bp_base + (size_t)n * K + s];
            }
        }
    }
}

// ------------------------------------------------------------------ standalone posteriors

// One CTA per (b, n) row: Z_n = ⊕_k α̂ + β̂, γ = exp(α̂ + β̂ − Z_n) (Eq. (15)).
__global__ void __launch_bounds__(256) k_posteriors(const Graph G, const float *alpha, const float *beta,
                                                    const int *lengths, const int *status, int B, int N_max,
                                                    int D, int pdf_level, float *post) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *g = (float *)smem_raw;  // K_max
    __shared__ double wz[2 * 32];
    const int row = blockIdx.x;
    const int b = row / N_max, n = row % N_max;
    const int gi = (G.G == 1) ? 0 : b;
    const int s0 = G.state_off[gi], K = G.state_off[gi + 1] - s0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, W = blockDim.x >> 5;
    const int N = lengths[b];
    const bool zero = (N < 1 || N > N_max || n >= N || (status && status[b] != 0));
    const size_t base = (size_t)N_max * (G.G == 1 ? (size_t)b * K : (size_t)s0) + (size_t)n * K;
    if (zero) {
        if (pdf_level) for (int d = tid; d < D; d += blockDim.x) post[((size_t)b * N_max + n) * D + d] = 0.f;
        else for (int j = tid; j < K; j += blockDim.x) post[base + j] = 0.f;
        return;
    }
    float zm = NEG_INF, zs = 0.f;
    for (int j = tid; j < K; j += blockDim.x) {
        float x = (__ldg(alpha + base + j) + __ldg(beta + base + j)) * kL2E;
        g[j] = x;
        lse_push(zm, zs, x);
    }
    warp_lse(zm, zs);
    if (lane == 0) { wz[2 * warp] = zm; wz[2 * warp + 1] = zs; }
    __syncthreads();
    float Z = block_lse_from<float>(wz, W, lane);
    for (int j = tid; j < K; j += blockDim.x) {
        float gam = (Z == NEG_INF) ? 0.f : ex2(g[j] - Z);
        if (pdf_level) g[j] = gam;
        else post[base + j] = gam;
    }
    if (!pdf_level) return;
    __syncthreads();
    const PdfMap &pm = G.pm;
    const int so = pm.slot_off[gi];
    const int *ps = pm.pdf_slot + (size_t)gi * D;
    float *out = post + ((size_t)b * N_max + n) * D;
    for (int d = tid; d < D; d += blockDim.x) {
        int sl = ps[d];
        float acc = 0.f;
        if (sl >= 0)
            for (int q = pm.slot_sptr[so + sl]; q < pm.slot_sptr[so + sl + 1]; ++q) acc += g[pm.slot_states[q]];
        out[d] = acc;
    }
}

// ------------------------------------------------------------------ numerator contribution

// grad[b, n, pdf(s)] += Γ_num[b, n, s] for every numerator slot s (distinct pdfs,
// so no two threads touch one element: deterministic); sequences flagged by the
// numerator or the denominator get a zero row.  One CTA per (b, n) row.
__global__ void __launch_bounds__(256) k_add_num(float *grad, const float *gnum, const int *slot_off,
                                               const int *slot_pdf, const int *lengths, const int *den_status,
                                               const int *num_status, int N_max, int D) {
    const int b = blockIdx.y, n = blockIdx.x;
    const int N = lengths[b];
    if (N < 1 || N > N_max || n >= N) return;  // padded rows were zeroed by the den backward
    float *row = grad + ((size_t)b * N_max + n) * D;
    if ((den_status[b] | num_status[b]) != 0) {
        for (int d = threadIdx.x; d < D; d += blockDim.x) row[d] = 0.f;
        return;
    }
    const int so = slot_off[b], U = slot_off[b + 1] - so;
    const float *g = gnum + (size_t)N_max * so + (size_t)n * U;
    for (int s = threadIdx.x; s < U; s += blockDim.x) row[slot_pdf[so + s]] += g[s];
}

// ------------------------------------------------------------------ totals

// loss_b = logZ_num − logZ_den (0 for flagged sequences) and the
// fixed-order float64 totals {Σ loss, Σ N_b, Σ logZ_num, Σ logZ_den, n_bad}.
__global__ void k_totals(const double *zn, const double *zd, const int *lengths, int *status, const int *num_status,
                         int B, double *loss, double *totals) {
    __shared__ double sh[5][256];
    const int tid = threadIdx.x;
    double t[5] = {0, 0, 0, 0, 0};
    // each thread sums a contiguous chunk in ascending b; chunks combine in a fixed tree
    const int chunk = (B + blockDim.x - 1) / blockDim.x;
    for (int b = tid * chunk; b < min(B, (tid + 1) * chunk); ++b) {
        status[b] |= num_status[b];
        if (status[b] == 0) {
            double l = zn[b] - zd[b];
            loss[b] = l;
            t[0] += l;
            t[1] += (double)lengths[b];
            t[2] += zn[b];
            t[3] += zd[b];
        } else {
            loss[b] = 0.0;
            t[4] += 1.0;
        }
    }
    for (int q = 0; q < 5; ++q) sh[q][tid] = t[q];
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (tid < o)
            for (int q = 0; q < 5; ++q) sh[q][tid] += sh[q][tid + o];
        __syncthreads();
    }
    if (tid == 0)
        for (int q = 0; q < 5; ++q) totals[q] = sh[q][0];
}

// ------------------------------------------------------------------ launch helpers

using KFn = void (*)(FBArgs);

template <bool BWD, int MODE, int MAXT>
static KFn pick_spt(int spt) {
    switch (spt) {
        case 1: return k_fb<BWD, MODE, 1, MAXT>;
        case 2: return k_fb<BWD, MODE, 2, MAXT>;
        case 3: return k_fb<BWD, MODE, 3, MAXT>;
        case 4: return k_fb<BWD, MODE, 4, MAXT>;
        case 6: return k_fb<BWD, MODE, 6, MAXT>;
        default: return k_fb<BWD, MODE, 8, MAXT>;
    }
}

// MAXT = 128 variants (six CTAs per SM) and 256 (two per SM) for small CTAs; 1024 otherwise.
template <bool BWD, int MODE>
static KFn pick_t(int spt, int T) {
    if (T <= 128) return pick_spt<BWD, MODE, 128>(spt);
    if (T <= 256) return pick_spt<BWD, MODE, 256>(spt);
    if constexpr (MODE == MODE_FACTORED || MODE == kModeFactoredTma)
        if (T <= 512) return pick_spt<BWD, MODE, 512>(spt);  // ≤ 128 registers per thread
    return pick_spt<BWD, MODE, 1024>(spt);
}

static KFn pick(bool bwd, int mode, int spt, int T) {
    if (bwd) {
        if (mode == kModeFactoredTma) return pick_t<true, kModeFactoredTma>(spt, T);
        if (mode == MODE_FACTORED) return pick_t<true, MODE_FACTORED>(spt, T);
        if (mode == MODE_RAW) return pick_t<true, MODE_RAW>(spt, T);
        return pick_t<true, MODE_EXACT>(spt, T);
    }
    if (mode == kModeFactoredTma) return pick_t<false, kModeFactoredTma>(spt, T);
    if (mode == MODE_FACTORED) return pick_t<false, MODE_FACTORED>(spt, T);
    if (mode == MODE_RAW) return pick_t<false, MODE_RAW>(spt, T);
    return pick_t<false, MODE_EXACT>(spt, T);
}

static fb_status check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_cuda_error(what, (int)e); return FB_ERR_CUDA; }
    return FB_OK;
}

// idle_sms > 0: launch only as many (persistent) CTAs as fit on that many SMs.
static fb_status launch_fb(bool bwd, const FBArgs &a, cudaStream_t s, bool raw = false, int idle_sms = 0) {
    const Graph &G = a.g;
    const bool post_pdf = bwd && a.post_kind != POST_NONE && a.post_kind != POST_STATE;
    size_t sm = smem_bytes(G, bwd, post_pdf) + (post_pdf ? pdf_region(a.post_kind, G.pm.U_max, a.D).bytes : 0);
    // φ rows through TMA when they are 16-byte aligned and the two row buffers fit
    const size_t tma_bytes = fbx_a16(2 * (size_t)a.D * 4) + 16;
    FBArgs aa = a;
    aa.tma = G.mode == MODE_FACTORED && !raw && (a.D % 4 == 0) && (((uintptr_t)a.emis & 15) == 0) &&
             sm + tma_bytes <= (size_t)kSmemLimit && std::getenv("FBX_NO_TMA") == nullptr;
    if (aa.tma) sm += tma_bytes;
    KFn fn = pick(bwd, raw ? (int)MODE_RAW : (aa.tma ? kModeFactoredTma : G.mode), G.spt, G.T);
    cudaError_t e = cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) { set_cuda_error("cudaFuncSetAttribute", (int)e); return FB_ERR_CUDA; }
    {
        ProfScope ps(bwd ? (G.G == 1 ? "k_fb_bwd[G=1]" : "k_fb_bwd[G=B]") : (G.G == 1 ? "k_fb_fwd[G=1]" : "k_fb_fwd[G=B]"), s);
        int grid = a.B;
        if (idle_sms > 0) {
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, G.T, sm);
            grid = std::max(1, std::min(a.B, idle_sms * std::max(occ, 1)));
        }
        fn<<<grid, G.T, sm, s>>>(aa);
    }
    return check_launch("k_fb launch");
}

static FBArgs base_args(fb_graph g, const float *emis, const int *lengths, int B, int N_max) {
    FBArgs a;
    std::memset(&a, 0, sizeof a);
    a.g = g->g;
    a.emis = emis;
    a.lengths = lengths;
    a.B = B;
    a.N_max = N_max;
    a.D = g->g.D;
    return a;
}

// side stream + events for the concurrent numerator pass of lfmmi_loss_grad
struct SideRes {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
static std::mutex g_side_mu;
static SideRes g_side[64];

static SideRes *side_res() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_side_mu);
    SideRes &r = g_side[dev & 63];
    if (!r.s) {
        cudaStreamCreateWithFlags(&r.s, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&r.join, cudaEventDisableTiming);
    }
    return &r;
}

struct WsLayout {
    size_t den_alpha, num_alpha, gnum, zn, zd, nst, total;
};
static size_t a256(size_t x) { return (x + 255) & ~size_t(255); }
static WsLayout ws_layout(const Graph &num, const Graph &den, int B, int N_max) {
    WsLayout w;
    size_t o = 0;
    w.den_alpha = o; o += a256((size_t)B * N_max * den.K_tot * 4);
    w.num_alpha = o; o += a256((size_t)N_max * num.K_tot * 8);  // float64 when the numerator runs raw
    w.gnum = o; o += a256((size_t)N_max * num.pm.U_tot * 4);
    w.zn = o; o += a256((size_t)B * 8);
    w.zd = o; o += a256((size_t)B * 8);
    w.nst = o; o += a256((size_t)B * 4);
    w.total = o;
    return w;
}

}  // namespace fbx

using namespace fbx;

// ------------------------------------------------------------------ C ABI

extern "C" fb_status fb_forward(fb_graph g, const float *log_emis, const int32_t *lengths, int32_t B,
                                int32_t N_max, float *alpha, double *alpha_scale, double *logZ,
                                int32_t *seq_status, void *stream) {
    if (!g || !log_emis || !lengths || !logZ || !seq_status || B < 1 || N_max < 1) return FB_ERR_INVALID_ARG;
    if (!(g->g.G == 1 || g->g.G == B) || g->g.dry) return FB_ERR_INVALID_ARG;
    if (alpha && !alpha_scale) return FB_ERR_INVALID_ARG;
    FBArgs a = base_args(g, log_emis, lengths, B, N_max);
    a.lat = alpha;
    a.scale = alpha_scale;
    a.logZ = logZ;
    a.status = seq_status;
    return launch_fb(false, a, (cudaStream_t)stream);
}

extern "C" fb_status fb_backward(fb_graph g, const float *log_emis, const int32_t *lengths, int32_t B,
                                 int32_t N_max, float *beta, double *beta_scale, double *logZ_beta,
                                 const float *alpha, float *post, int32_t pdf_level, int32_t *seq_status,
                                 void *stream) {
    if (!g || !log_emis || !lengths || !seq_status || B < 1 || N_max < 1) return FB_ERR_INVALID_ARG;
    if (!(g->g.G == 1 || g->g.G == B) || g->g.dry) return FB_ERR_INVALID_ARG;
    if (post && !alpha) return FB_ERR_INVALID_ARG;
    if (pdf_level != 0 && pdf_level != 1) return FB_ERR_INVALID_ARG;
    FBArgs a = base_args(g, log_emis, lengths, B, N_max);
    a.lat = beta;
    a.scale = beta_scale;
    a.logZ = logZ_beta;
    a.status = seq_status;
    a.alpha = alpha;
    a.post = post;
    a.post_kind = post ? (pdf_level ? POST_PDF_DENSE : POST_STATE) : POST_NONE;
    return launch_fb(true, a, (cudaStream_t)stream);
}

extern "C" fb_status fb_posteriors(fb_graph g, const float *alpha, const float *beta, const int32_t *lengths,
                                   const int32_t *seq_status, int32_t B, int32_t N_max, int32_t pdf_level,
                                   float *post, void *stream) {
    if (!g || !alpha || !beta || !lengths || !post || B < 1 || N_max < 1) return FB_ERR_INVALID_ARG;
    if (!(g->g.G == 1 || g->g.G == B) || g->g.dry) return FB_ERR_INVALID_ARG;
    if (pdf_level != 0 && pdf_level != 1) return FB_ERR_INVALID_ARG;
    const Graph &G = g->g;
    cudaStream_t s = (cudaStream_t)stream;
    size_t sm = (size_t)G.K_max * 4;
    cudaError_t e = cudaFuncSetAttribute((const void *)k_posteriors, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) { set_cuda_error("cudaFuncSetAttribute", (int)e); return FB_ERR_CUDA; }
    {
        ProfScope ps("k_posteriors", s);
        k_posteriors<<<(unsigned)((size_t)B * N_max), 256, sm, s>>>(G, alpha, beta, lengths, seq_status, B, N_max,
                                                                  G.D, pdf_level, post);
    }
    return check_launch("k_posteriors launch");
}

extern "C" size_t fb_workspace_bytes(fb_graph num, fb_graph den, int32_t B, int32_t N_max) {
    if (!num || !den || B < 1 || N_max < 1) return 0;
    return ws_layout(num->g, den->g, B, N_max).total;
}

extern "C" fb_status lfmmi_loss_grad(fb_graph num, fb_graph den, const float *log_emis, const int32_t *lengths,
                                     int32_t B, int32_t N_max, float *grad, double *loss, double *totals,
                                     int32_t *seq_status, void *workspace, size_t workspace_bytes,
                                     void *stream) {
    if (!num || !den || !log_emis || !lengths || !grad || !loss || !totals || !seq_status || B < 1 || N_max < 1)
        return FB_ERR_INVALID_ARG;
    if (num->g.G != B || den->g.G != 1 || num->g.D != den->g.D || num->g.dry || den->g.dry)
        return FB_ERR_INVALID_ARG;
    WsLayout L = ws_layout(num->g, den->g, B, N_max);
    if (!workspace || workspace_bytes < L.total) return FB_ERR_WORKSPACE;
    unsigned char *ws = (unsigned char *)workspace;
    float *den_alpha = (float *)(ws + L.den_alpha);
    float *num_alpha = (float *)(ws + L.num_alpha);
    double *num_alpha64 = (double *)(ws + L.num_alpha);
    const bool raw = num->g.mode == MODE_EXACT;  // numerator pass without per-frame normalisation
    float *gnum = (float *)(ws + L.gnum);
    double *zn = (double *)(ws + L.zn), *zd = (double *)(ws + L.zd);
    int *nst = (int *)(ws + L.nst);
    cudaStream_t s = (cudaStream_t)stream;
    SideRes *sr = side_res();
    fb_status r;
    // The fork point is recorded before the denominator forward so the numerator
    // pass depends only on prior work; the denominator forward is submitted first:
    // its B CTAs each take a whole SM (registers and shared memory), so the
    // numerator CTAs land on the SMs it leaves idle and the two run concurrently.
    cudaEventRecord(sr->fork, s);
    {
        FBArgs a = base_args(den, log_emis, lengths, B, N_max);
        a.lat = den_alpha; a.logZ = zd; a.status = seq_status;
        if ((r = launch_fb(false, a, s)) != FB_OK) return r;
    }
    cudaStreamWaitEvent(sr->s, sr->fork, 0);
    // SMs the denominator passes leave idle (one den CTA per SM)
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int idle = nsm - std::min(B, nsm);
    const int confine = idle >= 8 ? idle : 0;
    {
        FBArgs a = base_args(num, log_emis, lengths, B, N_max);
        a.logZ = zn; a.status = nst;
        if (raw) a.lat64 = num_alpha64; else a.lat = num_alpha;
        if ((r = launch_fb(false, a, sr->s, raw, confine)) != FB_OK) return r;
        FBArgs c = base_args(num, log_emis, lengths, B, N_max);
        c.status = nst; c.post = gnum; c.post_kind = POST_PDF_COMPACT;
        if (raw) { c.alpha64 = num_alpha64; c.logZ_in = zn; } else c.alpha = num_alpha;
        if ((r = launch_fb(true, c, sr->s, raw, confine)) != FB_OK) return r;
    }
    cudaEventRecord(sr->join, sr->s);
    // denominator backward + fused −Γ_den gradient epilogue: independent of the numerator
    {
        FBArgs c = base_args(den, log_emis, lengths, B, N_max);
        c.status = seq_status; c.alpha = den_alpha;
        c.post = grad; c.post_kind = POST_GRAD;
        if ((r = launch_fb(true, c, s)) != FB_OK) return r;
    }
    cudaStreamWaitEvent(s, sr->join, 0);
    {
        ProfScope ps("k_add_num", s);
        k_add_num<<<dim3((unsigned)N_max, (unsigned)B), 256, 0, s>>>(grad, gnum, num->g.pm.slot_off,
                                                                    num->g.pm.slot_pdf, lengths, seq_status, nst,
                                                                    N_max, num->g.D);
    }
    if ((r = check_launch("k_add_num launch")) != FB_OK) return r;
    {
        ProfScope ps("k_totals", s);
        k_totals<<<1, 256, 0, s>>>(zn, zd, lengths, seq_status, nst, B, loss, totals);
    }
    return check_launch("k_totals launch");
}

extern "C" size_t fb_viterbi_workspace_bytes(fb_graph g, int32_t B, int32_t N_max) {
    if (!g || B < 1 || N_max < 1) return 0;
    const Graph &G = g->g;
    const size_t per = G.K_max <= 32767 ? 2 : 4;
    return (size_t)B * G.K_max * (size_t)N_max * per + 256;
}

extern "C" fb_status fb_viterbi(fb_graph g, const float *log_emis, const int32_t *lengths, int32_t B,
                                int32_t N_max, double *score, int32_t *path, int32_t *seq_status,
                                void *workspace, size_t workspace_bytes, void *stream) {
    if (!g || !log_emis || !lengths || !score || !path || !seq_status || B < 1 || N_max < 1) return FB_ERR_INVALID_ARG;
    if (!(g->g.G == 1 || g->g.G == B) || g->g.dry) return FB_ERR_INVALID_ARG;
    if (!g->g.vit_ok) return FB_ERR_UNSUPPORTED;
    if (!workspace || workspace_bytes < fb_viterbi_workspace_bytes(g, B, N_max)) return FB_ERR_WORKSPACE;
    const Graph &G = g->g;
    VitArgs a;
    std::memset(&a, 0, sizeof a);
    a.g = G;
    a.emis = log_emis;
    a.lengths = lengths;
    a.B = B;
    a.N_max = N_max;
    a.D = G.D;
    a.score = score;
    a.path = path;
    a.status = seq_status;
    a.bp = workspace;
    a.bp16 = G.K_max <= 32767;
    using VFn = void (*)(VitArgs);
    VFn fn;
    const bool small = G.T <= 256;
    switch (G.spt) {
        case 1: fn = small ? k_viterbi<1, 256> : k_viterbi<1, 1024>; break;
        case 2: fn = small ? k_viterbi<2, 256> : k_viterbi<2, 1024>; break;
        case 3: fn = small ? k_viterbi<3, 256> : k_viterbi<3, 1024>; break;
        case 4: fn = small ? k_viterbi<4, 256> : k_viterbi<4, 1024>; break;
        case 6: fn = small ? k_viterbi<6, 256> : k_viterbi<6, 1024>; break;
        default: fn = small ? k_viterbi<8, 256> : k_viterbi<8, 1024>; break;
    }
    const size_t sm = viterbi_smem_bytes(G);
    cudaError_t e = cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) { set_cuda_error("cudaFuncSetAttribute", (int)e); return FB_ERR_CUDA; }
    cudaStream_t s = (cudaStream_t)stream;
    {
        ProfScope ps("k_viterbi", s);
        fn<<<B, G.T, sm, s>>>(a);
    }
    return check_launch("k_viterbi launch");
}

extern "C" void fb_profile_enable(int32_t on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = on != 0;
}

extern "C" void fb_profile_reset(void) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto &r : g_prof) { g_event_pool.push_back(r.a); g_event_pool.push_back(r.b); }
    g_prof.clear();
}

extern "C" fb_status fb_profile_collect(const char **names, int64_t *counts, double *ms, int32_t cap, int32_t *n) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    std::vector<const char *> nm;
    std::vector<int64_t> ct;
    std::vector<double> tm;
    for (auto &r : g_prof) {
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e != cudaSuccess) { set_cuda_error("cudaEventSynchronize", (int)e); return FB_ERR_CUDA; }
        float x = 0.f;
        cudaEventElapsedTime(&x, r.a, r.b);
        size_t i = 0;
        for (; i < nm.size(); ++i)
            if (std::strcmp(nm[i], r.name) == 0) break;
        if (i == nm.size()) { nm.push_back(r.name); ct.push_back(0); tm.push_back(0.0); }
        ct[i] += 1;
        tm[i] += x;
    }
    int m = (int)std::min<size_t>(nm.size(), (size_t)std::max(0, cap));
    for (int i = 0; i < m; ++i) {
        if (names) names[i] = nm[i];
        if (counts) counts[i] = ct[i];
        if (ms) ms[i] = tm[i];
    }
    if (n) *n = m;
    return FB_OK;
}

extern "C" const char *fb_status_str(fb_status s) {
    switch (s) {
        case FB_OK: return "ok";
        case FB_ERR_INVALID_ARG: return "invalid argument";
        case FB_ERR_SHAPE: return "shape mismatch";
        case FB_ERR_INVALID_GRAPH: return "invalid graph";
        case FB_ERR_CUDA: return "CUDA error";
        case FB_ERR_NOMEM: return "out of device memory";
        case FB_ERR_WORKSPACE: return "workspace too small";
        case FB_ERR_UNSUPPORTED: return "unsupported graph size for this build";
    }
    return "unknown status";
}

extern "C" const char *fb_last_cuda_error(void) {
    std::lock_guard<std::mutex> lk(g_err_mu);
    return g_err.c_str();
}
