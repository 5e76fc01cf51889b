// fb_device.cuh — device code of the forward/backward recursion kernel k_fb
// (shared by the kernel-instantiation units fb_inst.cu and the launcher
// fb_kernels.cu; see the top of fb_kernels.cu for the per-frame schedule).
#pragma once
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
    float *post;        // state / dense pdf / compact pdf / grad (−Γ_den; k_add_num adds Γ_num)
    int tma;            // stage φ rows in shared memory with TMA bulk copies
    int lat_int;        // private lfmmi α̂ lattice: one-CTA kernel rows of K; cluster kernel [cluster][n][K_int][S], log2
                        // (a private lfmmi workspace: coalesced stores and reloads)
    // MODE_RAW (lfmmi numerator): float64 log2 lattices, posteriors normalised by logZ_in
    double *lat64;
    const double *alpha64;
    const double *logZ_in;
    // kModeGradIZ (lfmmi den backward): the forward's per-frame offsets C_n (natural log,
    // [B][N_max]) and log Z, so the posterior normaliser of frame n is known up front:
    // Ẑ_n = log Z − C_n − D_n (Eq. (1) invariant)
    const double *ascale_in;
    const double *logZ_fwd;
};

// Exact max-then-sum over one row held by g lanes (fallback of factored mode,
// where weights are stored as e^{T}); `cur` is the slice, `lane` the group
// leader.  Accurate libm ops; rare.
static __device__ __noinline__ float exact_row(uint32_t cur, int L2, int g, int lane, uint32_t a_u,
                                               unsigned long long *ctr) {
    atomicAdd(ctr, 1ull);  // diagnostic: rows that needed the fallback (fb_graph_counters)
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
                                        uint32_t a_part, unsigned long long *ctr) {
    constexpr float kTiny = 8.271806125530277e-25f;  // 2^-80
    constexpr float kHuge = 1.329227995784916e+36f;  // 2^120
    constexpr uint32_t VS = sizeof(V);
    for (int q = 0; q < nsl; ++q) {
        const uint32_t h = lds_u32(cur + lane * 4);
        const int row = (int)(h & 0xFFFFu) - 1, lg = (int)((h >> 16) & 7u), L2 = (int)(h >> 19);
        uint32_t ia = cur + 128 + lane * 4;
        uint32_t wa = cur + 128 + (uint32_t)L2 * 128 + lane * 8;
        if (MODE == MODE_FACTORED) {
            float2 a2 = make_float2(0.f, 0.f);  // two accumulators, one packed FFMA2 per arc pair
#pragma unroll 1
            for (int s = 0; s < L2; ++s) {
                const uint32_t ix = lds_u32(ia);
                const float2 w2 = lds_f2(wa);
                const float p0 = lds_v(a_p + (ix & 0xFFFFu), 0.f), p1 = lds_v(a_p + (ix >> 16), 0.f);
                a2 = __ffma2_rn(make_float2(p0, p1), w2, a2);
                ia += 128;
                wa += 256;
            }
            float acc = a2.x + a2.y;
            if (lg) {
                for (int o = 1; o < (1 << lg); o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            }
            if (row >= 0)
                sts_v(a_part + (uint32_t)row * VS,
                      (V)((acc >= kTiny && acc <= kHuge) ? lg2(acc) : exact_row(cur, L2, 1 << lg, lane, a_u, ctr)));
        } else if (L2 <= 2) {
            // ≤ 4 arcs per lane (every slice of an exact-mode schedule with Lmax = 4 unless a
            // row exceeds 32 lanes × 4 arcs): gather all, then max-then-sum — no online
            // rescaling chain.  Null slots carry weight −∞ (x = −∞, 2^{x−m} = 0).
            const uint32_t ix0 = lds_u32(ia);
            const float2 w0 = lds_f2(wa);
            const V x0 = lds_v(a_u + (ix0 & 0xFFFFu), (V)0) + (V)w0.x;
            const V x1 = lds_v(a_u + (ix0 >> 16), (V)0) + (V)w0.y;
            V x2 = ninf<V>(), x3 = ninf<V>();
            if (L2 == 2) {
                const uint32_t ix1 = lds_u32(ia + 128);
                const float2 w1 = lds_f2(wa + 256);
                x2 = lds_v(a_u + (ix1 & 0xFFFFu), (V)0) + (V)w1.x;
                x3 = lds_v(a_u + (ix1 >> 16), (V)0) + (V)w1.y;
            }
            V m0 = fmax(fmax(x0, x1), fmax(x2, x3));
            const V ms = (m0 == ninf<V>()) ? (V)0 : m0;
            float s0 = (ex2((float)(x0 - ms)) + ex2((float)(x1 - ms))) + (ex2((float)(x2 - ms)) + ex2((float)(x3 - ms)));
            for (int o = 1; o < (1 << lg); o <<= 1) {
                V m2 = __shfl_xor_sync(0xffffffffu, m0, o);
                float s2 = __shfl_xor_sync(0xffffffffu, s0, o);
                lse_combine(m0, s0, m2, s2);
            }
            if (row >= 0) sts_v(a_part + (uint32_t)row * VS, (m0 == ninf<V>()) ? m0 : m0 + (V)lg2(s0));
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
#pragma unroll 1
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

// Phase A of the exp-factorised ⊕ (factored mode, the one-CTA den kernels): the same
// walk as phase_a<MODE_FACTORED>, with the per-slice bookkeeping cut down.
//  • the warp's first nsl0 slices hold unsplit rows (g = 1, fb_graph.cpp) and run in a
//    loop without the xor-combine; the split-row slices follow;
//  • the arc loop is a do-while over an end address (every slice has L ≥ 2 slots);
//  • every lane stores: lead = row + 1 for row leaders, 0 otherwise, so the store goes to
//    part[row] or to the scratch cell part[-1] (a_partm1 = &part[-1]) — no branch.  Only a
//    leader whose sum leaves [2^-80, 2^120] takes the exact fallback.
__device__ __forceinline__ void phase_a_fact(uint32_t cur, int nsl0, int nsl, int lane, uint32_t a_u, uint32_t a_p,
                                             uint32_t a_partm1, unsigned long long *ctr) {
    constexpr float kTiny = 8.271806125530277e-25f;  // 2^-80
    constexpr float kHuge = 1.329227995784916e+36f;  // 2^120
    const uint32_t l4 = (uint32_t)lane * 4u, l8 = (uint32_t)lane * 8u;
    auto slice = [&](auto split) {
        const uint32_t h = lds_u32(cur + l4);
        const uint32_t L2 = h >> 19;
        uint32_t ia = cur + 128u + l4;
        uint32_t wa = cur + 128u + L2 * 128u + l8;
        const uint32_t iend = ia + L2 * 128u;
        float2 a2 = make_float2(0.f, 0.f);
#pragma unroll 1
        do {
            const uint32_t ix = lds_u32(ia);
            const float2 w2 = lds_f2(wa);
            const float p0 = lds_v(a_p + (ix & 0xFFFFu), 0.f), p1 = lds_v(a_p + (ix >> 16), 0.f);
            a2 = __ffma2_rn(make_float2(p0, p1), w2, a2);
            ia += 128u;
            wa += 256u;
        } while (ia != iend);
        float acc = a2.x + a2.y;
        int g = 1;
        if (decltype(split)::value) {
            g = 1 << ((h >> 16) & 7u);
            for (int o = 1; o < g; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        }
        const uint32_t lead = h & 0xFFFFu;
        float v = lg2(acc);
        if (!(acc >= kTiny && acc <= kHuge) && lead) v = exact_row(cur, (int)L2, g, lane, a_u, ctr);
        sts_v(a_partm1 + lead * 4u, v);
        cur += 128u + L2 * 384u;
    };
    int q = 0;
    for (; q < nsl0; ++q) slice(std::false_type());
    for (; q < nsl; ++q) slice(std::true_type());
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
__device__ __forceinline__ void pdf_row(const FBArgs &a, uint32_t a_gbuf, uint32_t a_ssp, uint32_t a_pq, int gi,
                                        int b, int n, int tid, int T, float mul) {
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
    // dense / grad: pdf d sums its run gbuf[q0, q0 + count) of pq[d]
    const int D = a.D;
    float *row = a.post + ((size_t)b * a.N_max + n) * D;
    // mul: +1 (posteriors), −1 (grad: −Γ_den; Γ_num added by k_add_num), or −1/S when gbuf
    // holds unnormalised e = γ·S (kModeGradIZ)
    const float sgn = mul;
    auto run = [&](uint32_t w) {
        const uint32_t q0 = w & 0xFFFFu, c = w >> 16;
        float acc = 0.f;
        if (c >= 1) acc = lds_v(a_gbuf + 4 * q0, 0.f);  // ≤ 2 states per pdf branch-free, a loop beyond
        if (c >= 2) acc += lds_v(a_gbuf + 4 * (q0 + 1), 0.f);
        for (uint32_t i = 2; i < c; ++i) acc += lds_v(a_gbuf + 4 * (q0 + i), 0.f);
        return sgn * acc;
    };
    if ((D & 1) == 0 && ((uintptr_t)a.post & 7) == 0) {  // pairs of pdfs: one 8-byte map load, one 8-byte store
        for (int i = tid; 2 * i < D; i += T) {
            uint32_t w0, w1;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w0), "=r"(w1) : "r"(a_pq + 8 * (uint32_t)i));
            *reinterpret_cast<float2 *>(row + 2 * i) = make_float2(run(w0), run(w1));
        }
    } else {
        for (int d = tid; d < D; d += T) row[d] = run(lds_u32(a_pq + 4 * (uint32_t)d));
    }
}

// The gradient row of the IZ backward when no pdf has more than two states: pq[d] holds two
// byte offsets into the γ buffer (a state's e, or a zero cell), so a pdf costs two loads and
// an add — no count decode, no branches.
__device__ __forceinline__ void pdf_row_pair2(const FBArgs &a, uint32_t a_gbuf, uint32_t a_pq, int b, int n, int tid,
                                              int T, float mul) {
    const int D = a.D;
    float *row = a.post + ((size_t)b * a.N_max + n) * D;
    auto run = [&](uint32_t w) { return mul * (lds_v(a_gbuf + (w & 0xFFFFu), 0.f) + lds_v(a_gbuf + (w >> 16), 0.f)); };
    if ((D & 1) == 0 && ((uintptr_t)a.post & 7) == 0) {
        for (int i = tid; 2 * i < D; i += T) {
            uint32_t w0, w1;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w0), "=r"(w1) : "r"(a_pq + 8 * (uint32_t)i));
            *reinterpret_cast<float2 *>(row + 2 * i) = make_float2(run(w0), run(w1));
        }
    } else {
        for (int d = tid; d < D; d += T) row[d] = run(lds_u32(a_pq + 4 * (uint32_t)d));
    }
}

// Zero (posterior) / −∞ (lattice) rows for frames [n0, n1).
inline __device__ void write_pad_rows(const FBArgs &a, int gi, int b, int K, int s0, int n0, int n1, int tid, int T,
                               bool lattice, bool bwd) {
    const Graph &G = a.g;
    const size_t lat_base = (size_t)a.N_max * (G.G == 1 ? (size_t)b * K : (size_t)s0);
    for (int n = n0; n < n1; ++n) {
        if (lattice && a.lat && !a.lat_int)  // a private lfmmi lattice is never read past N_b
            for (int j = tid; j < K; j += T) a.lat[lat_base + (size_t)n * K + j] = NEG_INF;
        if (lattice && a.scale && !a.lat_int && tid == 0) a.scale[(size_t)b * a.N_max + n] = 0.0;
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
// arithmetic with φ rows staged through TMA), or kModeGradIZ (the same, backward
// with the −Γ_den gradient epilogue normalised through the forward's log Z).
//
// kModeGradIZ epilogue.  By Eq. (1) Σ_k α_n(k) β_n(k) = Z at every n, so in
// the normalised log2 units of the kernels the posterior normaliser of frame n is
// Ẑ_n = log2 Z − C_n − D_n, known before the frame is computed (C_n: the forward's
// offsets, D_n: this pass's).  Phase B then forms e_k = 2^{α̂_n(k) + β̂_n(k) − Ẑ_n}
// (one ex2 per state) straight into the γ buffer and sums it per warp; the next
// frame's phase A sums the 32 partials (every warp redundantly: no extra barrier)
// and writes the gradient row −Σ_{k∈pdf} e_k / S.  Dividing by the computed
// S = Σ_k e_k (≈ 1, off by the float32 rounding of the two recursions) keeps
// Σ_k γ_n(k) = 1 exactly as the two-pass max-then-sum normaliser did; it replaces
// that pass's per-state max reduction and second ex2, and the one-frame lag of γ.
constexpr int kModeFactoredTma = 4;
constexpr int kModeGradIZ = 5;
template <bool BWD, int MODEX, int SPT, int TT>
__device__ __forceinline__ void fb_sequence(const FBArgs &a, const int b) {
    constexpr bool IZ = BWD && MODEX == kModeGradIZ;
    constexpr bool TMA = MODEX == kModeFactoredTma || MODEX == kModeGradIZ;
    constexpr int MODE = TMA ? (int)MODE_FACTORED : MODEX;
    using V = typename std::conditional<MODE == MODE_FACTORED, float, double>::type;
    constexpr uint32_t VS = sizeof(V);
    constexpr bool RAW = MODE == MODE_RAW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Graph &G = a.g;
    const int gi = (G.G == 1) ? 0 : b;
    constexpr int T = TT, W = TT >> 5;  // the launch uses exactly TT threads (compile-time offsets)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s0 = G.state_off[gi];
    const int K = G.state_off[gi + 1] - s0;
    const int N = a.lengths[b];
    const Sched &S = BWD ? G.bwd : G.fwd;
    const bool want_post = IZ || (BWD && a.post_kind != POST_NONE);
    const bool pdf_post = IZ || (want_post && a.post_kind != POST_STATE);
    const SmemLayout SL = smem_layout(S.bytes_max, T * SPT, MODE != MODE_FACTORED, want_post && pdf_post);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t a_u = sb + (uint32_t)SL.u, a_p = sb + (uint32_t)SL.p, a_part = sb + (uint32_t)SL.part;
    const uint32_t a_wmax = sb + (uint32_t)SL.red, a_wz = a_wmax + 64 * 8, a_flag = a_wmax + 192 * 8;
    const uint32_t a_cz = a_wmax + 193 * 8;  // [2][2] V: (c, Z) of a frame, computed once by warp 0
    const PdfRegion PR = pdf_region(a.post_kind, G.pm.U_max, a.D);
    unsigned short *ssp = (unsigned short *)(smem_raw + SL.total + PR.ssp);
    uint32_t *pq = (uint32_t *)(smem_raw + SL.total + PR.pq);
    const uint32_t a_gbuf = sb + (uint32_t)SL.gbuf;
    // φ row staging (TMA): two row buffers + two mbarriers after the pdf region
    constexpr bool use_tma = TMA;
    const uint32_t rowbytes = (uint32_t)a.D * 4;
    const uint32_t a_ebuf = sb + (uint32_t)(SL.total + PR.bytes);
    const uint32_t a_mbar = a_ebuf + (uint32_t)fbx_a16(2 * (size_t)rowbytes);
    const uint32_t a_ssp = sb + (uint32_t)(SL.total + PR.ssp), a_pq = sb + (uint32_t)(SL.total + PR.pq);
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
    // IZ gradient rows with ≤ 2 states per pdf and a spare γ slot: the two-offset pq form
    const bool pair2 = IZ && G.pm.spp_max <= 2 && K < T * SPT && T * SPT * 4 <= 65536;
    // pdf-level epilogue maps → shared memory
    if (pdf_post) {
        const int so = G.pm.slot_off[gi], U = G.pm.slot_off[gi + 1] - so;
        const int base = G.pm.slot_sptr[so];
        if (a.post_kind == POST_PDF_COMPACT)
            for (int x = tid; x <= U; x += T) ssp[x] = (unsigned short)(G.pm.slot_sptr[so + x] - base);
        else
            for (int d = tid; d < a.D; d += T) {
                const int sl = G.pm.pdf_slot[(size_t)gi * a.D + d];
                const int q0 = sl < 0 ? 0 : G.pm.slot_sptr[so + sl] - base;
                const int c = sl < 0 ? 0 : G.pm.slot_sptr[so + sl + 1] - G.pm.slot_sptr[so + sl];
                if (pair2) {  // byte offsets of the pdf's (up to) two states, else of the zero cell
                    const uint32_t z = (uint32_t)(T * SPT - 1) * 4u;
                    pq[d] = (c >= 1 ? (uint32_t)q0 * 4u : z) | ((c >= 2 ? (uint32_t)(q0 + 1) * 4u : z) << 16);
                } else {
                    pq[d] = (uint32_t)q0 | ((uint32_t)c << 16);
                }
            }
        if (pair2 && tid == 0) sts_v(a_gbuf + (uint32_t)(T * SPT - 1) * 4u, 0.f);  // the zero cell (never a state's)
    }
    const int nsl = S.warp_nsl[gi * W + warp];
    const int nsl0 = S.warp_nsl0[gi * W + warp];
    const uint32_t mysl = sb + (uint32_t)SL.rec + (uint32_t)S.warp_off[gi * W + warp];
    const bool use_mask = BWD ? G.mask_bwd : G.mask_fwd;

    // Owned states j = tid + k*T (k < SPT).  Slots with j ≥ K are inert: their
    // partial stays 0̄, they are never viable (distance kInert) and never stored to
    // HBM, and they read the emission column of the member's state 0 — a column the
    // recursion reads anyway, so the non-finite check (vsum) sees exactly the
    // columns the graph reads (fb.h; the oracle's rule).
    constexpr int kInert = 0x3fffffff;
    int pdfk[SPT];   // emission column
    int distk[SPT];  // viability distance
    int posk[SPT];   // position in the slot-ordered γ buffer (pdf-level epilogue)
    const int pdf0 = G.pdf[s0];
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const int j = tid + k * T;
        pdfk[k] = pdf0;
        distk[k] = kInert;
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
        const size_t ro = lat_base + (size_t)min(max(n, 0), N - 1) * K + tid;  // one base pointer, immediate offsets
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const bool in = tid + k * T < K;
            // coherent L2 load: in k_fb_num this lattice was written by the same kernel
            if (RAW) v[k] = in ? (V)__ldcg(a.alpha64 + ro + k * T) : (V)0;
            else v[k] = in ? (V)__ldg(a.alpha + ro + k * T) : (V)0;
        }
    };
    // viable(k, n): forward — a final state is reachable in the N-1-n remaining
    // transitions; backward — the state is reachable from an initial state in n.
    // (graphs without masked states: every real state has distance 0, so the test
    // only rejects the inert slots)
    auto viable = [&](int k, int n) {
        return use_mask ? (BWD ? (distk[k] <= n) : (distk[k] <= N - 1 - n)) : distk[k] == 0;
    };

    // Ping-pong prefetch buffers (A: even steps, B: odd steps): a buffer is
    // consumed by its frame's phase B and immediately refilled with the frame
    // two steps ahead, so loads have a whole frame of slack and no register moves.
    float vA[SPT], vB[SPT];  // emissions
    V aA[SPT], aB[SPT];      // α̂ (backward epilogue), log2 units
    V uk[SPT];               // this thread's entries of the current vector u (log2)
    V xpost[SPT];            // α̂_n + β̂_n of the frame whose posterior is pending (not IZ)
    double scale = 0.0;      // C_n (fwd) / D_n (bwd), log2 units
    const float psgn = a.post_kind == POST_GRAD ? -1.f : 1.f;
    // IZ: log2 Z of the forward, and the normaliser Ẑ of the frame being emitted
    const double logZ2 = IZ ? a.logZ_fwd[b] * 1.4426950408889634 : 0.0;
    float zhat = 0.f;
    const uint32_t a_cnb = a_cz + 4u * 8u;  // IZ: [2] double, the forward's C of the next two steps' frames
    auto zhat_of = [&](double cn_nat) { return (float)(logZ2 - cn_nat * 1.4426950408889634 - scale); };
    const int dir = BWD ? -1 : 1;
    const int n_first = BWD ? N - 1 : 0;
    load_v(n_first, vA);
    load_v(n_first + dir, vB);
    tma_issue(0, n_first);
    tma_issue(1, n_first + dir);
    int tstep = 0;  // index of the frame being produced (t in tma_issue / fetch_v)
    if (want_post) { load_alpha(n_first, aA); load_alpha(n_first + dir, aB); }
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
        if (IZ) {  // e_k = 2^{α̂ + β̂ − Ẑ_n} into the γ buffer; per-warp Σ e
            float es = 0.f;
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                const float e = ex2((float)(acur[k] * L2E + h[k]) - zhat);  // 0 for non-viable / inert
                if (tid + k * T < K) sts_v(a_gbuf + 4 * (uint32_t)posk[k], e);
                es += e;
            }
            es = warp_sum(es);
            if (lane == 0) sts_v(a_wz + (uint32_t)(par * 64 + warp) * 8, es);
        }
        if (want_post && !IZ) {
#pragma unroll
            for (int k = 0; k < SPT; ++k)
                xpost[k] = (tid + k * T < K) ? (RAW ? acur[k] : acur[k] * L2E) + h[k] : NINF;
        }
        if (want_post && !RAW && !IZ) {
            V zm;
            float zs;
            warp_lse_vals<V, SPT>(xpost, zm, zs);
            if (lane == 0) {
                sts_v(a_wz + (uint32_t)(par * 64 + 2 * warp) * 8, zm);
                sts_v(a_wz + (uint32_t)(par * 64 + 2 * warp + 1) * 8, zs);
            }
        }
    };
    // γ of the frame whose x and Z (buffers [pp]) were produced one frame ago;
    // from_cz: Z was reduced once by warp 0 into cz[pp] (the steady-state step)
    auto posterior = [&](int pn, int pp, bool from_cz) {
        V Z;
        if (RAW) {  // unnormalised float64 lattices: Eq. (15) with the forward's logZ
            const double z = a.logZ_in[b];
            Z = (z > -INFINITY) ? (V)(z * 1.4426950408889634) : NINF;
        } else if (from_cz) {
            Z = lds_v(a_cz + (uint32_t)(2 * pp + 1) * 8, (V)0);
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
    auto iz_row = [&](int pn, int pp) {
        float sv = lane < W ? lds_v(a_wz + (uint32_t)(pp * 64 + lane) * 8, 0.f) : 0.f;
        sv = warp_sum(sv);  // every warp the same S (same partials, same order)
        const float mul = (sv > 0.f && sv < INFINITY) ? -__fdividef(1.f, sv) : 0.f;
        if (pair2) pdf_row_pair2(a, a_gbuf, a_pq, b, pn, tid, T, mul);
        else pdf_row(a, a_gbuf, a_ssp, a_pq, gi, b, pn, tid, T, mul);
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
        if (IZ) {
            zhat = zhat_of(a.ascale_in[(size_t)b * a.N_max + n_first]);
            if (tid == 0)  // C of the first step's frame (step 1) → cnb[1]
                sts_v(a_cnb + 8u, (double)a.ascale_in[(size_t)b * a.N_max + min(max(n_first + dir, 0), N - 1)]);
        }
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
        // IZ: the lagged normaliser c, the float64 offset and Ẑ of frame n_next are formed here,
        // off phase B's dependency chain (every warp reduces the per-warp maxima itself: an
        // exact max, the same in every warp)
        V c_iz = (V)0;
        if (IZ) {
            c_iz = block_max_prev(par);
            if (c_iz == NINF) c_iz = (V)0;
            scale += (double)c_iz;
            double cn;  // C of frame n_next: cp.async'd into cnb[tstep & 1] a step ago by thread 0
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(cn) : "r"(a_cnb + 8u * (uint32_t)(tstep & 1)));
            zhat = zhat_of(cn);
            if (tid == 0) {  // the next step's C (lands during this frame; waited at its end)
                const int nn = min(max(n_next + dir, 0), N - 1);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a_cnb + 8u * (uint32_t)((tstep + 1) & 1)),
                             "l"(a.ascale_in + (size_t)b * a.N_max + nn) : "memory");
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
        }
        if (!RAW && !IZ && warp == 0) {  // the frame's normaliser c and posterior Z, reduced once (read after the next barrier)
            const V cmax = block_max_prev(par);
            V Zr = (V)0;
            if (want_post && !IZ) {
                const V m = lane < W ? lds_v(a_wz + (uint32_t)(par * 64 + 2 * lane) * 8, (V)0) : NINF;
                const float s2 = lane < W ? lds_v(a_wz + (uint32_t)(par * 64 + 2 * lane + 1) * 8, 0.f) : 0.f;
                Zr = block_lse_pairs<V>(m, s2);
            }
            if (lane == 0) {
                sts_v(a_cz + (uint32_t)(2 * par) * 8, cmax);
                sts_v(a_cz + (uint32_t)(2 * par + 1) * 8, Zr);
            }
        }
        // ---- phase A of frame n_next (+ pdf-level row of the frame finished two frames ago)
        if (IZ) iz_row(n, par);  // gradient row of frame n (its e in gbuf, partials in wz[par])
        else if (pdf_post && pend_n != n) pdf_row(a, a_gbuf, a_ssp, a_pq, gi, b, pend_n, tid, T, psgn);
        if (MODE == MODE_FACTORED) phase_a_fact(mysl, nsl0, nsl, lane, a_u, a_p, a_part - 4, G.ctr);
        else phase_a<MODE, V>(mysl, nsl, lane, a_u, a_p, a_part, G.ctr);
        __syncthreads();
        // ---- phase B of frame n_next
        const int pp = par;
        par ^= 1;
        if (want_post && !IZ) posterior(n, pp, true);  // γ_n (its x is in registers, Z in cz[pp])
        pend_n = n;
        n = n_next;
        V c = c_iz;
        if (!IZ) {
            c = RAW ? (V)0 : lds_v(a_cz + (uint32_t)(2 * pp) * 8, (V)0);  // lagged normaliser: max of the previous u
            if (c == NINF) c = (V)0;                                       // no viable state: keep 0̄ everywhere
            scale += (double)c;
        }
        if (tid == 0 && a.scale) a.scale[(size_t)b * a.N_max + n] = scale * kLN2;
        V h[SPT];
        float vv[SPT];
        fetch_v(tstep, vb, vv);
        // graphs without masked states: every real state is viable and an inert slot's part
        // row is 0̄ (never written), so the test is skipped (a non-finite emission read by an
        // inert slot only reaches outputs of a sequence that vsum flags anyway)
        auto states = [&](auto masked) {
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                const V y = lds_v(a_part + (uint32_t)(tid + k * T) * VS, (V)0);
                const bool ok = decltype(masked)::value ? viable(k, n) : true;
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
        };
        if (use_mask) states(std::true_type());
        else states(std::false_type());
        emit(n, h, ab);
        if (IZ && tid == 0) asm volatile("cp.async.wait_all;" ::: "memory");  // next step's C (issued a frame ago)
        load_v(n + 2 * dir, vb);  // refill with the frame two steps ahead
        if (want_post) load_alpha(n + 2 * dir, ab);
        return true;
    };
    for (;;) {
        if (!step(vB, aB)) break;
        if (!step(vA, aA)) break;
    }
    // ---- flush the pending posterior rows
    if (IZ) {
        __syncthreads();  // gbuf and wz[par] of the last frame visible
        iz_row(n, par);
    } else if (want_post) {
        __syncthreads();  // wz[par] of the last frame visible; gbuf of pend_n complete
        if (pdf_post && pend_n != n) pdf_row(a, a_gbuf, a_ssp, a_pq, gi, b, pend_n, tid, T, psgn);
        if (pdf_post) __syncthreads();  // gbuf free again
        posterior(n, par, false);
        if (pdf_post) {
            __syncthreads();
            pdf_row(a, a_gbuf, a_ssp, a_pq, gi, b, n, tid, T, psgn);
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
                if (lds_i(a_flag) == 1) stt |= FB_SEQ_NONFINITE_INPUT;  // precedence (fb.h): non-finite,
                else if (!(z > -INFINITY)) stt |= FB_SEQ_EMPTY_LATTICE;  // else empty
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
// Work item of CTA c in round r when items are dealt serpentine over g CTAs.
__device__ __forceinline__ int serpentine(int r, int c, int g) { return r * g + ((r & 1) ? g - 1 - c : c); }

template <bool BWD, int MODEX, int SPT, int MAXT>
__global__ void __launch_bounds__(MAXT, (MAXT >= 512 ? 1 : (MAXT == 256 ? 2 : 7))) k_fb(const FBArgs a) {
    for (int r = 0;; ++r) {
        // per-sequence graphs: members in descending arc count, dealt serpentine
        // (round r runs forward or backward over the CTAs) so per-CTA loads balance
        const int i = serpentine(r, (int)blockIdx.x, (int)gridDim.x);
        if (i >= a.B) break;
        const int b = a.g.G == a.B ? a.g.morder[i] : i;
        fb_sequence<BWD, MODEX, SPT, MAXT>(a, b);
        __syncthreads();  // shared memory is reused by the next sequence
    }
}

// LF-MMI numerator pass: each (persistent) CTA runs the raw forward AND the raw
// backward of its sequences back to back, so the pass stays on the SMs it was
// launched on (a separate backward launch could land on SMs the denominator
// forward has just released and delay the denominator backward).
template <int SPT, int MAXT>
__global__ void __launch_bounds__(MAXT, (MAXT >= 512 ? 1 : (MAXT == 256 ? 2 : 7)))
    k_fb_num(const FBArgs af, const FBArgs ab) {
    for (int r = 0;; ++r) {
        const int i = serpentine(r, (int)blockIdx.x, (int)gridDim.x);
        if (i >= af.B) break;
        const int b = af.g.morder[i];  // heaviest numerator graphs first (G == B), dealt serpentine
        fb_sequence<false, MODE_RAW, SPT, MAXT>(af, b);
        __syncthreads();  // α, logZ and status of sequence b written (block scope suffices)
        fb_sequence<true, MODE_RAW, SPT, MAXT>(ab, b);
        __syncthreads();
    }
}

using KFn = void (*)(FBArgs);
// k_fb<BWD, MODE, spt, MAXT> for a graph's states-per-thread and CTA size;
// instantiated per (BWD, MODE) in its own translation unit (fb_inst.cu).
template <bool BWD, int MODE>
KFn pick_fb(int spt, int T);
#define FBX_PICK_EXTERN(B, M) extern template KFn pick_fb<B, M>(int, int);
FBX_PICK_EXTERN(false, 0) FBX_PICK_EXTERN(false, 1) FBX_PICK_EXTERN(false, 2) FBX_PICK_EXTERN(false, 4)
FBX_PICK_EXTERN(true, 0) FBX_PICK_EXTERN(true, 1) FBX_PICK_EXTERN(true, 2) FBX_PICK_EXTERN(true, 4)
FBX_PICK_EXTERN(true, 5)
#undef FBX_PICK_EXTERN

}  // namespace fbx
