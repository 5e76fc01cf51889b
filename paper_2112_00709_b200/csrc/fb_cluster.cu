// fb_cluster.cu — cluster-batched forward / backward recursion k_fbc for a
// shared (G == 1) factored graph (the LF-MMI denominator).
//
// One thread-block cluster of C CTAs runs S sequences in lockstep, frame by
// frame (batched as P:193-227).  The graph's states are split into C
// parts along pdf ranges (CPlan, fb_internal.h); CTA c owns part c and, per
// frame, computes its rows for all S sequences:
//
//   wait      mbarrier: the other parts' rows u_{t−1} (log2, normalised) and
//             their per-sequence extras (max, posterior normaliser partials)
//             have landed in this CTA's shared memory (bulk DSMEM copies)
//   convert   p = 2^u for the received rows (one ex2 per element)
//   barrier
//   posterior γ_{t−1} = 2^{x − Z} (backward; Z = LSE over all parts, Eq. (15))
//   phase A   the part's sliced-ELL rows: Σ_src p[src][0..S) · e^{T} — one
//             S-wide vector gather and S FMAs per arc (the arc record is read
//             once for S sequences)
//   barrier
//   pdf rows  Γ / −Γ_den of frame t−1 for the part's pdf range (part-local)
//   phase B   y = log2 Σ (exact max-then-sum fallback outside [2^-80, 2^120]),
//             emission, lagged per-sequence normaliser c_t = max u_{t−1}
//             (SURVEY §8(c4)), α̂/β̂ to HBM, new u and p of the part's rows
//   barrier
//   send      the part's u rows + extras to the C−1 other CTAs
//             (cp.async.bulk shared::cta → shared::cluster, complete_tx on the
//             receiver's mbarrier; double-buffered u, so no cluster barrier)
//
// Emission segments (the part's pdf range of each φ row) are staged with
// cp.async one frame ahead.  Per-sequence results are independent of the other
// sequences of the cluster (no cross-sequence arithmetic).
#include "fb_device.cuh"

#if !defined(FBX_BWD) || !defined(FBX_S)
#error "compile with -DFBX_BWD=<0|1> -DFBX_S=<2|4>"
#endif

namespace fbx {

__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_map(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ float cl_ldf(uint32_t a) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void bulk_s2s(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "r"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cl(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P1;\n"
        "WAITC_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAITC_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
// Wait for an mbarrier phase with a suspend-time hint: the warp sleeps in
// hardware until the phase completes instead of re-issuing the probe.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P1;\n"
        "WAITS_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        " @!P1 bra WAITS_%=;\n}\n" ::"r"(a),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void cpa16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa4(uint32_t dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// S-float vectors in shared memory
template <int S>
struct VS;
template <>
struct VS<2> {
    static __device__ __forceinline__ void ld(uint32_t a, float *v) {
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v[0]), "=f"(v[1]) : "r"(a));
    }
    static __device__ __forceinline__ void st(uint32_t a, const float *v) {
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v[0]), "f"(v[1]));
    }
};
template <>
struct VS<4> {
    static __device__ __forceinline__ void ld(uint32_t a, float *v) {
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(a));
    }
    static __device__ __forceinline__ void st(uint32_t a, const float *v) {
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]));
    }
};

// S-float vectors in global memory (the private α̂ lattice, 8/16-byte aligned)
template <int S>
struct VG;
template <>
struct VG<2> {
    static __device__ __forceinline__ void ldg(const float *p, float *v) {
        const float2 x = __ldg(reinterpret_cast<const float2 *>(p));
        v[0] = x.x; v[1] = x.y;
    }
    static __device__ __forceinline__ void stg(float *p, const float *v) { *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]); }
};
template <>
struct VG<4> {
    static __device__ __forceinline__ void ldg(const float *p, float *v) {
        const float4 x = __ldg(reinterpret_cast<const float4 *>(p));
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    }
    static __device__ __forceinline__ void stg(float *p, const float *v) {
        *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};

// Phase A over this warp's slices (Sched layout, fb_internal.h) with S-float
// gathered elements: lane l reduces one row segment for all S sequences.
// add: accumulate into the part row instead of storing (split schedules).
// NOP: the gathered array is u itself (log2) and each element is exponentiated
// on the fly (one MUFU ex2 per sequence-arc) — used when p = 2^u does not fit.
template <int S, bool NOP>
__device__ __forceinline__ void phase_a_vec(uint32_t cur, int nsl, int lane, uint32_t a_p, uint32_t a_part,
                                            bool add) {
    for (int q = 0; q < nsl; ++q) {
        const uint32_t h = lds_u32(cur + lane * 4);
        const int row = (int)(h & 0xFFFFu) - 1, lg = (int)((h >> 16) & 7u), L2 = (int)(h >> 19);
        uint32_t ia = cur + 128 + lane * 4;
        uint32_t wa = cur + 128 + (uint32_t)L2 * 128 + lane * 8;
        // sequence pairs accumulate with packed FFMA2 (sm_100 f32x2): one per arc and pair
        float2 a0[S / 2], a1[S / 2];
#pragma unroll
        for (int i = 0; i < S / 2; ++i) { a0[i] = make_float2(0.f, 0.f); a1[i] = make_float2(0.f, 0.f); }
#pragma unroll 4
        for (int s = 0; s < L2; ++s) {
            const uint32_t ix = lds_u32(ia);
            const float2 w2 = lds_f2(wa);
            float p0[S], p1[S];
            VS<S>::ld(a_p + (ix & 0xFFFFu), p0);
            VS<S>::ld(a_p + (ix >> 16), p1);
            if (NOP) {
#pragma unroll
                for (int i = 0; i < S; ++i) { p0[i] = ex2(p0[i]); p1[i] = ex2(p1[i]); }
            }
#pragma unroll
            for (int i = 0; i < S / 2; ++i) {
                a0[i] = __ffma2_rn(make_float2(p0[2 * i], p0[2 * i + 1]), make_float2(w2.x, w2.x), a0[i]);
                a1[i] = __ffma2_rn(make_float2(p1[2 * i], p1[2 * i + 1]), make_float2(w2.y, w2.y), a1[i]);
            }
            ia += 128;
            wa += 256;
        }
        float acc[S];
#pragma unroll
        for (int i = 0; i < S / 2; ++i) { acc[2 * i] = a0[i].x + a1[i].x; acc[2 * i + 1] = a0[i].y + a1[i].y; }
        for (int o = 1; o < (1 << lg); o <<= 1) {
#pragma unroll
            for (int i = 0; i < S; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
        }
        if (row >= 0) {
            const uint32_t pa = a_part + (uint32_t)row * (S * 4);
            if (add) {  // split schedules: the row's other pass wrote (or phase B zeroed) it
                float o[S];
                VS<S>::ld(pa, o);
#pragma unroll
                for (int i = 0; i < S; ++i) acc[i] += o[i];
            }
            VS<S>::st(pa, acc);
        }
        cur += 128 + (uint32_t)L2 * 384;
    }
}

// Exact max-then-sum of one row for sequence s over the previous frame's u
// (fallback of the factored sum; accurate libm ops; rare).
// PV: the buffer holds p = 2^u (no-p plans): u = log2 p, and p = 0 (u below the fp32
// range, 2^-126 under the frame's lagged maximum, or 0̄) reads as 0̄.
template <int S, bool PV>
static __device__ __noinline__ float exact_row_c(const int *ptr, const int *src, const float *w2, int row, int s,
                                                 uint32_t a_uprev, unsigned long long *ctr) {
    atomicAdd(ctr, 1ull);  // diagnostic: sequence-rows that needed the fallback (fb_graph_counters)
    float m = NEG_INF, sum = 0.f;
    for (int e = ptr[row]; e < ptr[row + 1]; ++e) {
        float uv = lds_v(a_uprev + (uint32_t)(src[e] * S + s) * 4, 0.f);
        if (PV) uv = uv > 0.f ? log2f(uv) : NEG_INF;
        const float x = uv + w2[e];
        if (x == NEG_INF) continue;
        if (x > m) { sum = sum * exp2f(m - x) + 1.f; m = x; }
        else sum += exp2f(x - m);
    }
    return m == NEG_INF ? NEG_INF : m + log2f(sum);
}

// Warp sums of S values per lane (S = 2^m) by reduce-scatter: at offsets 16, 8, …
// each lane keeps half of its values and adds its partner's copy of them, then a plain
// butterfly finishes; lane l ends with the sum of the sequence `seq` it returns
// (determined by its bits 4 … 5−m); lanes with those bits only (l % (32 >> m) == 0)
// hold distinct sequences.  log2(S) + 5 − log2(S) = 5 shuffles for all S sums.
template <int S>
__device__ __forceinline__ float warp_sum_scatter(const float (&v)[S], int lane, int &seq) {
    float cur[S];
#pragma unroll
    for (int i = 0; i < S; ++i) cur[i] = v[i];
    int base = 0, off = 16;
#pragma unroll
    for (int nn = S; nn > 1; nn >>= 1, off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < nn / 2; ++i) {
            const float keep = up ? cur[i + nn / 2] : cur[i];
            const float send = up ? cur[i] : cur[i + nn / 2];
            cur[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
        base += up ? nn / 2 : 0;
    }
    float r = cur[0];
    for (; off; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
    seq = base;
    return r;
}

// Combine (m, s) log-sum-exp pairs (m in log2, s ≥ 0) in a fixed order.
__device__ __forceinline__ void lse2(float &m, float &s, float m2, float s2) { lse_combine<float>(m, s, m2, s2); }

// IZ (backward, −Γ_den gradient of lfmmi_loss_grad): γ normalised through the forward's
// log Z as in the one-CTA kernel (kModeGradIZ, fb_device.cuh): phase B writes
// e = 2^{α̂ + β̂ − Ẑ_n} with Ẑ_n = log2 Z − C_n − D_n straight into xbuf, the parts exchange
// their Σe in the extras slot instead of a (max, sum) pair, and the next frame writes the
// pdf rows −Σ e / S before its phase A — no posterior pass and, for no-p plans, no extra
// barrier between the pdf rows and phase B's xbuf writes.
template <bool BWD, int S, int SPT, int T, bool NOP, bool IZ>
__global__ void __launch_bounds__(T, 1) k_fbc(const FBArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int W = T / 32;
    constexpr float kTiny = 8.271806125530277e-25f, kHuge = 1.329227995784916e+36f;  // 2^-80, 2^120
    const Graph &G = a.g;
    const CPlan &P = G.cp;
    const bool SPLIT = (P.split >> (BWD ? 1 : 0)) & 1;  // this direction's phase A is split around the wait
    const int C = P.C;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cr = (int)cl_rank();
    const int grp = (int)cl_id();
    const int K = G.K_tot, Kint = P.K_int, D = a.D, N_max = a.N_max;
    const int k0 = P.part_off[cr], Kc = P.part_off[cr + 1] - k0;
    const Sched &SC = BWD ? P.bwd : P.fwd;
    const bool want_post = BWD && a.post_kind != POST_NONE;
    const bool pdf_post = want_post && a.post_kind != POST_STATE;
    const CLayout L = cl_layout(SC.bytes_max, Kint, P.Kc_max, P.Dc_max, S, C, W, BWD, NOP);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t a_rec = sb + (uint32_t)L.rec, a_u0 = sb + (uint32_t)L.u, a_p = sb + (uint32_t)L.p;
    const uint32_t a_part = sb + (uint32_t)L.part, a_gbuf = sb + (uint32_t)L.gbuf, a_pq = sb + (uint32_t)L.pq;
    const uint32_t a_ebuf = sb + (uint32_t)L.ebuf, a_red = sb + (uint32_t)L.red, a_mbar = sb + (uint32_t)L.mbar;
    const uint32_t a_xbuf = sb + (uint32_t)L.xbuf;
    const uint32_t UB = (uint32_t)fbx_a16(L.ubytes), XOFF = (uint32_t)Kint * S * 4;
    const uint32_t DC4 = (uint32_t)P.Dc_max * 4;                 // one sequence's share of an emission buffer
    const uint32_t EB = (uint32_t)fbx_a16((size_t)S * DC4);      // one emission buffer
    const float L2E = 1.4426950408889634f, LN2 = 0.6931471805599453f;
    // u buffer `buf`: rows [Kint][S], then extras slots [C][S][kCX] (max, zm, zs, −)
    auto a_u = [&](int buf) { return a_u0 + (uint32_t)(buf & 1) * UB; };
    auto a_x = [&](int buf, int part, int s) { return a_u(buf) + XOFF + (uint32_t)((part * S + s) * kCX) * 4; };

    // ---- the cluster's sequences
    int bs[S], Ns[S], stt[S];
    int Tmax = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int b = grp * S + s;
        bs[s] = b;
        Ns[s] = 0;
        stt[s] = 0;
        if (b < a.B) {
            const int N = a.lengths[b];
            int st = 0;
            if (BWD) {
                st = a.status[b];
                if (a.status2) st |= a.status2[b];
            }
            if (N < 1 || N > N_max) st |= FB_SEQ_BAD_LENGTH;
            const bool skip = (st & FB_SEQ_BAD_LENGTH) || (BWD && st != 0);
            stt[s] = st;
            Ns[s] = skip ? 0 : N;
            Tmax = max(Tmax, Ns[s]);
        }
    }
    // all S sequences of the cluster have one length: the backward reads one frame for all of
    // them, so the private α̂ lattice is reloaded one vector per state
    bool eqlen = true;
#pragma unroll
    for (int s = 1; s < S; ++s) eqlen = eqlen && Ns[s] == Ns[0];
    // part's pdf range and its emission segment [e_lo, e_lo + e_len)
    const int d_lo = P.pdf_lo[cr], d_hi = P.pdf_lo[cr + 1];
    // the segment is staged interleaved, [pdf][S]: phase B reads a state's emission for all S
    // sequences with one vector load (4-byte cp.async per element)
    const int e_lo = d_lo;
    const int e_len = d_hi - d_lo;

    // ---- padded / skipped frames: −∞ lattice rows, zero posterior rows (own states / own pdf range)
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int b = bs[s];
        if (b >= a.B) continue;
        const bool lattice = !(stt[s] & FB_SEQ_BAD_LENGTH);
        for (int n = Ns[s]; n < N_max; ++n) {
            const size_t rowb = ((size_t)b * N_max + n);
            for (int j = tid; j < Kc; j += T) {
                const int o = P.perm[k0 + j];
                if (o < 0) continue;
                if (lattice && a.lat && !a.lat_int) a.lat[rowb * K + o] = NEG_INF;
                if (want_post && a.post_kind == POST_STATE) a.post[rowb * K + o] = 0.f;
            }
            if (pdf_post)
                for (int d = d_lo + tid; d < d_hi; d += T) a.post[rowb * D + d] = 0.f;
            if (lattice && a.scale && cr == 0 && tid == 0) a.scale[rowb] = 0.0;
        }
    }
    if (Tmax == 0) {  // nothing to run in this cluster (identical decision in every CTA)
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (cr == 0 && tid == s && bs[s] < a.B) {
                if (a.logZ) a.logZ[bs[s]] = -INFINITY;
                a.status[bs[s]] = stt[s];
            }
        return;
    }
    auto frame = [&](int s, int t) { return BWD ? Ns[s] - 1 - t : t; };

    // ---- schedule and pdf map → shared memory; mbarriers
    {
        const int m0 = SPLIT ? 2 * cr : cr;  // split: members 2c, 2c+1 back to back
        for (int m = m0; m <= (SPLIT ? m0 + 1 : m0); ++m) {
            const uint4 *src = (const uint4 *)(SC.rec + SC.rec_off[m]);
            uint4 *dst = (uint4 *)(smem_raw + L.rec + (m > m0 ? SC.rec_bytes[m0] : 0));
            const int n16 = SC.rec_bytes[m] >> 4;
            for (int x = tid; x < n16; x += T) dst[x] = src[x];
        }
        // part rows start at 0 whatever the plan: rows without arcs (states with no in-arcs
        // in the forward / no out-arcs in the backward) are never written by phase A and
        // must read as an empty sum (→ exact fallback → 0̄); split plans accumulate both
        // passes into the rows and phase B re-zeroes them
        for (int x = tid; x < P.Kc_max * S; x += T) sts_v(a_part + 4u * (uint32_t)x, 0.f);
    }
    if (pdf_post)
        for (int d = d_lo + tid; d < d_hi; d += T) sts_i(a_pq + 4u * (uint32_t)(d - d_lo), (int)P.pq[d]);
    if (tid == 0) {
        mbar_init(a_mbar, 1);
        mbar_init(a_mbar + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // bytes one frame brings from the other parts
    const uint32_t rx_bytes = (uint32_t)(Kint - Kc) * S * 4 + (uint32_t)(C - 1) * S * kCX * 4;

    // ---- emission segments of step t → ebuf[t & 1] (cp.async, one commit group per step)
    auto emis_issue = [&](int t) {
        if (t < Tmax) {
            const uint32_t base = a_ebuf + (uint32_t)(t & 1) * EB;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (t >= Ns[s] || tid >= e_len) continue;  // only the copying threads
                const float *src = a.emis + ((size_t)bs[s] * N_max + frame(s, t)) * D + e_lo;
                const uint32_t dst = base + (uint32_t)s * 4u;
                for (int x = tid; x < e_len; x += T) cpa4(dst + (uint32_t)(x * S) * 4u, src + x);
            }
        }
        cpa_commit();
    };
    // both emission buffers start at 0: a sequence past its end (or a padding sequence) then
    // reads finite values it has read before (or 0), so vsum needs no per-element guard
    for (int x = tid; 4 * x < 2 * (int)EB; x += T) sts_v(a_ebuf + 4u * (uint32_t)x, 0.f);
    __syncthreads();
    emis_issue(0);
    emis_issue(1);

    // ---- owned states j = tid + k·T (< Kc); padding / out-of-part slots read a
    // real emission of the part and are never viable (distance INT_MAX)
    int pdfk[SPT], distk[SPT], origk[SPT];
    const int pdf_first = P.ipdf[k0] - e_lo;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const int j = tid + k * T;
        pdfk[k] = pdf_first * S * 4;  // byte offset of the pdf's S-vector in the staged segment
        distk[k] = INT_MAX;
        origk[k] = -1;
        if (j < Kc) {
            const int i = k0 + j;
            origk[k] = P.perm[i];
            if (origk[k] >= 0) {
                pdfk[k] = (P.ipdf[i] - e_lo) * S * 4;
                distk[k] = BWD ? P.idist_start[i] : P.idist_fin[i];
                if (!(BWD ? G.mask_bwd : G.mask_fwd)) distk[k] = 0;
            }
        }
    }
    float ar[SPT][S];  // α̂ of the frame being produced (backward posteriors), log2 units
    auto load_alpha = [&](int t) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const bool act = t < Ns[s];
            if (a.lat_int) {  // private layout [cluster][n][K_int][S], log2 units (store_lat)
                if (eqlen) {   // every sequence of the cluster reads the same frame: one vector per state
                    if (s == 0) {
                        const size_t row = ((size_t)grp * N_max + (size_t)(act ? frame(0, t) : 0)) * Kint + k0 + tid;
#pragma unroll
                        for (int k = 0; k < SPT; ++k) {
                            float v[S];
                            if (act && origk[k] >= 0) {
                                VG<S>::ldg(a.alpha + (row + (size_t)k * T) * S, v);
                            } else {
#pragma unroll
                                for (int q = 0; q < S; ++q) v[q] = NEG_INF;
                            }
#pragma unroll
                            for (int q = 0; q < S; ++q) ar[k][q] = v[q];
                        }
                    }
                    continue;
                }
                const float *ro = a.alpha + (act ? ((size_t)grp * N_max + frame(s, t)) * Kint * S : 0) + (size_t)(k0 + tid) * S + s;
#pragma unroll
                for (int k = 0; k < SPT; ++k) ar[k][s] = (act && origk[k] >= 0) ? __ldg(ro + (size_t)k * T * S) : NEG_INF;
                continue;
            }
            const float *ro = a.alpha + (act ? ((size_t)bs[s] * N_max + frame(s, t)) * K : 0);
#pragma unroll
            for (int k = 0; k < SPT; ++k) ar[k][s] = (act && origk[k] >= 0) ? __ldg(ro + origk[k]) * L2E : NEG_INF;
        }
    };
    // x = α̂·log2e + β̂ of the frame whose posterior is pending: xbuf[j][s] (shared memory)
    double scale[S];   // C_n / D_n (log2) — identical in every CTA of the cluster
    float vsum[S];
    // IZ: log2 Z of each sequence's forward; the forward's C of the frame being produced is
    // staged by lanes s < S of warp 0 (loaded one frame ahead) into cnbuf[s]
    float zhat[S];
    double logZ2[S];
    double cn_reg = 0.0;
    const uint32_t a_cn = a_red + (uint32_t)((W + 2) * S * kCX) * 4 - 8u * S;  // last S doubles of red
#pragma unroll
    for (int s = 0; s < S; ++s) {
        zhat[s] = 0.f;
        logZ2[s] = (IZ && 0 < Ns[s]) ? a.logZ_fwd[bs[s]] * 1.4426950408889634 : 0.0;
    }
    auto cn_load = [&](int t) {  // lanes s < S of warp 0: the forward's C_n (natural) of step t
        if (IZ && tid < S) {
            int Nss = Ns[0], bss = bs[0];
#pragma unroll
            for (int q = 1; q < S; ++q) { Nss = tid == q ? Ns[q] : Nss; bss = tid == q ? bs[q] : bss; }
            cn_reg = (t < Nss) ? __ldg(a.ascale_in + (size_t)bss * N_max + (Nss - 1 - t)) : 0.0;
        }
    };
#pragma unroll
    for (int s = 0; s < S; ++s) { scale[s] = 0.0; vsum[s] = 0.f; }
    // termination pairs are reduced per warp at each sequence's last frame: red fields 3, 4
    for (int x = tid; x < W * S; x += T) {
        sts_v(a_red + (uint32_t)(x * kCX + 3) * 4, NEG_INF);
        sts_v(a_red + (uint32_t)(x * kCX + 4) * 4, 0.f);
    }

    // Store frame t's values h (α̂/β̂, log2) and u of the owned rows; per-warp
    // reductions (max u, posterior pair) into red[warp][s]; termination pair.
    auto emit = [&](int t, float (&h)[SPT][S], float (&u)[SPT][S]) {
        const uint32_t ub = a_u(t);
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const int j = tid + k * T;
            if (j < Kc) {
                float pv[S];
#pragma unroll
                for (int s = 0; s < S; ++s) pv[s] = ex2(u[k][s]);
                // no-p plans exchange and gather p = 2^u itself (one ex2 per owned element
                // instead of one per gathered arc); with-p plans keep u and convert on receipt
                VS<S>::st(ub + (uint32_t)((k0 + j) * S) * 4, NOP ? pv : u[k]);
                if (!NOP) VS<S>::st(a_p + (uint32_t)((k0 + j) * S) * 4, pv);
            }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (t >= Ns[s]) continue;  // CTA-uniform
            float mx = u[0][s];
#pragma unroll
            for (int k = 1; k < SPT; ++k) mx = fmaxf(mx, u[k][s]);
            mx = warp_max_fast(mx);
            if (lane == 0) sts_v(a_red + (uint32_t)((warp * S + s) * kCX) * 4, mx);
            if (IZ) {
                // below, for all sequences at once
            } else if (want_post) {
                float x[SPT];
#pragma unroll
                for (int k = 0; k < SPT; ++k) {
                    x[k] = ar[k][s] + h[k][s];
                    if (tid + k * T < Kc) sts_v(a_xbuf + (uint32_t)((tid + k * T) * S + s) * 4, x[k]);
                }
                float zm, zs;
                warp_lse_vals<float, SPT>(x, zm, zs);
                if (lane == 0) {
                    sts_v(a_red + (uint32_t)((warp * S + s) * kCX + 1) * 4, zm);
                    sts_v(a_red + (uint32_t)((warp * S + s) * kCX + 2) * 4, zs);
                }
            }
            if (t == Ns[s] - 1) {  // termination pair (fwd: u ⊗ ω; bwd: π ⊗ u) — once per sequence
                float tm = NEG_INF, ts = 0.f;
#pragma unroll
                for (int k = 0; k < SPT; ++k) {
                    const int j = tid + k * T;
                    if (j < Kc && origk[k] >= 0) {
                        const float w = BWD ? P.iinit2[k0 + j] : P.ifinal2[k0 + j];
                        lse_push<float>(tm, ts, u[k][s] + w);
                    }
                }
                warp_lse(tm, ts);
                if (lane == 0) {
                    sts_v(a_red + (uint32_t)((warp * S + s) * kCX + 3) * 4, tm);
                    sts_v(a_red + (uint32_t)((warp * S + s) * kCX + 4) * 4, ts);
                }
            }
        }
        if (IZ) {  // e = 2^{x − Ẑ} into xbuf (one vector store per state), per-warp Σ e into red field 1
            float es[S];
#pragma unroll
            for (int s = 0; s < S; ++s) es[s] = 0.f;
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                float e[S];
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    e[s] = ex2(ar[k][s] + h[k][s] - zhat[s]);  // 0 for non-viable / padding / inactive
                    es[s] += e[s];
                }
                if (tid + k * T < Kc) VS<S>::st(a_xbuf + (uint32_t)((tid + k * T) * S) * 4, e);
            }
            int sq = 0;
            const float r = warp_sum_scatter<S>(es, lane, sq);
            if ((lane & ((32 / S) - 1)) == 0) sts_v(a_red + (uint32_t)((warp * S + sq) * kCX + 1) * 4, r);
        }
    };
    // α̂/β̂ rows of frame t to HBM — issued after the frame has been shipped, so the
    // proxy fence before the bulk copies does not wait for these stores
    auto store_lat = [&](int t, float (&h)[SPT][S]) {
        if (!a.lat) return;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (t >= Ns[s]) continue;
            if (a.lat_int) {  // private lfmmi workspace [cluster][n][K_int][S], log2 units: one vector per state
                // (frame t = step t for every sequence of the forward; a sequence past its end writes
                // values no one reads)
                if (s == 0) {
                    float *latn = a.lat + (((size_t)grp * N_max + t) * Kint + k0 + tid) * S;
#pragma unroll
                    for (int k = 0; k < SPT; ++k)
                        if (tid + k * T < Kc) VG<S>::stg(latn + (size_t)k * T * S, h[k]);
                }
                continue;
            }
            float *latn = a.lat + ((size_t)bs[s] * N_max + frame(s, t)) * K;
#pragma unroll
            for (int k = 0; k < SPT; ++k)
                if (origk[k] >= 0) latn[origk[k]] = h[k][s] * LN2;
        }
    };
    // warp 0: per-warp reductions → this part's extras slot of buffer t; lane 0 ships the frame
    auto send = [&](int t) {
        if (warp != 0) return;
        if constexpr (S == 2) {
            // lane w < W holds warp w's partials: one warp-wide max (REDUX) and one shuffle
            // sum per sequence (max-first log-sum-exp instead of a serial chain over W warps;
            // the register-saturated S = 4 kernels keep the one-lane-per-sequence loop)
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const uint32_t r = a_red + (uint32_t)((lane * S + s) * kCX) * 4;
                const float mx = warp_max_fast(lane < W ? lds_v(r, 0.f) : NEG_INF);
                float zm = NEG_INF, zs = 0.f;
                if (IZ) {
                    zm = warp_sum(lane < W ? lds_v(r + 4, 0.f) : 0.f);  // the part's Σ e
                } else if (want_post) {
                    const float pm = lane < W ? lds_v(r + 4, 0.f) : NEG_INF;
                    const float ps = lane < W ? lds_v(r + 8, 0.f) : 0.f;
                    zm = warp_max_fast(pm);
                    zs = warp_sum((pm == NEG_INF) ? 0.f : ps * ex2(pm - zm));
                }
                if (lane == s) {
                    const uint32_t x = a_x(t, cr, s);
                    sts_v(x, mx);
                    sts_v(x + 4, zm);
                    sts_v(x + 8, zs);
                }
            }
        } else {
            // S = 4: lane l folds the (warp, sequence) entries w ≡ l/4 (mod 8), s = l % 4, then
            // three xor shuffles (4, 8, 16) combine the lanes of one sequence
            const int s = lane & 3;
            float mx = NEG_INF, zm = NEG_INF, zs = 0.f;
            for (int w = lane >> 2; w < W; w += 8) {
                const uint32_t r = a_red + (uint32_t)((w * S + s) * kCX) * 4;
                mx = fmaxf(mx, lds_v(r, 0.f));
                if (IZ) zs += lds_v(r + 4, 0.f);
                else if (want_post) lse2(zm, zs, lds_v(r + 4, 0.f), lds_v(r + 8, 0.f));
            }
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                if (IZ) {
                    zs += __shfl_xor_sync(0xffffffffu, zs, o);
                } else if (want_post) {
                    const float m2 = __shfl_xor_sync(0xffffffffu, zm, o), s2 = __shfl_xor_sync(0xffffffffu, zs, o);
                    lse2(zm, zs, m2, s2);
                }
            }
            if (lane < S) {
                const uint32_t x = a_x(t, cr, s);
                sts_v(x, mx);
                sts_v(x + 4, IZ ? zs : zm);
                sts_v(x + 8, zs);
            }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
            if (t + 1 < Tmax) mbar_arrive_tx(a_mbar + 8u * (uint32_t)((t + 1) & 1), rx_bytes);
            const uint32_t rows = a_u(t) + (uint32_t)(k0 * S) * 4, xs = a_x(t, cr, 0);
            const uint32_t mb = a_mbar + 8u * (uint32_t)(t & 1);
            for (int q = 0; q < C; ++q) {
                if (q == cr) continue;
                bulk_s2s(cl_map(rows, q), rows, (uint32_t)Kc * S * 4, cl_map(mb, q));
                bulk_s2s(cl_map(xs, q), xs, (uint32_t)S * kCX * 4, cl_map(mb, q));
            }
        }
    };

    // ---- frame 0: π ⊗ v_0 (fwd, L6) / β̂_{N−1} = ω (bwd, L7), exact cluster-wide max
    if (want_post) load_alpha(0);
    cpa_wait1();
    __syncthreads();  // schedule, pq, mbarrier init, step-0 emissions
    cl_sync();        // every CTA's mbarriers initialised
    if (tid == 0) mbar_arrive_tx(a_mbar, rx_bytes);
    float h[SPT][S], u[SPT][S];
    {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const bool act = 0 < Ns[s];
            const int lim = act ? (BWD ? frame(s, 0) : Ns[s] - 1) : -1;
            float mx = NEG_INF;
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                const int j = tid + k * T;
                const bool ok = distk[k] <= lim;
                const float v = lds_v(a_ebuf + (uint32_t)pdfk[k] + 4u * (uint32_t)s, 0.f);
                if (act) vsum[s] += v;
                const float v2 = v * L2E;
                const int jj = min(j, Kc - 1);
                if (!BWD) {
                    h[k][s] = ok ? P.iinit2[k0 + jj] + v2 : NEG_INF;
                    u[k][s] = h[k][s];
                } else {
                    h[k][s] = ok ? P.ifinal2[k0 + jj] : NEG_INF;
                    u[k][s] = ok ? h[k][s] + v2 : NEG_INF;
                }
                mx = fmaxf(mx, u[k][s]);
            }
            mx = warp_max_fast(mx);
            if (lane == 0) sts_v(a_red + (uint32_t)((warp * S + s) * kCX) * 4, mx);
        }
        __syncthreads();
        const uint32_t init_slot = a_red + (uint32_t)(W * S * kCX) * 4;
        if (warp == 0 && lane < S) {
            float mx = NEG_INF;
            for (int w = 0; w < W; ++w) mx = fmaxf(mx, lds_v(a_red + (uint32_t)((w * S + lane) * kCX) * 4, 0.f));
            sts_v(init_slot + 4u * (uint32_t)lane, mx);
        }
        cl_sync();  // every part's frame-0 maximum visible cluster-wide
#pragma unroll
        for (int s = 0; s < S; ++s) {
            float c = NEG_INF;
            for (int q = 0; q < C; ++q) c = fmaxf(c, cl_ldf(cl_map(init_slot + 4u * (uint32_t)s, q)));
            if (c == NEG_INF) c = 0.f;
            if (0 < Ns[s]) scale[s] = (double)c;
#pragma unroll
            for (int k = 0; k < SPT; ++k) { h[k][s] -= c; u[k][s] -= c; }
            if (cr == 0 && tid == 0 && a.scale && 0 < Ns[s])
                a.scale[(size_t)bs[s] * N_max + frame(s, 0)] = scale[s] * kLN2;
            if (IZ && 0 < Ns[s])
                zhat[s] = (float)(logZ2[s] - __ldg(a.ascale_in + (size_t)bs[s] * N_max + frame(s, 0)) * 1.4426950408889634 -
                                  scale[s]);
        }
        emit(0, h, u);
        fence_async_smem();
        __syncthreads();
        send(0);
        store_lat(0, h);
    }

    // ---- frames 1 … Tmax−1 (+ one flush step t = Tmax for the last posterior rows)
    const int split = SPLIT;
    const int mr = split ? 2 * cr + 1 : cr;  // remote-source (or whole) member
    const int nsl = SC.warp_nsl[mr * W + warp];
    const uint32_t mysl = a_rec + (uint32_t)(split ? SC.rec_bytes[2 * cr] : 0) + (uint32_t)SC.warp_off[mr * W + warp];
    const int nsl_loc = split ? SC.warp_nsl[2 * cr * W + warp] : 0;
    const uint32_t mysl_loc = a_rec + (uint32_t)(split ? SC.warp_off[2 * cr * W + warp] : 0);
    const int own0 = k0 * S, own1 = (k0 + Kc) * S;  // this part's element range of u / p
    cn_load(1);
    // pdf-level rows of frame t−1 for this part's pdf range (ascending states, ledger L9); IZ: the
    // e of xbuf scaled by mul[s] = −1/S_{t−1}, else γ of gbuf with the sign of the output kind
    auto pdf_rows = [&](int t, const float (&mul)[S]) {
        const float sgn = a.post_kind == POST_GRAD ? -1.f : 1.f;
        const uint32_t src = IZ ? a_xbuf : a_gbuf;
        // four lanes per (pdf, sequence) pair (a part owns few pdfs with many states: N2 ~21 pdfs ×
        // ~36 states): lane i of the quad sums states i, i + 4, …, two xor shuffles combine the quad,
        // so the rows cost every warp a few gathers instead of ~36 serial ones on three warps
        constexpr int PL = 4;
        const int nd = d_hi - d_lo, npairs = nd * S;
        for (int base = 0; base < npairs * PL; base += T) {  // CTA-uniform trip count (full-warp shuffles)
            const int idx = base + tid, pr = idx / PL, sub = idx & (PL - 1);
            const bool on = pr < npairs;
            int s = 0, d = d_lo;
            float acc = 0.f;
            if (on) {
                s = pr / nd;
                d = d_lo + pr % nd;
                const uint32_t w = lds_u32(a_pq + 4u * (uint32_t)(d - d_lo));
                const uint32_t q0 = w & 0xFFFFu, c = w >> 16;
                for (uint32_t i = (uint32_t)sub; i < c; i += PL) acc += lds_v(src + ((q0 + i) * S + (uint32_t)s) * 4u, 0.f);
            }
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            if (!on || sub != 0) continue;
            int Nss = Ns[0], bss = bs[0];
            float ms = mul[0];
#pragma unroll
            for (int q = 1; q < S; ++q) {
                Nss = s == q ? Ns[q] : Nss;
                bss = s == q ? bs[q] : bss;
                ms = s == q ? mul[q] : ms;
            }
            if (t - 1 >= Nss) continue;
            a.post[((size_t)bss * N_max + (BWD ? Nss - 1 - (t - 1) : t - 1)) * D + d] = (IZ ? ms : sgn) * acc;
        }
    };
    for (int t = 1; t <= Tmax; ++t) {
        const bool last = t == Tmax;
        if (IZ && tid < S) {  // w_s = log2 Z − C_t − D_{t−1} of sequence s = tid → cnbuf (Ẑ_t = w_s − c_t);
                              // the forward's C of step t was loaded last frame; load step t + 1's
            double sc = scale[0];
#pragma unroll
            for (int q = 1; q < S; ++q) sc = tid == q ? scale[q] : sc;
            double lz = logZ2[0];
#pragma unroll
            for (int q = 1; q < S; ++q) lz = tid == q ? logZ2[q] : lz;
            sts_v(a_cn + 4u * (uint32_t)tid, (float)(lz - cn_reg * 1.4426950408889634 - sc));
            cn_load(t + 1);
        }
        if (!last) {
            if (want_post) load_alpha(t);
            emis_issue(t + 1);
            // split: this part's own-source arcs while the other parts' rows are in flight
            if (split) phase_a_vec<S, false>(mysl_loc, nsl_loc, lane, NOP ? a_u(t - 1) : a_p, a_part, true);
        }
        // no-p plans: warp 0 alone polls the exchange barrier (acquire); the CTA barrier below
        // orders the other warps' reads of the received rows after it (with-p plans convert
        // the received rows before that barrier, so every warp waits)
        if (!NOP || warp == 0) mbar_wait_sleep(a_mbar + 8u * (uint32_t)((t - 1) & 1), (uint32_t)(((t - 1) >> 1) & 1));
        const uint32_t up = a_u(t - 1);
        if (!last && !NOP) {  // p = 2^u of the other parts' rows
            for (int e = 4 * tid; e < Kint * S; e += 4 * T) {
                if (e >= own0 && e < own1) continue;
                float v[4];
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                             : "r"(up + 4u * (uint32_t)e));
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a_p + 4u * (uint32_t)e), "f"(ex2(v[0])),
                             "f"(ex2(v[1])), "f"(ex2(v[2])), "f"(ex2(v[3])));
            }
        }
        __syncthreads();  // p complete; this part's extras slot of frame t−1 visible
        // cluster-wide extras of frame t−1: lane q·S + s holds part q's (max, Z pair) of
        // sequence s; a log2(C)-step xor tree over q (C·S ≤ 32; the combine is commutative,
        // so every lane — and every CTA of the cluster — gets bitwise the same result),
        // then lane s broadcasts sequence s
        float cmax[S], Z[S];
        {
            float mx = NEG_INF, zm = IZ ? 0.f : NEG_INF, zs = 0.f;
            if (lane < C * S) {
                const uint32_t x = a_x(t - 1, lane / S, lane % S);
                mx = lds_v(x, 0.f);
                if (IZ) zm = lds_v(x + 4, 0.f);
                else if (want_post) { zm = lds_v(x + 4, 0.f); zs = lds_v(x + 8, 0.f); }
            }
            for (int o = S; o < C * S; o <<= 1) {
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                if (IZ) {
                    zm += __shfl_xor_sync(0xffffffffu, zm, o);  // Σ e over the parts (commutative tree)
                } else if (want_post) {
                    const float m2 = __shfl_xor_sync(0xffffffffu, zm, o), s2 = __shfl_xor_sync(0xffffffffu, zs, o);
                    lse2(zm, zs, m2, s2);
                }
            }
            // IZ: Z[s] carries the pdf-row multiplier −1/S (0 if S is not a positive finite sum)
            const float zl = IZ ? ((zm > 0.f && zm < INFINITY) ? -__fdividef(1.f, zm) : 0.f)
                                : ((zm == NEG_INF) ? NEG_INF : zm + lg2(zs));
#pragma unroll
            for (int s = 0; s < S; ++s) {
                cmax[s] = __shfl_sync(0xffffffffu, mx, s);
                Z[s] = want_post ? __shfl_sync(0xffffffffu, zl, s) : NEG_INF;
            }
        }
        if (IZ) pdf_rows(t, Z);  // frame t−1's e (xbuf) is complete; phase B refills xbuf after the barrier
        // posteriors of frame t−1 (Eq. (15), normalised by Z_{t−1} = LSE_k(α̂ + β̂))
        if (want_post && !IZ) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (t - 1 >= Ns[s]) continue;
                const float Zs = (Z[s] == NEG_INF) ? 0.f : Z[s];
                if (a.post_kind == POST_STATE) {
                    float *prow = a.post + ((size_t)bs[s] * N_max + frame(s, t - 1)) * K;
#pragma unroll
                    for (int k = 0; k < SPT; ++k)
                        if (origk[k] >= 0)  // implies tid + k·T < Kc
                            prow[origk[k]] = (Z[s] == NEG_INF)
                                                 ? 0.f
                                                 : ex2(lds_v(a_xbuf + (uint32_t)((tid + k * T) * S + s) * 4, 0.f) - Zs);
                } else {
#pragma unroll
                    for (int k = 0; k < SPT; ++k) {
                        const int j = tid + k * T;
                        if (j < Kc)
                            sts_v(a_gbuf + (uint32_t)(j * S + s) * 4,
                                  (Z[s] == NEG_INF || origk[k] < 0)
                                      ? 0.f
                                      : ex2(lds_v(a_xbuf + (uint32_t)(j * S + s) * 4, 0.f) - Zs));
                    }
                }
            }
        }
        if (!last) phase_a_vec<S, false>(mysl, nsl, lane, NOP ? up : a_p, a_part, split);
        cpa_wait1();
        __syncthreads();  // part rows, γ rows, step-t emissions complete
        if (pdf_post && !IZ) {
            pdf_rows(t, Z);
            if (NOP) __syncthreads();  // γ lives in xbuf, which phase B refills with the next x
        }
        if (last) break;
        // ---- phase B of frame t: y = log2 Σ, emission, lagged normaliser, mask
        const uint32_t eb = a_ebuf + (uint32_t)(t & 1) * EB;
        float c[S];
        int lim[S];
        // the float64 offsets are kept by warp 0 (IZ: its lanes s < S stage Ẑ's float64 part;
        // part 0: termination, the scale output) — a CTA-uniform branch
        const bool keep_scale = warp == 0 && (IZ || cr == 0);
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const bool act = t < Ns[s];
            c[s] = (cmax[s] == NEG_INF) ? 0.f : cmax[s];  // no viable state: keep 0̄ everywhere
            lim[s] = act ? (BWD ? frame(s, t) : Ns[s] - 1 - t) : -1;
        }
        if (keep_scale) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (t >= Ns[s]) continue;
                scale[s] += (double)c[s];
                if (cr == 0 && tid == 0 && a.scale) a.scale[(size_t)bs[s] * N_max + frame(s, t)] = scale[s] * kLN2;
            }
        }
        if (IZ) {
#pragma unroll
            for (int s = 0; s < S; ++s) zhat[s] = lds_v(a_cn + 4u * (uint32_t)s, 0.f) - c[s];  // Ẑ_t = w_s − c_t
        }
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const int j = tid + k * T;
            float acc[S] = {};
            if (j < Kc) VS<S>::ld(a_part + (uint32_t)(j * S) * 4, acc);  // inert slots read nothing (racecheck-clean)
            if (split && j < Kc) {
                const float z[S] = {};
                VS<S>::st(a_part + (uint32_t)(j * S) * 4, z);
            }
            float alo = 1.f, ahi = 1.f;  // range of the viable sums (the fallback test, once per state)
            float ev[S];
            VS<S>::ld(eb + (uint32_t)pdfk[k], ev);
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const float v = ev[s];
                vsum[s] += v;  // inactive sequences read stale finite values or 0 (zeroed buffers)
                const bool ok = distk[k] <= lim[s];
                const float am = ok ? acc[s] : 1.f;
                alo = fminf(alo, am);
                ahi = fmaxf(ahi, am);
                const float y = lg2(acc[s]);
                if (!BWD) {
                    h[k][s] = ok ? y + fmaf(v, L2E, -c[s]) : NEG_INF;
                    u[k][s] = h[k][s];
                } else {
                    h[k][s] = ok ? y - c[s] : NEG_INF;
                    u[k][s] = ok ? fmaf(v, L2E, h[k][s]) : NEG_INF;
                }
            }
            if (!(alo >= kTiny && ahi <= kHuge)) {  // exact max-then-sum rows (rare)
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    if (!(distk[k] <= lim[s]) || (acc[s] >= kTiny && acc[s] <= kHuge)) continue;
                    const float y = exact_row_c<S, NOP>(BWD ? P.bptr : P.fptr, BWD ? P.bsrc : P.fsrc, BWD ? P.bw2 : P.fw2,
                                                   k0 + j, s, up, G.ctr + 1);
                    const float v = lds_v(eb + (uint32_t)pdfk[k] + 4u * (uint32_t)s, 0.f);
                    if (!BWD) {
                        h[k][s] = y + fmaf(v, L2E, -c[s]);
                        u[k][s] = h[k][s];
                    } else {
                        h[k][s] = y - c[s];
                        u[k][s] = fmaf(v, L2E, h[k][s]);
                    }
                }
            }
        }
        emit(t, h, u);
        fence_async_smem();
        __syncthreads();  // u / p rows and reductions of frame t complete
        send(t);
        store_lat(t, h);
    }

    // ---- termination: logZ = C + ⊕_k α̂ ⊗ ω (fwd) / logZ_β = D + ⊕_k π ⊗ β̂_0 ⊗ v_0 (bwd);
    // non-finite emissions flag; both combined over the cluster in fixed order
    __syncthreads();
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const float vs = warp_sum(vsum[s]);
        if (lane == 0) sts_v(a_red + (uint32_t)((warp * S + s) * kCX) * 4 + 20, vs);
    }
    __syncthreads();
    const uint32_t fin = a_red + (uint32_t)((W + 1) * S * kCX) * 4;  // after the frame-0 slot
    if (warp == 0 && lane < S) {
        float m = NEG_INF, q = 0.f, vs = 0.f;
        for (int w = 0; w < W; ++w) {
            const uint32_t r = a_red + (uint32_t)((w * S + lane) * kCX) * 4;
            lse2(m, q, lds_v(r + 12, 0.f), lds_v(r + 16, 0.f));
            vs += lds_v(r + 20, 0.f);
        }
        sts_v(fin + 16u * (uint32_t)lane, m);
        sts_v(fin + 16u * (uint32_t)lane + 4, q);
        sts_v(fin + 16u * (uint32_t)lane + 8, vs);
    }
    cl_sync();
#pragma unroll
    for (int s = 0; s < S; ++s) {
        if (!(cr == 0 && tid == 0 && bs[s] < a.B)) continue;
        // float64 combine of the parts' (max, sum) pairs in part order
        double M = -INFINITY, vq = 0.0;
        for (int q = 0; q < C; ++q) {
            const float mq = cl_ldf(cl_map(fin + 16u * (uint32_t)s, q));
            vq += (double)cl_ldf(cl_map(fin + 16u * (uint32_t)s + 8, q));
            if (mq != NEG_INF) M = fmax(M, (double)mq);
        }
        double tot = 0.0;
        for (int q = 0; q < C; ++q) {
            const float mq = cl_ldf(cl_map(fin + 16u * (uint32_t)s, q));
            if (mq != NEG_INF) tot += (double)cl_ldf(cl_map(fin + 16u * (uint32_t)s + 4, q)) * exp2((double)mq - M);
        }
        int st = stt[s];
        double z = -INFINITY;
        if (Ns[s] > 0) {
            z = (M == -INFINITY) ? -INFINITY : (scale[s] + M + log2(tot)) * kLN2;
            if (!(vq < INFINITY)) st |= FB_SEQ_NONFINITE_INPUT;  // precedence as in fb.h: non-finite, else empty
            else if (!(z > -INFINITY)) st |= FB_SEQ_EMPTY_LATTICE;
        }
        if (st) z = -INFINITY;
        if (a.logZ) a.logZ[bs[s]] = z;
        a.status[bs[s]] = st;
    }
    cl_sync();  // peers' shared memory stays alive until every remote read is done
}

using KFn = void (*)(FBArgs);
// T = 1024 threads (SPT ≤ 4, ≤ 64 registers) or 512 (SPT ≤ 8, ≤ 128 registers);
// nop (S = 4 only): no p array
template <bool BWD, int S, bool NOP, bool IZ>
static KFn pick_fbc_t(int spt, int T) {
    if (T == 1024) {
        switch (spt) {
            case 1: return k_fbc<BWD, S, 1, 1024, NOP, IZ>;
            case 2: return k_fbc<BWD, S, 2, 1024, NOP, IZ>;
            case 3: return k_fbc<BWD, S, 3, 1024, NOP, IZ>;
            default: return k_fbc<BWD, S, 4, 1024, NOP, IZ>;
        }
    }
    switch (spt) {
        case 1: return k_fbc<BWD, S, 1, 512, NOP, IZ>;
        case 2: return k_fbc<BWD, S, 2, 512, NOP, IZ>;
        case 3: return k_fbc<BWD, S, 3, 512, NOP, IZ>;
        case 4: return k_fbc<BWD, S, 4, 512, NOP, IZ>;
        case 6: return k_fbc<BWD, S, 6, 512, NOP, IZ>;
        default: return k_fbc<BWD, S, 8, 512, NOP, IZ>;
    }
}
// iz (backward only): the lfmmi −Γ_den epilogue normalised through the forward's log Z
template <bool BWD, int S>
KFn pick_fbc(int spt, int T, int nop, int iz) {
    if constexpr (BWD) {
        if (iz) {
            if constexpr (S == 4) {
                if (nop) return pick_fbc_t<BWD, S, true, true>(spt, T);
            }
            return pick_fbc_t<BWD, S, false, true>(spt, T);
        }
    }
    if constexpr (S == 4) {
        if (nop) return pick_fbc_t<BWD, S, true, false>(spt, T);
    }
    return pick_fbc_t<BWD, S, false, false>(spt, T);
}
template KFn pick_fbc<(bool)FBX_BWD, FBX_S>(int, int, int, int);

}  // namespace fbx
