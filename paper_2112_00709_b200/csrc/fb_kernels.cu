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
#include <map>
#include <memory>

#include "fb_device.cuh"

namespace fbx {

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

// The same over a schedule left in global memory (graphs whose Viterbi schedule
// exceeds shared memory, e.g. the paper's 50,984-arc denominator): records are
// read through the read-only path (L2-resident: every CTA streams the same
// blob each frame), four arc pairs in flight per lane.
__device__ __forceinline__ void phase_a_max_g(const unsigned char *cur, int nsl, int lane, uint32_t a_u,
                                              uint32_t a_best, uint32_t a_arg) {
    for (int q = 0; q < nsl; ++q) {
        const uint32_t h = __ldg((const uint32_t *)cur + lane);
        const int row = (int)(h & 0xFFFFu) - 1, lg = (int)((h >> 16) & 7u), L2 = (int)(h >> 19);
        const uint32_t *ia = (const uint32_t *)(cur + 128) + lane;
        const float2 *wa = (const float2 *)(cur + 128 + (size_t)L2 * 128) + lane;
        double b0 = NEG_INF_D, b1 = NEG_INF_D;
        int g0 = 0x7fffffff, g1 = 0x7fffffff;
#pragma unroll 4
        for (int s = 0; s < L2; ++s) {
            const uint32_t ix = __ldg(ia + 32 * s);
            const float2 w2 = __ldg(wa + 32 * s);
            const uint32_t o0 = ix & 0xFFFFu, o1 = ix >> 16;
            vit_consider(b0, g0, lds_v(a_u + o0, 0.0) + (double)w2.x, (int)(o0 >> 3));
            vit_consider(b1, g1, lds_v(a_u + o1, 0.0) + (double)w2.y, (int)(o1 >> 3));
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
        cur += 128 + (size_t)L2 * 384;
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
// GLOB: the schedule stays in global memory (Graph::vit_global), shared memory
// holds only the float64 vectors.
template <int SPT, int MAXT, bool GLOB>
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
    const SmemLayout SL = smem_layout(GLOB ? 0 : S.bytes_max, T * SPT, true, false);
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
    if (!GLOB) {
        const uint4 *src = (const uint4 *)(S.rec + S.rec_off[gi]);
        uint4 *dst = (uint4 *)(smem_raw + SL.rec);
        const int n16 = S.rec_bytes[gi] >> 4;
        for (int x = tid; x < n16; x += T) dst[x] = src[x];
    }
    const int nsl = S.warp_nsl[gi * W + warp];
    const uint32_t mysl = sb + (uint32_t)SL.rec + (uint32_t)S.warp_off[gi * W + warp];
    const unsigned char *mysl_g = S.rec + S.rec_off[gi] + S.warp_off[gi * W + warp];
    int pdfk[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const int j = tid + k * T;
        pdfk[k] = G.pdf[s0 + (j < K ? j : 0)];  // inert slots read a column the graph reads (status parity)
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
        if (GLOB) phase_a_max_g(mysl_g, nsl, lane, a_u, a_best, a_arg);
        else phase_a_max(mysl, nsl, lane, a_u, a_best, a_arg);
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
            if (bad) st |= FB_SEQ_NONFINITE_INPUT;  // precedence as in fb.h: non-finite, else empty
            else if (best == NEG_INF_D) st |= FB_SEQ_EMPTY_LATTICE;
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

// ------------------------------------------------------------------ Eq. (1) invariant diagnostic

// One CTA per sequence: gap_b = max_{n<N_b} |Z_n + C_n + D_n − logZ_b| with
// Z_n = ⊕_k α̂_n(k) ⊗ β̂_n(k) (block log-sum-exp, natural log, float64 combine).
// By Eq. (1) every frame's α·β sum is the same log Z, so the gap
// measures the accumulated rounding of the normalised fp32 lattices.
__global__ void __launch_bounds__(256) k_gap(const Graph G, const float *alpha, const double *ascale,
                                             const float *beta, const double *bscale, const double *logZ,
                                             const int *lengths, const int *status, int B, int N_max,
                                             double *gap) {
    __shared__ double wz[2 * 8];
    const int b = blockIdx.x;
    const int gi = (G.G == 1) ? 0 : b;
    const int s0 = G.state_off[gi], K = G.state_off[gi + 1] - s0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, W = blockDim.x >> 5;
    const int N = lengths[b];
    if (N < 1 || N > N_max || (status && status[b] != 0) || !(logZ[b] > -INFINITY)) {
        if (tid == 0) gap[b] = 0.0;  // flagged sequences: no invariant to check (the oracle's convention)
        return;
    }
    const size_t base = (size_t)N_max * (G.G == 1 ? (size_t)b * K : (size_t)s0);
    double gmax = 0.0;
    for (int n = 0; n < N; ++n) {
        double m = NEG_INF_D;
        for (int j = tid; j < K; j += blockDim.x)
            m = fmax(m, (double)__ldg(alpha + base + (size_t)n * K + j) + (double)__ldg(beta + base + (size_t)n * K + j));
        m = warp_max(m);
        if (lane == 0) wz[warp] = m;
        __syncthreads();
        m = lane < W ? wz[lane] : NEG_INF_D;
        m = warp_max(m);
        double s = 0.0;
        if (m > NEG_INF_D)
            for (int j = tid; j < K; j += blockDim.x)
                s += exp((double)__ldg(alpha + base + (size_t)n * K + j) +
                         (double)__ldg(beta + base + (size_t)n * K + j) - m);
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        __syncthreads();
        if (lane == 0) wz[8 + warp] = s;
        __syncthreads();
        s = lane < W ? wz[8 + lane] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const double zn = (m > NEG_INF_D) ? m + log(s) + ascale[(size_t)b * N_max + n] + bscale[(size_t)b * N_max + n]
                                          : NEG_INF_D;
        gmax = fmax(gmax, (zn > NEG_INF_D) ? fabs(zn - logZ[b]) : INFINITY);
        __syncthreads();
    }
    if (tid == 0) gap[b] = gmax;
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

static KFn pick(bool bwd, int mode, int spt, int T) {
    if (bwd) {
        if (mode == kModeGradIZ) return pick_fb<true, kModeGradIZ>(spt, T);
        if (mode == kModeFactoredTma) return pick_fb<true, kModeFactoredTma>(spt, T);
        if (mode == MODE_FACTORED) return pick_fb<true, MODE_FACTORED>(spt, T);
        if (mode == MODE_RAW) return pick_fb<true, MODE_RAW>(spt, T);
        return pick_fb<true, MODE_EXACT>(spt, T);
    }
    if (mode == kModeFactoredTma) return pick_fb<false, kModeFactoredTma>(spt, T);
    if (mode == MODE_FACTORED) return pick_fb<false, MODE_FACTORED>(spt, T);
    if (mode == MODE_RAW) return pick_fb<false, MODE_RAW>(spt, T);
    return pick_fb<false, MODE_EXACT>(spt, T);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel) and
// size: later launches needing no more shared memory skip the driver call.
static fb_status set_smem(const void *fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    size_t &cur = done[{dev, fn}];
    if (bytes <= cur) return FB_OK;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) { set_cuda_error("cudaFuncSetAttribute", (int)e); return FB_ERR_CUDA; }
    cur = bytes;
    return FB_OK;
}

static fb_status check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_cuda_error(what, (int)e); return FB_ERR_CUDA; }
    return FB_OK;
}

template <bool BWD, int S>
KFn pick_fbc(int spt, int T, int nop, int iz);
extern template KFn pick_fbc<false, 2>(int, int, int, int);
extern template KFn pick_fbc<false, 4>(int, int, int, int);
extern template KFn pick_fbc<true, 2>(int, int, int, int);
extern template KFn pick_fbc<true, 4>(int, int, int, int);

// Does this launch run the cluster-batched kernel k_fbc (fb_cluster.cu)?
static bool use_cluster(bool bwd, const FBArgs &a, bool raw) {
    const Graph &G = a.g;
    if (!G.cp.ok || raw || G.G != 1 || G.mode != MODE_FACTORED) return false;
    return !bwd || a.post_kind != POST_PDF_COMPACT;
}

// CTAs a launch occupies (one per SM): what lfmmi leaves to the numerator pass.
static int den_ctas(const Graph &G, const FBArgs &a) {
    if (use_cluster(false, a, false)) return G.cp.C * ((a.B + G.cp.S - 1) / G.cp.S);
    return a.B;
}

static fb_status launch_fbc(bool bwd, const FBArgs &a, cudaStream_t s) {
    const Graph &G = a.g;
    const CPlan &P = G.cp;
    FBArgs aa = a;
    aa.tma = (a.D % 4 == 0) && (((uintptr_t)a.emis & 15) == 0);  // 16-byte emission copies
    // the lfmmi den backward normalises γ through the forward's log Z (IZ, fb_cluster.cu)
    const int iz = bwd && a.post_kind == POST_GRAD && a.ascale_in && a.logZ_fwd;
    KFn fn = bwd ? (P.S == 4 ? pick_fbc<true, 4>(P.spt, P.T, P.nop, iz) : pick_fbc<true, 2>(P.spt, P.T, 0, iz))
                 : (P.S == 4 ? pick_fbc<false, 4>(P.spt, P.T, P.nop, 0) : pick_fbc<false, 2>(P.spt, P.T, 0, 0));
    const size_t sm = cl_layout(bwd ? P.bwd.bytes_max : P.fwd.bytes_max, P.K_int, P.Kc_max, P.Dc_max, P.S, P.C,
                                P.T / 32, bwd, P.nop != 0).total;
    if (fb_status r0 = set_smem((const void *)fn, sm); r0 != FB_OK) return r0;
    cudaError_t e_launch = cudaSuccess;
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3((unsigned)(P.C * ((a.B + P.S - 1) / P.S)), 1, 1);
    cfg.blockDim = dim3((unsigned)P.T, 1, 1);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)P.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    {
        ProfScope ps(bwd ? "k_fbc_bwd[G=1]" : "k_fbc_fwd[G=1]", s);
        e_launch = cudaLaunchKernelEx(&cfg, fn, aa);
    }
    if (e_launch != cudaSuccess) { set_cuda_error("k_fbc launch", (int)e_launch); return FB_ERR_CUDA; }
    return check_launch("k_fbc launch");
}

// Numerator forward + backward in one persistent launch (k_fb_num), for CTA
// sizes 128 / 256; returns FB_ERR_UNSUPPORTED otherwise (the caller then issues
// the two passes separately).
using KFnNum = void (*)(FBArgs, FBArgs);
static KFnNum pick_fb_num(int spt, int T) {
    if (T == 128) {
        switch (spt) {
            case 1: return k_fb_num<1, 128>;
            case 2: return k_fb_num<2, 128>;
            case 3: return k_fb_num<3, 128>;
            case 4: return k_fb_num<4, 128>;
            case 6: return k_fb_num<6, 128>;
            default: return k_fb_num<8, 128>;
        }
    }
    if (T == 256) {
        switch (spt) {
            case 1: return k_fb_num<1, 256>;
            case 2: return k_fb_num<2, 256>;
            case 3: return k_fb_num<3, 256>;
            case 4: return k_fb_num<4, 256>;
            case 6: return k_fb_num<6, 256>;
            default: return k_fb_num<8, 256>;
        }
    }
    return nullptr;
}
static fb_status launch_fb_num(const FBArgs &af, const FBArgs &ab, cudaStream_t s, int idle_sms) {
    const Graph &G = af.g;
    KFnNum fn = pick_fb_num(G.spt, G.T);
    if (!fn) return FB_ERR_UNSUPPORTED;
    const size_t sm = std::max(smem_bytes(G, false, false),
                               smem_bytes(G, true, true) + pdf_region(POST_PDF_COMPACT, G.pm.U_max, G.D).bytes);
    if (fb_status r0 = set_smem((const void *)fn, sm); r0 != FB_OK) return r0;
    int grid = af.B;
    if (idle_sms > 0) {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, G.T, sm);
        grid = std::max(1, std::min(af.B, idle_sms * std::max(occ, 1)));
    }
    {
        ProfScope ps("k_fb_num[G=B]", s);
        fn<<<grid, G.T, sm, s>>>(af, ab);
    }
    return check_launch("k_fb_num launch");
}

// idle_sms > 0: launch only as many (persistent) CTAs as fit on that many SMs.
static fb_status launch_fb(bool bwd, const FBArgs &a, cudaStream_t s, bool raw = false, int idle_sms = 0) {
    const Graph &G = a.g;
    if (use_cluster(bwd, a, raw)) return launch_fbc(bwd, a, s);
    if (!G.legacy_ok) return FB_ERR_UNSUPPORTED;
    const bool post_pdf = bwd && a.post_kind != POST_NONE && a.post_kind != POST_STATE;
    size_t sm = smem_bytes(G, bwd, post_pdf) + (post_pdf ? pdf_region(a.post_kind, G.pm.U_max, a.D).bytes : 0);
    // φ rows through TMA when they are 16-byte aligned and the two row buffers fit
    const size_t tma_bytes = fbx_a16(2 * (size_t)a.D * 4) + 16;
    FBArgs aa = a;
    aa.tma = G.mode == MODE_FACTORED && !raw && (a.D % 4 == 0) && (((uintptr_t)a.emis & 15) == 0) &&
             sm + tma_bytes <= (size_t)kSmemLimit && std::getenv("FBX_NO_TMA") == nullptr;
    if (aa.tma) sm += tma_bytes;
    // the lfmmi den backward normalises γ through the forward's log Z (kModeGradIZ, fb_device.cuh)
    const bool iz = bwd && aa.tma && a.post_kind == POST_GRAD && a.ascale_in && a.logZ_fwd;
    KFn fn = pick(bwd, raw ? (int)MODE_RAW : (iz ? kModeGradIZ : (aa.tma ? kModeFactoredTma : G.mode)), G.spt, G.T);
    if (fb_status r0 = set_smem((const void *)fn, sm); r0 != FB_OK) return r0;
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

// Side stream + fork/join events for the concurrent numerator pass of
// lfmmi_loss_grad, one set per (device, caller stream): calls on different
// caller streams never share events or side streams, and a per-set mutex is held
// from the fork record to the join wait, so concurrent host threads calling on
// the same stream cannot interleave their fork/join pairs either (§8(b):
// re-entrant entry points, multiple streams allowed).
struct SideRes {
    int dev = -1;
    cudaStream_t caller = nullptr;
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    std::mutex mu;
};
static std::mutex g_side_mu;
static std::vector<std::unique_ptr<SideRes>> g_side;

static SideRes *side_res(int dev, cudaStream_t caller, fb_status &err) {
    std::lock_guard<std::mutex> lk(g_side_mu);
    for (auto &r : g_side)
        if (r->dev == dev && r->caller == caller) return r.get();
    auto r = std::make_unique<SideRes>();
    r->dev = dev;
    r->caller = caller;
    cudaError_t e = cudaStreamCreateWithFlags(&r->s, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->join, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        set_cuda_error("lfmmi side stream/events", (int)e);
        err = FB_ERR_CUDA;
        return nullptr;
    }
    g_side.push_back(std::move(r));
    return g_side.back().get();
}

// Per-device SM count (cached: the attribute query is not free on every call).
static int sm_count(int dev) {
    static std::mutex mu;
    static int cache[64] = {0};
    std::lock_guard<std::mutex> lk(mu);
    int &c = cache[dev & 63];
    if (!c) cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    return c > 0 ? c : 148;
}

struct WsLayout {
    size_t den_alpha, num_alpha, gnum, zn, zd, nst, den_scale, total;
};
static size_t a256(size_t x) { return (x + 255) & ~size_t(255); }
static WsLayout ws_layout(const Graph &num, const Graph &den, int B, int N_max) {
    WsLayout w;
    size_t o = 0;
    // den α̂: rows of K (one CTA per sequence) or of the cluster plan's K_int (internal order)
    // den α̂: rows of K (one CTA per sequence) or, for the cluster plan, [cluster][n][K_int][S]
    // (the S sequences of a cluster interleaved per state: one vector access per state)
    const size_t Bp = den.cp.ok ? (size_t)((B + den.cp.S - 1) / den.cp.S) * den.cp.S : (size_t)B;
    w.den_alpha = o; o += a256(Bp * N_max * std::max(den.K_tot, den.cp.ok ? den.cp.K_int : 0) * 4);
    w.num_alpha = o; o += a256((size_t)N_max * num.K_tot * 8);  // float64 when the numerator runs raw
    w.gnum = o; o += a256((size_t)N_max * num.pm.U_tot * 4);
    w.zn = o; o += a256((size_t)B * 8);
    w.zd = o; o += a256((size_t)B * 8);
    w.nst = o; o += a256((size_t)B * 4);
    w.den_scale = o; o += a256((size_t)B * N_max * 8);  // the den forward's per-frame offsets C_n
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
    if (fb_status r0 = set_smem((const void *)k_posteriors, sm); r0 != FB_OK) return r0;
    {
        ProfScope ps("k_posteriors", s);
        k_posteriors<<<(unsigned)((size_t)B * N_max), 256, sm, s>>>(G, alpha, beta, lengths, seq_status, B, N_max,
                                                                  G.D, pdf_level, post);
    }
    return check_launch("k_posteriors launch");
}

extern "C" fb_status fb_gap(fb_graph g, const float *alpha, const double *alpha_scale, const float *beta,
                            const double *beta_scale, const double *logZ, const int32_t *lengths,
                            const int32_t *seq_status, int32_t B, int32_t N_max, double *gap, void *stream) {
    if (!g || !alpha || !alpha_scale || !beta || !beta_scale || !logZ || !lengths || !gap || B < 1 || N_max < 1)
        return FB_ERR_INVALID_ARG;
    if (!(g->g.G == 1 || g->g.G == B) || g->g.dry) return FB_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    {
        ProfScope ps("k_gap", s);
        k_gap<<<(unsigned)B, 256, 0, s>>>(g->g, alpha, alpha_scale, beta, beta_scale, logZ, lengths, seq_status, B,
                                          N_max, gap);
    }
    return check_launch("k_gap launch");
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
    // the bank-relabelled twin of a shared factored graph (fb_graph.cpp): same sequences, same
    // pdf-level gradient; only the private α̂ lattice is in its state order
    if (den->perm) den = den->perm;
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
    double *den_scale = (double *)(ws + L.den_scale);
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return FB_ERR_CUDA;
    fb_status r = FB_OK;
    SideRes *sr = side_res(dev, s, r);
    if (!sr) return r;
    std::lock_guard<std::mutex> side_lock(sr->mu);  // fork record … join wait of this call
    // The fork point is recorded before the denominator forward so the numerator
    // pass depends only on prior work; the denominator forward is submitted first:
    // its B CTAs each take a whole SM (registers and shared memory), so the
    // numerator CTAs land on the SMs it leaves idle and the two run concurrently.
    cudaEventRecord(sr->fork, s);
    {
        FBArgs a = base_args(den, log_emis, lengths, B, N_max);
        a.lat = den_alpha; a.logZ = zd; a.status = seq_status; a.lat_int = 1;
        a.scale = den_scale;
        if ((r = launch_fb(false, a, s)) != FB_OK) return r;
    }
    cudaStreamWaitEvent(sr->s, sr->fork, 0);
    // SMs the denominator passes leave idle (one den CTA per SM)
    const int nsm = sm_count(dev);
    const int idle = nsm - std::min(den_ctas(den->g, base_args(den, log_emis, lengths, B, N_max)), nsm);
    const int confine = idle >= 8 ? idle : 0;
    {
        FBArgs a = base_args(num, log_emis, lengths, B, N_max);
        a.logZ = zn; a.status = nst;
        if (raw) a.lat64 = num_alpha64; else a.lat = num_alpha;
        FBArgs c = base_args(num, log_emis, lengths, B, N_max);
        c.status = nst; c.post = gnum; c.post_kind = POST_PDF_COMPACT;
        if (raw) { c.alpha64 = num_alpha64; c.logZ_in = zn; } else c.alpha = num_alpha;
        r = (raw && !std::getenv("FBX_NUM_SPLIT")) ? launch_fb_num(a, c, sr->s, confine) : FB_ERR_UNSUPPORTED;
        if (r == FB_ERR_UNSUPPORTED) {
            if ((r = launch_fb(false, a, sr->s, raw, confine)) != FB_OK) return r;
            r = launch_fb(true, c, sr->s, raw, confine);
        }
        if (r != FB_OK) return r;
    }
    cudaEventRecord(sr->join, sr->s);
    // denominator backward + fused −Γ_den gradient epilogue: independent of the numerator
    {
        FBArgs c = base_args(den, log_emis, lengths, B, N_max);
        c.status = seq_status; c.alpha = den_alpha; c.lat_int = 1;
        c.post = grad; c.post_kind = POST_GRAD;
        if (!std::getenv("FBX_NO_IZ")) { c.ascale_in = den_scale; c.logZ_fwd = zd; }
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
    const bool glob = G.vit_global != 0;
#define FBX_VIT(S) (glob ? (small ? k_viterbi<S, 256, true> : k_viterbi<S, 1024, true>) \
                         : (small ? k_viterbi<S, 256, false> : k_viterbi<S, 1024, false>))
    switch (G.spt) {
        case 1: fn = FBX_VIT(1); break;
        case 2: fn = FBX_VIT(2); break;
        case 3: fn = FBX_VIT(3); break;
        case 4: fn = FBX_VIT(4); break;
        case 6: fn = FBX_VIT(6); break;
        default: fn = FBX_VIT(8); break;
    }
#undef FBX_VIT
    const size_t sm = viterbi_smem_bytes(G, glob);
    if (fb_status r0 = set_smem((const void *)fn, sm); r0 != FB_OK) return r0;
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
