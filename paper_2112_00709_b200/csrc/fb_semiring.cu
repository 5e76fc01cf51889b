// fb_semiring.cu — the fused one-CTA-per-sequence forward (Eq. (13))
// written once for any semiring ("trivial to extend to other
// semirings"): the same arc schedule, shared-memory vector and
// per-frame phase A (rows ⊕ over in-arcs of u ⊗ T) / phase B (⊗ emission) as the
// log-semiring kernels, instantiated for
//   FB_SEMIRING_LOG       ⊕ = log-sum-exp (max-then-sum), ⊗ = +   → log Z_b
//   FB_SEMIRING_TROPICAL  ⊕ = max,                        ⊗ = +   → best-path score
//   FB_SEMIRING_PROB      ⊕ = +,                          ⊗ = ×   → Z_b (linear domain)
// in float64 without normalisation, so the probability instance underflows to 0
// exactly where the paper says the linear domain does while the log and
// tropical ones stay finite.  It runs over the tropical kernel's schedule
// (natural-log weights, float64 gathered elements; Graph::vit), from shared
// memory or streamed from L2 when it does not fit (Graph::vit_global).
// A semiring-generic companion of the tuned kernels, not a replacement: the
// log-semiring hot path (k_fb) keeps its exp-factorised fp32 arithmetic.
#include "fb_device.cuh"

namespace fbx {

template <int SR>
struct FSr;
template <>
struct FSr<FB_SEMIRING_LOG> {
    static __device__ __forceinline__ double zero() { return -INFINITY; }
    static __device__ __forceinline__ double lift(double logx) { return logx; }  // a natural-log weight / emission
    static __device__ __forceinline__ double times(double a, double b) { return a + b; }
    struct Acc {  // running (m, s): value m + log s
        double m = -INFINITY, s = 0.0;
        __device__ __forceinline__ void add(double x) {
            if (x == -INFINITY) return;
            if (x > m) { s = s * exp(m - x) + 1.0; m = x; }
            else s += exp(x - m);
        }
        __device__ __forceinline__ void merge(const Acc &o) {
            if (o.m == -INFINITY) return;
            if (m == -INFINITY) { *this = o; return; }
            if (o.m > m) { s = s * exp(m - o.m) + o.s; m = o.m; }
            else s += o.s * exp(o.m - m);
        }
        __device__ __forceinline__ double value() const { return m == -INFINITY ? -INFINITY : m + log(s); }
    };
};
template <>
struct FSr<FB_SEMIRING_TROPICAL> {
    static __device__ __forceinline__ double zero() { return -INFINITY; }
    static __device__ __forceinline__ double lift(double logx) { return logx; }
    static __device__ __forceinline__ double times(double a, double b) { return a + b; }
    struct Acc {
        double m = -INFINITY, s = 0.0;  // s unused
        __device__ __forceinline__ void add(double x) { m = fmax(m, x); }
        __device__ __forceinline__ void merge(const Acc &o) { m = fmax(m, o.m); }
        __device__ __forceinline__ double value() const { return m; }
    };
};
template <>
struct FSr<FB_SEMIRING_PROB> {
    static __device__ __forceinline__ double zero() { return 0.0; }
    static __device__ __forceinline__ double lift(double logx) { return exp(logx); }
    static __device__ __forceinline__ double times(double a, double b) { return a * b; }
    struct Acc {
        double m = 0.0, s = 0.0;  // m = the sum
        __device__ __forceinline__ void add(double x) { m += x; }
        __device__ __forceinline__ void merge(const Acc &o) { m += o.m; }
        __device__ __forceinline__ double value() const { return m; }
    };
};

// Fixed-order warp merge of accumulators (xor tree: bitwise the same in every lane).
template <int SR>
__device__ __forceinline__ void warp_merge(typename FSr<SR>::Acc &a) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        typename FSr<SR>::Acc b;
        b.m = __shfl_xor_sync(0xffffffffu, a.m, o);
        b.s = __shfl_xor_sync(0xffffffffu, a.s, o);
        // lanes l and l^o must combine in the same order: the lower lane's value first
        if (threadIdx.x & o) { typename FSr<SR>::Acc c = b; c.merge(a); a = c; }
        else a.merge(b);
    }
}

struct SrArgs {
    Graph g;
    const float *emis;
    const int *lengths;
    int B, N_max, D;
    double *score;
    int *status;
};

// One CTA per sequence; phase A walks the schedule's slices (header | index |
// weight layout of Sched, fb_internal.h): lane l ⊕-reduces its row segment, the
// g lanes of a split row merge by a fixed xor tree, the leader stores the row.
template <int SR, int SPT, int MAXT, bool GLOB>
__global__ void __launch_bounds__(MAXT, (MAXT == 1024 ? 1 : 2)) k_fwd_sr(const SrArgs a) {
    using R = FSr<SR>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Graph &G = a.g;
    const Sched &S = G.vit;
    const int b = blockIdx.x;
    const int gi = (G.G == 1) ? 0 : b;
    const int T = blockDim.x;  // the schedule's CTA size (Graph::T ≤ MAXT)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = T >> 5;
    const int s0 = G.state_off[gi];
    const int K = G.state_off[gi + 1] - s0;
    const int N = a.lengths[b];
    const SmemLayout SL = smem_layout(GLOB ? 0 : S.bytes_max, T * SPT, true, false);
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t a_u = sb + (uint32_t)SL.u, a_row = sb + (uint32_t)SL.part, a_red = sb + (uint32_t)SL.red;
    if (N < 1 || N > a.N_max) {
        if (tid == 0) { a.score[b] = R::zero(); a.status[b] = FB_SEQ_BAD_LENGTH; }
        return;
    }
    if (!GLOB) {
        const uint4 *src = (const uint4 *)(S.rec + S.rec_off[gi]);
        uint4 *dst = (uint4 *)(smem_raw + SL.rec);
        for (int x = tid; x < (S.rec_bytes[gi] >> 4); x += T) dst[x] = src[x];
    }
    const int nsl = S.warp_nsl[gi * W + warp];
    const uint32_t mysl = sb + (uint32_t)SL.rec + (uint32_t)S.warp_off[gi * W + warp];
    const unsigned char *mysl_g = S.rec + S.rec_off[gi] + S.warp_off[gi * W + warp];
    int pdfk[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const int j = tid + k * T;
        pdfk[k] = G.pdf[s0 + (j < K ? j : 0)];  // inert slots read a column the graph reads
        sts_v(a_row + (uint32_t)j * 8, R::zero());  // rows without in-arcs stay 0̄
    }
    const float *em = a.emis + (size_t)b * a.N_max * a.D;
    float vsum = 0.f;
    double uk[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) {  // frame 0: π ⊗ v_0 (ledger L6)
        const int j = tid + k * T;
        const float v = __ldg(em + pdfk[k]);
        vsum += j < K ? v : 0.f;
        uk[k] = j < K ? R::times(R::lift((double)G.init_nat[s0 + j]), R::lift((double)v)) : R::zero();
        sts_v(a_u + (uint32_t)j * 8, uk[k]);
    }
    for (int n = 1; n < N; ++n) {
        __syncthreads();  // u of frame n-1 visible
        // ---- phase A: rows ⊕_{i→j} u(i) ⊗ T_ij
        const unsigned char *gcur = mysl_g;
        uint32_t cur = mysl;
        for (int q = 0; q < nsl; ++q) {
            const uint32_t h = GLOB ? __ldg((const uint32_t *)gcur + lane) : lds_u32(cur + lane * 4);
            const int row = (int)(h & 0xFFFFu) - 1, lg = (int)((h >> 16) & 7u), L2 = (int)(h >> 19);
            typename R::Acc acc;
            for (int s = 0; s < L2; ++s) {
                uint32_t ix;
                float2 w2;
                if (GLOB) {
                    ix = __ldg((const uint32_t *)(gcur + 128) + lane + 32 * s);
                    w2 = __ldg((const float2 *)(gcur + 128 + (size_t)L2 * 128) + lane + 32 * s);
                } else {
                    ix = lds_u32(cur + 128 + (uint32_t)s * 128 + lane * 4);
                    w2 = lds_f2(cur + 128 + (uint32_t)L2 * 128 + (uint32_t)s * 256 + lane * 8);
                }
                // null slots carry weight −∞ (natural log): 0̄ in every semiring after lift
                acc.add(R::times(lds_v(a_u + (ix & 0xFFFFu), 0.0), R::lift((double)w2.x)));
                acc.add(R::times(lds_v(a_u + (ix >> 16), 0.0), R::lift((double)w2.y)));
            }
            for (int o = 1; o < (1 << lg); o <<= 1) {
                typename R::Acc other;
                other.m = __shfl_xor_sync(0xffffffffu, acc.m, o);
                other.s = __shfl_xor_sync(0xffffffffu, acc.s, o);
                if (lane & o) { typename R::Acc c = other; c.merge(acc); acc = c; }
                else acc.merge(other);
            }
            if (row >= 0) sts_v(a_row + (uint32_t)row * 8, acc.value());
            cur += 128 + (uint32_t)L2 * 384;
            gcur += 128 + (size_t)L2 * 384;
        }
        __syncthreads();
        // ---- phase B: ⊗ v_n
        const float *rowp = em + (size_t)n * a.D;
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const int j = tid + k * T;
            const float v = __ldg(rowp + pdfk[k]);
            vsum += j < K ? v : 0.f;
            uk[k] = j < K ? R::times(lds_v(a_row + (uint32_t)j * 8, 0.0), R::lift((double)v)) : R::zero();
            sts_v(a_u + (uint32_t)j * 8, uk[k]);
        }
    }
    // ---- termination: ⊕_j u(j) ⊗ ω(j), fixed-order block reduction
    typename R::Acc acc;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
        const int j = tid + k * T;
        if (j < K) acc.add(R::times(uk[k], R::lift((double)G.final_nat[s0 + j])));
    }
    warp_merge<SR>(acc);
    const int bad = __syncthreads_or(!(vsum < INFINITY));
    if (lane == 0) {
        sts_v(a_red + (uint32_t)warp * 16, acc.m);
        sts_v(a_red + (uint32_t)warp * 16 + 8, acc.s);
    }
    __syncthreads();
    if (warp == 0) {
        typename R::Acc t;
        if (lane < W) { t.m = lds_v(a_red + (uint32_t)lane * 16, 0.0); t.s = lds_v(a_red + (uint32_t)lane * 16 + 8, 0.0); }
        warp_merge<SR>(t);
        if (lane == 0) {
            const double z = t.value();
            int st = 0;
            if (bad) st |= FB_SEQ_NONFINITE_INPUT;  // precedence as in fb.h: non-finite, else empty
            else if (!(SR == FB_SEMIRING_PROB ? z > 0.0 : z > -INFINITY)) st |= FB_SEQ_EMPTY_LATTICE;
            // an underflowed linear-domain Z is reported as computed (0), flagged empty like 0̄
            a.score[b] = st & FB_SEQ_NONFINITE_INPUT ? R::zero() : z;
            a.status[b] = st;
        }
    }
}

using SrFn = void (*)(SrArgs);
template <int SR, bool GLOB>
static SrFn pick_sr(int spt, bool small) {
#define FBX_SR(S) (small ? k_fwd_sr<SR, S, 256, GLOB> : k_fwd_sr<SR, S, 1024, GLOB>)
    switch (spt) {
        case 1: return FBX_SR(1);
        case 2: return FBX_SR(2);
        case 3: return FBX_SR(3);
        case 4: return FBX_SR(4);
        case 6: return FBX_SR(6);
        default: return FBX_SR(8);
    }
#undef FBX_SR
}

}  // namespace fbx

using namespace fbx;

extern "C" fb_status fb_forward_semiring(fb_graph g, int32_t semiring, const float *log_emis, const int32_t *lengths,
                                         int32_t B, int32_t N_max, double *score, int32_t *seq_status, void *stream) {
    if (!g || !log_emis || !lengths || !score || !seq_status || B < 1 || N_max < 1) return FB_ERR_INVALID_ARG;
    if (!(g->g.G == 1 || g->g.G == B) || g->g.dry) return FB_ERR_INVALID_ARG;
    if (!g->g.vit_ok) return FB_ERR_UNSUPPORTED;
    const Graph &G = g->g;
    const bool small = G.T <= 256, glob = G.vit_global != 0;
    SrFn fn = nullptr;
    switch (semiring) {
        case FB_SEMIRING_LOG: fn = glob ? pick_sr<FB_SEMIRING_LOG, true>(G.spt, small) : pick_sr<FB_SEMIRING_LOG, false>(G.spt, small); break;
        case FB_SEMIRING_TROPICAL:
            fn = glob ? pick_sr<FB_SEMIRING_TROPICAL, true>(G.spt, small) : pick_sr<FB_SEMIRING_TROPICAL, false>(G.spt, small);
            break;
        case FB_SEMIRING_PROB: fn = glob ? pick_sr<FB_SEMIRING_PROB, true>(G.spt, small) : pick_sr<FB_SEMIRING_PROB, false>(G.spt, small); break;
        default: return FB_ERR_INVALID_ARG;
    }
    // the tropical kernel's shared-memory size (schedule + float64 u + rows), without its arg array
    const size_t sm = smem_layout(glob ? 0 : G.vit.bytes_max, G.T * G.spt, true, false).total;
    cudaError_t e = cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) { set_cuda_error("cudaFuncSetAttribute(k_fwd_sr)", (int)e); return FB_ERR_CUDA; }
    SrArgs a;
    std::memset(&a, 0, sizeof a);
    a.g = G; a.emis = log_emis; a.lengths = lengths; a.B = B; a.N_max = N_max; a.D = G.D; a.score = score;
    a.status = seq_status;
    fn<<<(unsigned)B, (unsigned)G.T, sm, (cudaStream_t)stream>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) { set_cuda_error("k_fwd_sr launch", (int)e); return FB_ERR_CUDA; }
    return FB_OK;
}
