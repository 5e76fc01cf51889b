// fb_literal.cu — the paper's own execution strategy, semiring-generic
// (SURVEY §8(f) N4), kept as an in-framework A/B baseline for the fused kernels.
//
// a batch of B sequences is one block-diagonal transition matrix
// (one block per sequence's graph), sequences shorter than the batch are padded
// with a phony state (ledger L8: arcs s → phony weighted ω(s), a 1̄ self-loop;
// v(phony) = 0̄ for n < N_b and 1̄ after, real states 0̄ after), and every frame
// is ONE sparse matrix-vector product over the whole batch vector:
//   x_n = v_n ⊗ Tᵀ x_{n−1}          (Eq. (13))
// run for N_max + 1 frames, so that x_{N_max}(phony_b) = ⊕ over accepting paths
// (Eq. (1) with final weights, ledger L4).  This is generic in the semiring
// ("trivial to extend to other semirings"):
//   SR_LOG      ⊕ = log-sum-exp, ⊗ = +   → log Z_b                  (forward algorithm)
//   SR_TROPICAL ⊕ = max,         ⊗ = +   → best path score          (Viterbi score)
//   SR_PROB     ⊕ = +,           ⊗ = ×   → Z_b in the linear domain (underflows)
// One thread per row of the composed matrix, one kernel launch per frame, float64
// values: deliberately the plain strategy, not the B200 design of fb_kernels.cu.
#include "fb_device.cuh"

namespace fbx {

template <int SR>
struct Semiring;
template <>
struct Semiring<FB_SEMIRING_LOG> {
    static __device__ __forceinline__ double zero() { return -INFINITY; }
    static __device__ __forceinline__ double one() { return 0.0; }
    static __device__ __forceinline__ double times(double a, double b) { return a + b; }
    static __device__ __forceinline__ double lift_w(double logw) { return logw; }  // natural-log weights
    // online ⊕ accumulator: (m, s) with value m + log s
    struct Acc {
        double m = -INFINITY, s = 0.0;
        __device__ __forceinline__ void add(double x) {
            if (x == -INFINITY) return;
            if (x > m) { s = s * exp(m - x) + 1.0; m = x; }
            else s += exp(x - m);
        }
        __device__ __forceinline__ double value() const { return m == -INFINITY ? -INFINITY : m + log(s); }
    };
};
template <>
struct Semiring<FB_SEMIRING_TROPICAL> {
    static __device__ __forceinline__ double zero() { return -INFINITY; }
    static __device__ __forceinline__ double one() { return 0.0; }
    static __device__ __forceinline__ double times(double a, double b) { return a + b; }
    static __device__ __forceinline__ double lift_w(double logw) { return logw; }
    struct Acc {
        double m = -INFINITY;
        __device__ __forceinline__ void add(double x) { m = fmax(m, x); }
        __device__ __forceinline__ double value() const { return m; }
    };
};
template <>
struct Semiring<FB_SEMIRING_PROB> {
    static __device__ __forceinline__ double zero() { return 0.0; }
    static __device__ __forceinline__ double one() { return 1.0; }
    static __device__ __forceinline__ double times(double a, double b) { return a * b; }
    static __device__ __forceinline__ double lift_w(double logw) { return exp(logw); }
    struct Acc {
        double s = 0.0;
        __device__ __forceinline__ void add(double x) { s += x; }
        __device__ __forceinline__ double value() const { return s; }
    };
};

// One frame of the batch SpMV.  Rows of instance b are [inst_off(b), +K_b + 1);
// local row K_b is the phony state.  Member g's augmented in-arc lists
// (CSC with the phony arcs) start at lit.row_off[g] (rows) / arcs global.
template <int SR>
__global__ void __launch_bounds__(256) k_literal_frame(const Graph G, const float *emis, const int *lengths,
                                                       int B, int N_max, int n, const double *x_prev, double *x_next,
                                                       double *score) {
    using R = Semiring<SR>;
    const LitPlan &P = G.lit;
    const long long rows = P.rows_per_batch(B);
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
        int b, j;
        P.locate(r, B, b, j);
        const int g = (G.G == 1) ? 0 : b;
        const int K = G.state_off[g + 1] - G.state_off[g];
        const int N = lengths[b];
        const long long base = r - j;  // instance row 0
        double v;                      // v_n(j) in the semiring
        if (j == K) v = (n < N) ? R::zero() : R::one();
        else if (n >= N) v = R::zero();
        else {
            const double phi = (double)emis[((size_t)b * N_max + n) * G.D + G.pdf[G.state_off[g] + j]];
            v = (SR == FB_SEMIRING_PROB) ? exp(phi) : phi;
        }
        double out;
        if (n == 0) {
            const double pi = (j == K) ? -INFINITY : (double)G.init_nat[G.state_off[g] + j];
            out = (j == K) ? R::zero() : R::times(R::lift_w(pi), v);
        } else {
            typename R::Acc acc;
            const int row = P.row_off[g] + j;
            for (int e = P.ptr[row]; e < P.ptr[row + 1]; ++e) acc.add(R::times(x_prev[base + P.src[e]], R::lift_w(P.w[e])));
            out = R::times(acc.value(), v);
        }
        x_next[r] = out;
        if (j == K && n == N_max) score[b] = (SR == FB_SEMIRING_PROB) ? out : out;
    }
}

// Host driver: N_max + 1 launches (one SpMV per frame), ping-pong state vectors in the workspace.
template <int SR>
static fb_status run_literal(const Graph &G, const float *emis, const int *lengths, int B, int N_max, double *score,
                             double *x0, double *x1, cudaStream_t s) {
    const long long rows = G.lit.rows_per_batch(B);
    const int grid = (int)std::min<long long>((rows + 255) / 256, 148 * 16);
    for (int n = 0; n <= N_max; ++n) {
        const double *xp = (n & 1) ? x0 : x1;
        double *xn = (n & 1) ? x1 : x0;
        k_literal_frame<SR><<<grid, 256, 0, s>>>(G, emis, lengths, B, N_max, n, xp, xn, score);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_cuda_error("k_literal_frame launch", (int)e); return FB_ERR_CUDA; }
    return FB_OK;
}

}  // namespace fbx

using namespace fbx;

extern "C" size_t fb_literal_workspace_bytes(fb_graph g, int32_t B) {
    if (!g || B < 1 || !(g->g.G == 1 || g->g.G == B)) return 0;
    return 2 * (size_t)g->g.lit.rows_per_batch(B) * sizeof(double) + 256;
}

extern "C" fb_status fb_forward_literal(fb_graph g, int32_t semiring, const float *log_emis, const int32_t *lengths,
                                        int32_t B, int32_t N_max, double *score, void *workspace,
                                        size_t workspace_bytes, void *stream) {
    if (!g || !log_emis || !lengths || !score || B < 1 || N_max < 1) return FB_ERR_INVALID_ARG;
    if (!(g->g.G == 1 || g->g.G == B) || g->g.dry) return FB_ERR_INVALID_ARG;
    if (!workspace || workspace_bytes < fb_literal_workspace_bytes(g, B)) return FB_ERR_WORKSPACE;
    const Graph &G = g->g;
    const size_t half = (size_t)G.lit.rows_per_batch(B);
    double *x0 = (double *)workspace, *x1 = x0 + half;
    cudaStream_t s = (cudaStream_t)stream;
    switch (semiring) {
        case FB_SEMIRING_LOG: return run_literal<FB_SEMIRING_LOG>(G, log_emis, lengths, B, N_max, score, x0, x1, s);
        case FB_SEMIRING_TROPICAL:
            return run_literal<FB_SEMIRING_TROPICAL>(G, log_emis, lengths, B, N_max, score, x0, x1, s);
        case FB_SEMIRING_PROB: return run_literal<FB_SEMIRING_PROB>(G, log_emis, lengths, B, N_max, score, x0, x1, s);
        default: return FB_ERR_INVALID_ARG;
    }
}
