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

// Backward frame of the same batch matrix (Eq. (14) with ledger L2):
//   y_n(i) = ⊕_{i→j} T'_ij ⊗ v_{n+1}(j) ⊗ y_{n+1}(j),   y_{N_max} = 1̄ on phony, 0̄ elsewhere
// (the final weights live on the arcs into phony), over the augmented out-arc
// lists; the same launch writes the frame's posteriors (Eq. (15), read as
// semifield division, ledger L5) from the stored forward lattice X:
//   post_n(k) = X_n(k) ⊗ y_n(k) ⊘ Z_b,   Z_b = X_{N_max}(phony_b)
// for real states k and n < N_b (0 otherwise; layout of fb.h: [B][N_max][K] for
// G == 1, packed per sequence for G == B).  Log: γ = exp(x + y − log Z); prob:
// γ = x·y / Z; tropical: the max-marginal ratio exp(x + y − best) ∈ [0, 1], 1 on
// the states a best path visits.
template <int SR>
__global__ void __launch_bounds__(256) k_literal_bwd_frame(const Graph G, const float *emis, const int *lengths,
                                                           int B, int N_max, int n, const double *X,
                                                           const double *y_next, double *y_cur, double *post) {
    using R = Semiring<SR>;
    const LitPlan &P = G.lit;
    const long long rows = P.rows_per_batch(B);
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
        int b, j;
        P.locate(r, B, b, j);
        const int g = (G.G == 1) ? 0 : b;
        const int s0 = G.state_off[g];
        const int K = G.state_off[g + 1] - s0;
        const int N = lengths[b];
        const long long base = r - j;
        double y;
        if (n == N_max) {
            y = (j == K) ? R::one() : R::zero();
        } else {
            typename R::Acc acc;
            const int row = P.row_off[g] + j;
            for (int e = P.optr[row]; e < P.optr[row + 1]; ++e) {
                const int d = P.odst[e];
                double v;  // v_{n+1}(d)
                if (d == K) v = (n + 1 < N) ? R::zero() : R::one();
                else if (n + 1 >= N) v = R::zero();
                else {
                    const double phi = (double)emis[((size_t)b * N_max + n + 1) * G.D + G.pdf[s0 + d]];
                    v = (SR == FB_SEMIRING_PROB) ? exp(phi) : phi;
                }
                acc.add(R::times(R::times(R::lift_w(P.ow[e]), v), y_next[base + d]));
            }
            y = acc.value();
        }
        y_cur[r] = y;
        if (post && j < K && n < N_max) {
            const size_t o = (G.G == 1 ? (size_t)b * N_max * K : (size_t)N_max * s0) + (size_t)n * K + j;
            const double Z = X[(size_t)N_max * rows + base + K];  // x_{N_max}(phony_b)
            double gam = 0.0;
            if (n < N && N <= N_max) {
                const double xy = R::times(X[(size_t)n * rows + r], y);
                if (SR == FB_SEMIRING_PROB) gam = (Z > 0.0) ? xy / Z : 0.0;
                else gam = (Z > -INFINITY && xy > -INFINITY) ? exp(xy - Z) : 0.0;
            }
            post[o] = gam;
        }
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

// Forward storing every frame's batch vector X_n (n = 0 … N_max), then N_max + 1
// backward launches writing the posteriors frame by frame.
template <int SR>
static fb_status run_literal_fb(const Graph &G, const float *emis, const int *lengths, int B, int N_max, double *score,
                                double *post, double *X, double *y0, double *y1, cudaStream_t s) {
    const long long rows = G.lit.rows_per_batch(B);
    const int grid = (int)std::min<long long>((rows + 255) / 256, 148 * 16);
    for (int n = 0; n <= N_max; ++n)
        k_literal_frame<SR><<<grid, 256, 0, s>>>(G, emis, lengths, B, N_max, n, X + (size_t)(n ? n - 1 : 0) * rows,
                                                 X + (size_t)n * rows, score);
    for (int n = N_max; n >= 0; --n) {
        const double *yn = (n & 1) ? y0 : y1;
        double *yc = (n & 1) ? y1 : y0;
        k_literal_bwd_frame<SR><<<grid, 256, 0, s>>>(G, emis, lengths, B, N_max, n, X, yn, yc, post);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_cuda_error("k_literal launch", (int)e); return FB_ERR_CUDA; }
    return FB_OK;
}

}  // namespace fbx

using namespace fbx;

extern "C" size_t fb_literal_fb_workspace_bytes(fb_graph g, int32_t B, int32_t N_max) {
    if (!g || B < 1 || N_max < 1 || !(g->g.G == 1 || g->g.G == B)) return 0;
    return ((size_t)N_max + 3) * (size_t)g->g.lit.rows_per_batch(B) * sizeof(double) + 256;
}

extern "C" fb_status fb_forward_backward_literal(fb_graph g, int32_t semiring, const float *log_emis,
                                                 const int32_t *lengths, int32_t B, int32_t N_max, double *score,
                                                 double *post, void *workspace, size_t workspace_bytes, void *stream) {
    if (!g || !log_emis || !lengths || !score || B < 1 || N_max < 1) return FB_ERR_INVALID_ARG;
    if (!(g->g.G == 1 || g->g.G == B) || g->g.dry) return FB_ERR_INVALID_ARG;
    if (!workspace || workspace_bytes < fb_literal_fb_workspace_bytes(g, B, N_max)) return FB_ERR_WORKSPACE;
    const Graph &G = g->g;
    const size_t rows = (size_t)G.lit.rows_per_batch(B);
    double *X = (double *)workspace, *y0 = X + ((size_t)N_max + 1) * rows, *y1 = y0 + rows;
    cudaStream_t s = (cudaStream_t)stream;
    switch (semiring) {
        case FB_SEMIRING_LOG:
            return run_literal_fb<FB_SEMIRING_LOG>(G, log_emis, lengths, B, N_max, score, post, X, y0, y1, s);
        case FB_SEMIRING_TROPICAL:
            return run_literal_fb<FB_SEMIRING_TROPICAL>(G, log_emis, lengths, B, N_max, score, post, X, y0, y1, s);
        case FB_SEMIRING_PROB:
            return run_literal_fb<FB_SEMIRING_PROB>(G, log_emis, lengths, B, N_max, score, post, X, y0, y1, s);
        default: return FB_ERR_INVALID_ARG;
    }
}

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
