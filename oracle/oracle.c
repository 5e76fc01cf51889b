/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, float64 CPU implementation of what the hot path computes,
 * written from the paper (arXiv 2112.00709, /root/reference/PAPER.md, cited
 * as P:<line>) and the readings listed in DESIGN.md §"Readings of the paper".
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant with the CUDA path (paper_2112_00709_b200/csrc).
 *
 * Everything is the textbook recursion, unnormalised, in double precision:
 *   α_0(k)   = π(k) ⊗ v_0(k)                                  (ledger L6)
 *   α_n(j)   = v_n(j) ⊗ ⊕_{i→j} α_{n-1}(i) ⊗ T_ij            (P:86-88 with L1)
 *   β_{N-1}  = ω                                              (ledger L7)
 *   β_n(i)   = ⊕_{i→j} T_ij ⊗ v_{n+1}(j) ⊗ β_{n+1}(j)         (P:179-181 with L2)
 *   logZ     = ⊕_k α_{N-1}(k) ⊗ ω(k)                          (P:82 with L4)
 *   γ_n(k)   = exp(α_n(k) ⊗ β_n(k) ⊘ logZ)                    (P:81-83, P:182 with L5)
 *   Γ_n(d)   = Σ_{k : pdf_of[k] = d} γ_n(k)                   (ledger L9)
 *   ℒ        = logZ_num − logZ_den
 *   ∂ℒ/∂φ    = Γ_num − Γ_den
 * with ⊕ = log(e^a + e^b), ⊗ = + (P:166-167), ⊘ = −,
 * 0̄ = −∞, 1̄ = 0, and v_n(k) = φ[n, pdf_of[k]].
 *
 * ⊕ over a list is evaluated max-shifted in ascending index order; a list of
 * only −∞ returns −∞ without forming (−∞) − (−∞) (ledger L13).  There is no
 * per-frame normalisation: float64 keeps |α| ≤ ~1e4 exact to ~1e-12.
 *
 * Parity pins: tests/test_oracle_pins.py (brute force, closed forms,
 * torch ctc_loss, finite differences, invariants).  See DESIGN.md §Oracle.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NEG_INF (-INFINITY)

/* ⊕ of two elements. */
double oracle_logaddexp(double a, double b) {
    if (a == NEG_INF) return b;
    if (b == NEG_INF) return a;
    double m = a > b ? a : b;
    return m + log(exp(a - m) + exp(b - m));
}

/* ⊕ of a list, ascending index order (ledger L13, L14). */
static double lse_list(const double *x, long n) {
    double m = NEG_INF;
    for (long i = 0; i < n; ++i)
        if (x[i] > m) m = x[i];
    if (m == NEG_INF) return NEG_INF;
    double s = 0.0;
    for (long i = 0; i < n; ++i) s += exp(x[i] - m);
    return m + log(s);
}

/* One member graph of a block-diagonal composition, local ids. */
typedef struct {
    int K;              /* states */
    int nnz;            /* arcs */
    const int *row_ptr; /* global CSR row pointer, rows [off, off+K] */
    const int *col;     /* global destination ids */
    const float *logw;
    const float *log_init;
    const float *log_final;
    const int *pdf_of;
    int off;            /* first global state id */
    int arc0;           /* first arc index */
} graph_t;

static graph_t member(int G, const int *state_offsets, const int *row_ptr, const int *col,
                      const float *logw, const float *log_init, const float *log_final,
                      const int *pdf_of, int b) {
    int g = (G == 1) ? 0 : b;
    graph_t m;
    m.off = state_offsets[g];
    m.K = state_offsets[g + 1] - state_offsets[g];
    m.arc0 = row_ptr[m.off];
    m.nnz = row_ptr[m.off + m.K] - m.arc0;
    m.row_ptr = row_ptr + m.off;
    m.col = col;
    m.logw = logw;
    m.log_init = log_init + m.off;
    m.log_final = log_final + m.off;
    m.pdf_of = pdf_of + m.off;
    return m;
}

/* In-arc lists (CSC of T = CSR of Tᵀ, ledger L3), ascending source order. */
typedef struct { int *ptr; int *src; double *w; } inarcs_t;

static inarcs_t build_inarcs(const graph_t *g) {
    inarcs_t t;
    t.ptr = (int *)calloc((size_t)g->K + 1, sizeof(int));
    t.src = (int *)malloc(sizeof(int) * (size_t)(g->nnz > 0 ? g->nnz : 1));
    t.w = (double *)malloc(sizeof(double) * (size_t)(g->nnz > 0 ? g->nnz : 1));
    for (int i = 0; i < g->K; ++i)
        for (int a = g->row_ptr[i]; a < g->row_ptr[i + 1]; ++a) t.ptr[g->col[a] - g->off + 1]++;
    for (int j = 0; j < g->K; ++j) t.ptr[j + 1] += t.ptr[j];
    int *fill = (int *)calloc((size_t)g->K, sizeof(int));
    for (int i = 0; i < g->K; ++i)
        for (int a = g->row_ptr[i]; a < g->row_ptr[i + 1]; ++a) {
            int j = g->col[a] - g->off;
            int p = t.ptr[j] + fill[j]++;
            t.src[p] = i;
            t.w[p] = (double)g->logw[a];
        }
    free(fill);
    return t;
}

static void free_inarcs(inarcs_t *t) { free(t->ptr); free(t->src); free(t->w); }

static inline double emis_at(const double *emis_b, long D, int n, int pdf) {
    return emis_b[(long)n * D + pdf];
}

/* Returns 1 if anything the recursion reads is NaN or +∞ (−∞ is a legal 0̄). */
static int bad_value(double x) { return isnan(x) || (isinf(x) && x > 0); }

static int nonfinite_inputs(const graph_t *g, const double *emis_b, long D, int N) {
    for (int a = g->arc0; a < g->arc0 + g->nnz; ++a)
        if (bad_value(g->logw[a])) return 1;
    for (int k = 0; k < g->K; ++k)
        if (bad_value(g->log_init[k]) || bad_value(g->log_final[k])) return 1;
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < g->K; ++k)
            if (bad_value(emis_b[(long)n * D + g->pdf_of[k]])) return 1;
    return 0;
}

/* Forward, P:86-88 / P:176-178: alpha[N][K] (true log α). Returns logZ. */
static double forward_seq(const graph_t *g, const inarcs_t *in, const double *emis_b, long D, int N,
                          double *alpha, double *scratch) {
    int K = g->K;
    for (int k = 0; k < K; ++k)
        alpha[k] = (double)g->log_init[k] + emis_at(emis_b, D, 0, g->pdf_of[k]);
    for (int n = 1; n < N; ++n) {
        const double *prev = alpha + (long)(n - 1) * K;
        double *cur = alpha + (long)n * K;
        for (int j = 0; j < K; ++j) {
            long deg = in->ptr[j + 1] - in->ptr[j];
            for (long q = 0; q < deg; ++q) {
                long a = in->ptr[j] + q;
                scratch[q] = prev[in->src[a]] + in->w[a];
            }
            cur[j] = emis_at(emis_b, D, n, g->pdf_of[j]) + lse_list(scratch, deg);
        }
    }
    const double *last = alpha + (long)(N - 1) * K;
    for (int k = 0; k < K; ++k) scratch[k] = last[k] + (double)g->log_final[k];
    return lse_list(scratch, K);
}

/* Backward, P:89-90 / P:179-181 with v_{n+1} (ledger L2): beta[N][K]. Returns logZ_β. */
static double backward_seq(const graph_t *g, const double *emis_b, long D, int N, double *beta,
                           double *scratch) {
    int K = g->K;
    double *last = beta + (long)(N - 1) * K;
    for (int k = 0; k < K; ++k) last[k] = (double)g->log_final[k];
    for (int n = N - 2; n >= 0; --n) {
        const double *next = beta + (long)(n + 1) * K;
        double *cur = beta + (long)n * K;
        for (int i = 0; i < K; ++i) {
            long deg = 0;
            for (int a = g->row_ptr[i]; a < g->row_ptr[i + 1]; ++a) {
                int j = g->col[a] - g->off;
                scratch[deg++] = (double)g->logw[a] + emis_at(emis_b, D, n + 1, g->pdf_of[j]) + next[j];
            }
            cur[i] = lse_list(scratch, deg);
        }
    }
    for (int k = 0; k < K; ++k)
        scratch[k] = (double)g->log_init[k] + emis_at(emis_b, D, 0, g->pdf_of[k]) + beta[k];
    return lse_list(scratch, K);
}

enum { ST_OK = 0, ST_EMPTY = 1, ST_NONFINITE = 2, ST_BADLEN = 4 };

/* Per-sequence full forward-backward.  Outputs (any may be NULL):
 *   alpha, beta    [N_max][K]  true log α, β (−∞ for n ≥ N)
 *   post           [N_max][K]  γ (0 for n ≥ N)
 *   post_pdf       [N_max][D]  Γ (0 for n ≥ N)
 * Returns status bits; *logZ, *logZ_b, *gap filled. */
static int fb_seq(const graph_t *g, const double *emis_b, long D, int N, int N_max, double *alpha,
                  double *beta, double *post, double *post_pdf, double *logZ, double *logZ_b,
                  double *gap) {
    int K = g->K;
    long KN = (long)K * N_max;
    if (alpha) for (long x = 0; x < KN; ++x) alpha[x] = NEG_INF;
    if (beta) for (long x = 0; x < KN; ++x) beta[x] = NEG_INF;
    if (post) memset(post, 0, sizeof(double) * KN);
    if (post_pdf) memset(post_pdf, 0, sizeof(double) * (long)D * N_max);
    *logZ = NEG_INF; *logZ_b = NEG_INF; *gap = 0.0;
    if (N < 1 || N > N_max) return ST_BADLEN;
    if (nonfinite_inputs(g, emis_b, D, N)) return ST_NONFINITE;

    long maxdeg = K;
    for (int i = 0; i < K; ++i) {
        long d = g->row_ptr[i + 1] - g->row_ptr[i];
        if (d > maxdeg) maxdeg = d;
    }
    inarcs_t in = build_inarcs(g);
    for (int j = 0; j < K; ++j) {
        long d = in.ptr[j + 1] - in.ptr[j];
        if (d > maxdeg) maxdeg = d;
    }
    double *scratch = (double *)malloc(sizeof(double) * (size_t)(maxdeg + 1));
    double *A = (double *)malloc(sizeof(double) * (size_t)K * N);
    double *Bt = (double *)malloc(sizeof(double) * (size_t)K * N);
    double z = forward_seq(g, &in, emis_b, D, N, A, scratch);
    double zb = backward_seq(g, emis_b, D, N, Bt, scratch);
    *logZ = z; *logZ_b = zb;
    int st = ST_OK;
    if (z == NEG_INF) st = ST_EMPTY;
    if (alpha) memcpy(alpha, A, sizeof(double) * (size_t)K * N);
    if (beta) memcpy(beta, Bt, sizeof(double) * (size_t)K * N);
    if (st == ST_OK) {
        double gmax = 0.0;
        for (int n = 0; n < N; ++n) {
            for (int k = 0; k < K; ++k) scratch[k] = A[(long)n * K + k] + Bt[(long)n * K + k];
            double zn = lse_list(scratch, K);
            double d = fabs(zn - z);
            if (d > gmax) gmax = d;
            for (int k = 0; k < K; ++k) {
                double gk = exp(A[(long)n * K + k] + Bt[(long)n * K + k] - z); /* exp(−∞) = 0 exactly */
                if (post) post[(long)n * K + k] = gk;
                if (post_pdf) post_pdf[(long)n * D + g->pdf_of[k]] += gk; /* ascending k */
            }
        }
        *gap = gmax;
    } else {
        *logZ = NEG_INF;
    }
    free(scratch); free(A); free(Bt); free_inarcs(&in);
    return st;
}

static long packed_offset(int G, const int *state_offsets, int b, int N_max, int K0) {
    if (G == 1) return (long)b * N_max * K0;
    return (long)N_max * state_offsets[b];
}

/*
 * Batched forward-backward, one sequence at a time (OpenMP across
 * sequences only).  Layouts follow include/fb.h: G == 1 → [B][N_max][K];
 * G == B → packed, sequence b at N_max * state_offsets[b].
 * Any output pointer may be NULL.  Returns 0, or -1 on bad arguments.
 */
int oracle_fb_batch(int G, const int *state_offsets, const int *row_ptr, const int *col,
                    const float *logw, const float *log_init, const float *log_final,
                    const int *pdf_of, int D, const double *emis, const int *lengths, int B,
                    int N_max, double *alpha, double *beta, double *post, double *post_pdf,
                    double *logZ, double *logZ_beta, double *gap, int *status) {
    if (!(G == 1 || G == B) || B < 1 || N_max < 1 || D < 1) return -1;
    int K0 = state_offsets[1] - state_offsets[0];
#pragma omp parallel for schedule(dynamic, 1)
    for (int b = 0; b < B; ++b) {
        graph_t g = member(G, state_offsets, row_ptr, col, logw, log_init, log_final, pdf_of, b);
        long off = packed_offset(G, state_offsets, b, N_max, K0);
        double z, zb, gp;
        int st = fb_seq(&g, emis + (long)b * N_max * D, D, lengths[b], N_max,
                        alpha ? alpha + off : NULL, beta ? beta + off : NULL,
                        post ? post + off : NULL, post_pdf ? post_pdf + (long)b * N_max * D : NULL,
                        &z, &zb, &gp);
        if (logZ) logZ[b] = z;
        if (logZ_beta) logZ_beta[b] = zb;
        if (gap) gap[b] = gp;
        if (status) status[b] = st;
    }
    return 0;
}

/*
 * LF-MMI loss and gradient: per sequence b,
 *   loss_b = logZ_num,b − logZ_den,b,   grad[b,n,d] = Γ_num,n(d) − Γ_den,n(d)
 * for n < N_b; padded frames 0 (ledger L17).  Flagged sequences (empty num or
 * den lattice, non-finite input, bad length) get loss 0, grad 0 and are
 * excluded from totals = {Σ loss, Σ N_b, Σ logZ_num, Σ logZ_den, n_bad}
 * summed in ascending b (ledger L10).
 */
int oracle_lfmmi_batch(const int *num_offsets, const int *num_row_ptr, const int *num_col,
                       const float *num_logw, const float *num_init, const float *num_final,
                       const int *num_pdf, const int *den_offsets, const int *den_row_ptr,
                       const int *den_col, const float *den_logw, const float *den_init,
                       const float *den_final, const int *den_pdf, int D, const double *emis,
                       const int *lengths, int B, int N_max, double *grad, double *loss,
                       double *logZ_num, double *logZ_den, int *status, double *totals) {
    if (B < 1 || N_max < 1 || D < 1) return -1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int b = 0; b < B; ++b) {
        graph_t gn = member(B, num_offsets, num_row_ptr, num_col, num_logw, num_init, num_final, num_pdf, b);
        graph_t gd = member(1, den_offsets, den_row_ptr, den_col, den_logw, den_init, den_final, den_pdf, b);
        const double *eb = emis + (long)b * N_max * D;
        double *Gn = (double *)calloc((size_t)N_max * D, sizeof(double));
        double *Gd = (double *)calloc((size_t)N_max * D, sizeof(double));
        double zn, zd, zb, gp;
        int sn = fb_seq(&gn, eb, D, lengths[b], N_max, NULL, NULL, NULL, Gn, &zn, &zb, &gp);
        int sd = fb_seq(&gd, eb, D, lengths[b], N_max, NULL, NULL, NULL, Gd, &zd, &zb, &gp);
        int st = sn | sd;
        double *gb = grad + (long)b * N_max * D;
        if (st == ST_OK) {
            for (long x = 0; x < (long)N_max * D; ++x) gb[x] = Gn[x] - Gd[x];
            loss[b] = zn - zd;
        } else {
            memset(gb, 0, sizeof(double) * (size_t)N_max * D);
            loss[b] = 0.0;
        }
        if (logZ_num) logZ_num[b] = (st == ST_OK) ? zn : NEG_INF;
        if (logZ_den) logZ_den[b] = (st == ST_OK) ? zd : NEG_INF;
        status[b] = st;
        free(Gn); free(Gd);
    }
    if (totals) {
        double t[5] = {0, 0, 0, 0, 0};
        for (int b = 0; b < B; ++b) {
            if (status[b] == ST_OK) {
                t[0] += loss[b];
                t[1] += (double)lengths[b];
                t[2] += logZ_num[b];
                t[3] += logZ_den[b];
            } else {
                t[4] += 1.0;
            }
        }
        memcpy(totals, t, sizeof t);
    }
    return 0;
}

/*
 * Viterbi (the tropical semiring, ⊕ = max): the best path score
 * max over paths of π ⊗ Π v ⊗ Π T ⊗ ω and its state sequence, ties broken by
 * the lowest state index at every argmax (SPEC S:418 reading).  path[N_max]
 * gets −1 beyond N.  Returns status bits per sequence.
 */
static int viterbi_seq(const graph_t *g, const double *emis_b, long D, int N, int N_max,
                       double *score, int *path) {
    int K = g->K;
    for (int n = 0; n < N_max; ++n) path[n] = -1;
    *score = NEG_INF;
    if (N < 1 || N > N_max) return ST_BADLEN;
    if (nonfinite_inputs(g, emis_b, D, N)) return ST_NONFINITE;
    inarcs_t in = build_inarcs(g);
    double *A = (double *)malloc(sizeof(double) * (size_t)K * N);
    int *bp = (int *)malloc(sizeof(int) * (size_t)K * N);
    for (int k = 0; k < K; ++k) {
        A[k] = (double)g->log_init[k] + emis_at(emis_b, D, 0, g->pdf_of[k]);
        bp[k] = -1;
    }
    for (int n = 1; n < N; ++n) {
        for (int j = 0; j < K; ++j) {
            double best = NEG_INF;
            int arg = -1;
            for (int a = in.ptr[j]; a < in.ptr[j + 1]; ++a) {
                double x = A[(long)(n - 1) * K + in.src[a]] + in.w[a];
                if (x > best) { /* in-arcs ascend by source: first max = lowest index */
                    best = x;
                    arg = in.src[a];
                }
            }
            A[(long)n * K + j] = (best == NEG_INF) ? NEG_INF : best + emis_at(emis_b, D, n, g->pdf_of[j]);
            bp[(long)n * K + j] = (best == NEG_INF) ? -1 : arg;
        }
    }
    double best = NEG_INF;
    int arg = -1;
    for (int k = 0; k < K; ++k) {
        double x = A[(long)(N - 1) * K + k] + (double)g->log_final[k];
        if (x > best) { best = x; arg = k; }
    }
    int st = ST_OK;
    if (best == NEG_INF) {
        st = ST_EMPTY;
    } else {
        *score = best;
        int s = arg;
        for (int n = N - 1; n >= 0; --n) {
            path[n] = s;
            s = bp[(long)n * K + s];
        }
    }
    free(A); free(bp); free_inarcs(&in);
    return st;
}

int oracle_viterbi_batch(int G, const int *state_offsets, const int *row_ptr, const int *col,
                         const float *logw, const float *log_init, const float *log_final,
                         const int *pdf_of, int D, const double *emis, const int *lengths, int B,
                         int N_max, double *score, int *path, int *status) {
    if (!(G == 1 || G == B) || B < 1 || N_max < 1 || D < 1) return -1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int b = 0; b < B; ++b) {
        graph_t g = member(G, state_offsets, row_ptr, col, logw, log_init, log_final, pdf_of, b);
        status[b] = viterbi_seq(&g, emis + (long)b * N_max * D, D, lengths[b], N_max, &score[b],
                                path + (long)b * N_max);
    }
    return 0;
}
