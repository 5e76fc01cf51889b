/*
 * fb.h — C ABI of libfb: batched log-semiring forward-backward and the LF-MMI
 * gradient on NVIDIA B200 (sm_100a).
 *
 * The method is arXiv 2112.00709 (/root/reference/PAPER.md, cited P:<line>):
 * the forward-backward recursions written as sparse matrix-vector products in
 * the log semifield 𝒮(ℝ, ⊕, ⊗, ⊘, 0̄, 1̄), batched over
 * variable-length sequences, and the LF-MMI loss/gradient built on
 * them.  Readings of ambiguous passages (ledger L1-L19) are listed
 * in DESIGN.md; the ones that fix this interface are repeated next to each call.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  • Pointers are DEVICE pointers unless marked [host].  The caller allocates
 *    and owns every buffer; the library owns only the fb_graph handle.
 *  • `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every compute call is asynchronous on `stream`, never synchronizes the
 *    host and never allocates device memory.
 *  • Synchronous errors: a non-zero fb_status is returned for host-checkable
 *    problems (null pointers, non-positive sizes, G ∉ {1, B}, numerator /
 *    denominator D mismatch, workspace too small, unsupported graph sizes);
 *    nothing is enqueued then.  The emission width is not an argument: log_emis
 *    must have exactly the D columns the graph was created with, and buffers
 *    must have the sizes stated per call — the library cannot check either
 *    (the Python binding does, and raises ValueError).
 *  • Threading: entry points are re-entrant; handles are immutable (except the
 *    diagnostic counters, see fb_graph_counters) and may be used from several
 *    host threads and streams at once.
 *  • Asynchronous, data-dependent problems never abort a batch: they set
 *    per-sequence bits in seq_status[b] (FB_SEQ_*): empty lattice (logZ = 0̄),
 *    NaN or +∞ in an emission the recursion reads (−∞ is a legal 0̄), and
 *    N_b ∉ [1, N_max].  Per graph at most one bit is set, in this precedence:
 *    BAD_LENGTH, else NONFINITE_INPUT, else EMPTY_LATTICE (lfmmi_loss_grad ORs
 *    the numerator's and the denominator's bits).  Flagged sequences get logZ = −∞; their lattice contents
 *    are unspecified; their posterior / gradient rows are written as 0 and they
 *    are excluded from lfmmi totals.
 *  • Units: every log quantity crossing this boundary is a natural log.
 *  • Determinism: outputs are bitwise reproducible for identical inputs and are
 *    independent of batch composition and order (one CTA per sequence, fixed
 *    reduction trees, no floating-point atomics).
 *  • Layout of per-state lattices (alpha, beta, state-level post):
 *      G == 1 (one shared graph of K states):  [B][N_max][K]
 *      G == B (graph b per sequence b):        packed; sequence b occupies
 *          [N_max][K_b] starting at element N_max * state_offsets[b].
 *    Frames n ≥ N_b: alpha/beta = −∞, post = 0.
 *  • Normalised lattices: alpha holds α̂ with α_true[b,n,k] = alpha[b,n,k] +
 *    alpha_scale[b,n] (scale in float64); likewise beta / beta_scale.  Each
 *    frame is shifted so that its largest viable entry is 0.
 *
 * Status codes of asynchronous kernels are only meaningful after the stream
 * has been synchronised by the caller.
 */
#ifndef FB_H
#define FB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FB_OK = 0,
    FB_ERR_INVALID_ARG = 1,   /* null pointer, non-positive size, G ∉ {1, B}, D mismatch */
    FB_ERR_SHAPE = 2,         /* buffer/graph shapes inconsistent */
    FB_ERR_INVALID_GRAPH = 3, /* bad CSR, arc outside its block, pdf out of range, NaN/+∞ weight */
    FB_ERR_CUDA = 4,          /* a CUDA runtime call failed (see fb_last_cuda_error) */
    FB_ERR_NOMEM = 5,         /* device allocation failed in fb_graph_create */
    FB_ERR_WORKSPACE = 6,     /* workspace NULL or smaller than fb_workspace_bytes */
    FB_ERR_UNSUPPORTED = 7    /* graph exceeds this build's on-chip limits */
} fb_status;

enum {
    FB_SEQ_OK = 0,
    FB_SEQ_EMPTY_LATTICE = 1,   /* no accepting path: logZ = 0̄ */
    FB_SEQ_NONFINITE_INPUT = 2, /* NaN or +∞ among the emissions read */
    FB_SEQ_BAD_LENGTH = 4       /* N_b < 1 or N_b > N_max */
};

/* fb_graph_create flags */
enum {
    FB_GRAPH_DEFAULT = 0,
    FB_GRAPH_FORCE_EXACT = 1,    /* every ⊕ row evaluated max-then-sum (one exp per arc) */
    FB_GRAPH_FORCE_FACTORED = 2, /* exp-factorised ⊕ with exact fallback */
    FB_GRAPH_CLUSTER = 4,        /* shared (G = 1) factored graphs: run the cluster-batched kernel
                                    (C CTAs × S sequences per thread-block cluster) even when one
                                    sequence's schedule fits one SM; graphs that do not fit one SM
                                    (e.g. the paper's 50,984-arc denominator) always use it */
    FB_GRAPH_DRY_RUN = 256       /* run the host compiler only: no device allocation; the handle
                                    supports fb_graph_info/destroy, compute calls reject it */
};

typedef struct fb_graph_s *fb_graph; /* opaque, immutable after create */

/*
 * fb_graph_create — compile G weighted automata (T, π, ω) into a device handle.
 *
 * Paper: T is the K×K transition matrix with row = previous state
 * (ledger L3), stored sparse with absent entries meaning 0̄ = −∞
 * (P:136-137).  Batches are the block-diagonal
 * composition diag(T_1 … T_G).  π (initial) and ω (final) weights
 * generalise the paper's start condition and Eq. (1) normaliser (ledger L4, L6).
 *
 *   G                 number of member graphs (1 = shared denominator graph,
 *                     B = one numerator graph per sequence).
 *   state_offsets     [host][G+1] graph g owns global states
 *                     [state_offsets[g], state_offsets[g+1]); strictly increasing, [0] = 0.
 *   row_ptr, col,     [host] CSR over the K_tot = state_offsets[G] global states:
 *   log_w             arcs row_ptr[i]..row_ptr[i+1]-1 leave state i for col[a] with
 *                     natural-log weight log_w[a] (−∞ allowed; NaN/+∞ rejected).
 *                     Every arc must stay inside its member's block.  Duplicate
 *                     arcs are ⊕-combined.
 *   log_init, log_final [host][K_tot] π and ω (natural log, −∞ allowed).
 *   pdf_of            [host][K_tot] emission column of each state (ledger L9),
 *                     each in [0, D); NULL = identity (requires every K_g ≤ D).
 *   D                 number of emission columns of log_emis.
 *   flags             FB_GRAPH_* (0 = choose the ⊕ evaluation per member graph).
 *
 * All preprocessing (CSC for the forward pull, CSR for the backward pull,
 * nnz-balanced per-thread arc schedules, BFS viability distances, inverse pdf
 * maps) runs on the host; the result is uploaded once.  The call is
 * synchronous; the handle must outlive all work enqueued with it.
 * Returns FB_ERR_UNSUPPORTED if a member graph exceeds K_g > 8192 states or its
 * schedule does not fit 227 KB of shared memory.
 */
fb_status fb_graph_create(fb_graph *out, int32_t G, const int32_t *state_offsets, const int32_t *row_ptr,
                          const int32_t *col, const float *log_w, const float *log_init,
                          const float *log_final, const int32_t *pdf_of, int32_t D, int32_t flags);

/* Frees the handle's device memory (synchronizes the device first). NULL is a no-op. */
fb_status fb_graph_destroy(fb_graph g);

/*
 * fb_graph_info — [host] out[16] int64: {G, K_tot, nnz, D, threads_per_cta,
 * states_per_thread, mode (0 factored / 1 exact / 2 mixed), fwd_smem_bytes,
 * bwd_smem_bytes, K_max, nnz_max, fwd_slots_max, bwd_slots_max, U_max,
 * cluster_C, cluster_S}: cluster_C > 0 when a shared factored graph runs the
 * cluster-batched kernel (C CTAs per cluster, S sequences per cluster).
 */
fb_status fb_graph_info(fb_graph g, int64_t *out);

/*
 * fb_graph_counters — [host] out[2] int64 diagnostic counters of the handle since
 * creation or the last reset: out[0] = row evaluations of the exp-factorised ⊕
 * that fell back to the exact max-then-sum because
 * the factored sum left [2^-80, 2^120] (one-CTA kernel, per row and frame), out[1] =
 * the same in the cluster kernel (per row, sequence and frame).  Rows of masked
 * (non-viable) states count too.  reset != 0 zeroes them afterwards.  Synchronous:
 * waits for all device work (cudaMemcpy).  The counters are the only device state
 * of a handle that kernels modify (atomic adds); they never influence results.
 */
fb_status fb_graph_counters(fb_graph g, int64_t *out, int32_t reset);

/*
 * fb_forward — Eq. (13), the log-domain form of Eq. (2)/(4)
 * with ledger L1 (sum over z_{n-1}) and L6
 * (α_0 = π ⊗ v_0):  α_n(j) = v_n(j) ⊗ ⊕_{i→j} α_{n-1}(i) ⊗ T_ij,
 * v_n(k) = log_emis[b, n, pdf_of[k]].  Termination:
 * logZ[b] = ⊕_k α_{N_b-1}(k) ⊗ ω(k).
 *
 *   log_emis    [B][N_max][D] float32, read-only.
 *   lengths     [B] int32 N_b.
 *   alpha       [lattice layout] float32 α̂ out (may be NULL).
 *   alpha_scale [B][N_max] float64 out (may be NULL only if alpha is NULL).
 *   logZ        [B] float64 out.
 *   seq_status  [B] int32 out (overwritten).
 */
fb_status fb_forward(fb_graph g, const float *log_emis, const int32_t *lengths, int32_t B, int32_t N_max,
                     float *alpha, double *alpha_scale, double *logZ, int32_t *seq_status, void *stream);

/*
 * fb_backward — Eq. (14) read with v_{n+1} as in Eq. (3)
 * (ledger L2) and β_{N_b-1} = ω (ledger L7):
 *   β_n(i) = ⊕_{i→j} T_ij ⊗ v_{n+1}(j) ⊗ β_{n+1}(j).
 * logZ_beta[b] = ⊕_k π(k) ⊗ v_0(k) ⊗ β_0(k) (equals logZ; a consistency check).
 *
 * Optional fused posterior epilogue (Eq. (15), read as semifield
 * division, ledger L5): if `post` is non-NULL, alpha must be fb_forward's
 * output and  post = exp(α̂_n + β̂_n − Z_n)  with the per-frame normaliser
 * Z_n = ⊕_k α̂_n(k) ⊗ β̂_n(k)  (= logZ − C_n − D_n by the α·β invariant, so
 * the result is Eq. (1) exactly).
 *   pdf_level = 0: post has the lattice layout (state posteriors γ);
 *   pdf_level = 1: post is [B][N_max][D], Γ_n(d) = Σ_{pdf_of[k]=d} γ_n(k).
 * seq_status is read (bits set by fb_forward are kept; flagged sequences get
 * zero posterior rows) and updated.  beta/beta_scale/logZ_beta may be NULL.
 */
fb_status fb_backward(fb_graph g, const float *log_emis, const int32_t *lengths, int32_t B, int32_t N_max,
                      float *beta, double *beta_scale, double *logZ_beta, const float *alpha,
                      float *post, int32_t pdf_level, int32_t *seq_status, void *stream);

/*
 * fb_posteriors — standalone Eq. (15)/(1): post = exp(α̂_n + β̂_n − Z_n) from
 * stored fb_forward / fb_backward lattices (scales cancel in the per-frame
 * normaliser, see fb_backward).  pdf_level as in fb_backward.  Sequences with
 * seq_status[b] != 0 or N_b ∉ [1, N_max] get zero rows.
 */
fb_status fb_posteriors(fb_graph g, const float *alpha, const float *beta, const int32_t *lengths,
                        const int32_t *seq_status, int32_t B, int32_t N_max, int32_t pdf_level,
                        float *post, void *stream);

/*
 * fb_gap — the Eq. (1) invariant as a per-sequence diagnostic (SURVEY
 * §8(a) S5 gap_n, §8(c3)): every frame's Σ_k α_n(k) β_n(k) is the same p(X):
 *   gap[b] = max_{n < N_b} | ⊕_k (α̂_n(k) ⊗ β̂_n(k)) + C_n + D_n − logZ[b] |
 * from fb_forward's (alpha, alpha_scale, logZ) and fb_backward's (beta,
 * beta_scale) of the same inputs; natural log, float64 combine.  A healthy run
 * has gap ≈ fp32 rounding of the lattices (≲ 1e-5·|logZ|); a frame whose α·β
 * sum is 0̄ gives +∞.  Sequences with seq_status[b] != 0 (seq_status may be
 * NULL), N_b ∉ [1, N_max] or logZ = 0̄ get gap = 0.
 *   gap         [B] float64 out.
 */
fb_status fb_gap(fb_graph g, const float *alpha, const double *alpha_scale, const float *beta,
                 const double *beta_scale, const double *logZ, const int32_t *lengths, const int32_t *seq_status,
                 int32_t B, int32_t N_max, double *gap, void *stream);

/*
 * fb_workspace_bytes — device workspace lfmmi_loss_grad needs for (num, den, B, N_max):
 * the α̂ lattices of both graphs, the denominator forward's per-frame offsets C_n,
 * both log Z vectors and the numerator pdf posteriors.
 */
size_t fb_workspace_bytes(fb_graph num, fb_graph den, int32_t B, int32_t N_max);

/*
 * lfmmi_loss_grad — LF-MMI objective and gradient:
 *   loss[b] = log p(X_b | G_num,b) − log p(X_b | G_den) = logZ_num − logZ_den
 *   grad[b,n,d] = ∂ℒ/∂φ_{n,d} = Γ_num,n(d) − Γ_den,n(d)
 * for n < N_b, 0 for padded frames (ledger L17).  ℒ is per utterance,
 * unnormalised, the ascent direction as printed (ledger L10).  Γ_den of frame n
 * is normalised through the forward's log Z (Eq. (1); ledger L22):
 * e_k = exp(α̂_n(k) + β̂_n(k) − (log Z − C_n − D_n)), Γ_den,n(d) = Σ_{pdf(k)=d} e_k / Σ_k e_k.
 * The numerator and denominator passes run concurrently (the numerator on the
 * SMs the denominator leaves idle); the call is ordered on `stream` as a whole.
 *
 *   num         G == B graph handle (one numerator graph per sequence).
 *   den         G == 1 graph handle (shared denominator graph); num->D == den->D.
 *   log_emis    [B][N_max][D] float32 network outputs φ.
 *   grad        [B][N_max][D] float32 out, written once.
 *   loss        [B] float64 out (0 for flagged sequences).
 *   totals      [5] float64 out: {Σ loss, Σ N_b, Σ logZ_num, Σ logZ_den, n_bad}
 *               over sequences with seq_status == 0, summed in ascending b.
 *   seq_status  [B] int32 out: OR of the numerator and denominator bits.
 *   workspace   device buffer of ≥ fb_workspace_bytes(num, den, B, N_max) bytes.
 */
fb_status lfmmi_loss_grad(fb_graph num, fb_graph den, const float *log_emis, const int32_t *lengths,
                          int32_t B, int32_t N_max, float *grad, double *loss, double *totals,
                          int32_t *seq_status, void *workspace, size_t workspace_bytes, void *stream);

/*
 * fb_viterbi — the tropical-semiring instance of Eq. (13) (⊕ = max):
 * score[b] = max over accepting paths of π ⊗ Π v ⊗ Π T ⊗ ω and path[b][n] its
 * state sequence (local state ids; −1 for n ≥ N_b), ties broken by the lowest
 * state index at every argmax.  workspace ≥ fb_viterbi_workspace_bytes(g, B, N_max)
 * holds the int16/int32 backpointer lattice.  One CTA per sequence; a schedule too
 * large for shared memory (e.g. the paper's 50,984-arc denominator) is streamed
 * from global memory (L2) each frame.  FB_ERR_UNSUPPORTED only for K_g > 8192.
 */
size_t fb_viterbi_workspace_bytes(fb_graph g, int32_t B, int32_t N_max);
fb_status fb_viterbi(fb_graph g, const float *log_emis, const int32_t *lengths, int32_t B, int32_t N_max,
                     double *score, int32_t *path, int32_t *seq_status, void *workspace,
                     size_t workspace_bytes, void *stream);

/*
 * fb_forward_literal — the paper's own execution strategy, generic in the
 * semiring: the batch is one
 * block-diagonal matrix (G == 1: B copies of the shared graph; G == B: graph b
 * for sequence b), each block augmented with a phony state (arcs s → phony
 * weighted ω(s), a 1̄ self-loop; emissions 0̄/1̄ past N_b, ledger L8), and
 * every frame is ONE sparse matrix-vector product x_n = v_n ⊗ Tᵀ x_{n−1}
 * (Eq. (13)) over the whole batch, one kernel launch per frame, N_max + 1
 * frames, float64, no normalisation.  score[b] = x_{N_max}(phony_b):
 *   FB_SEMIRING_LOG       log Z_b (natural log; equals fb_forward's logZ),
 *   FB_SEMIRING_TROPICAL  the best-path score (equals fb_viterbi's score),
 *   FB_SEMIRING_PROB      Z_b in the probability domain (exp of weights and
 *                         emissions; underflows to 0 on long inputs).
 * Sequences with N_b ∉ [1, N_max] get the semiring's 0̄.  A reference /
 * A/B baseline for the fused kernels, not a fast path.  workspace ≥
 * fb_literal_workspace_bytes(g, B) (two batch vectors).
 */
enum { FB_SEMIRING_LOG = 0, FB_SEMIRING_TROPICAL = 1, FB_SEMIRING_PROB = 2 };
size_t fb_literal_workspace_bytes(fb_graph g, int32_t B);
fb_status fb_forward_literal(fb_graph g, int32_t semiring, const float *log_emis, const int32_t *lengths,
                             int32_t B, int32_t N_max, double *score, void *workspace, size_t workspace_bytes,
                             void *stream);

/*
 * fb_forward_semiring — the fused one-CTA-per-sequence forward of Eq. (13)
 * instantiated for any of the three semirings (SURVEY
 * §8(f) N4): score[b] = ⊕ over accepting paths of π ⊗ Π v ⊗ Π T ⊗ ω, float64,
 * no normalisation — FB_SEMIRING_LOG: log Z_b (= fb_forward's logZ);
 * FB_SEMIRING_TROPICAL: the best-path score (= fb_viterbi's score);
 * FB_SEMIRING_PROB: Z_b in the linear domain (0 where it underflows, P:93-96;
 * the sequence is then flagged FB_SEQ_EMPTY_LATTICE like a true 0̄).  Same arc
 * schedule and per-frame phases as the tuned kernels; seq_status as fb_forward.
 * FB_ERR_UNSUPPORTED for member graphs over 8192 states.
 */
fb_status fb_forward_semiring(fb_graph g, int32_t semiring, const float *log_emis, const int32_t *lengths,
                              int32_t B, int32_t N_max, double *score, int32_t *seq_status, void *stream);

/*
 * fb_forward_backward_literal — the literal strategy's full forward-backward
 * (SURVEY §8(f) N4): fb_forward_literal's forward storing every frame's batch
 * vector X_n, then the backward of the same block-diagonal matrix, one SpMV per
 * frame over the augmented out-arc lists (Eq. (14) with v_{n+1}, ledger L2,
 * P:179-181; y_{N_max} = 1̄ on each phony state), writing the frame's
 * posteriors (Eq. (15), semifield division, ledger L5) in the same launch:
 *   post[b,n,k] = X_n(k) ⊗ y_n(k) ⊘ score[b]   for n < N_b, real states k; else 0,
 * with post in the lattice layout of fb_forward (may be NULL: score only), float64.
 *   FB_SEMIRING_LOG       γ = exp(x + y − log Z)  (the state posteriors of fb_backward)
 *   FB_SEMIRING_PROB      γ = x·y / Z             (linear domain; 0 where Z underflows)
 *   FB_SEMIRING_TROPICAL  exp(x + y − best) ∈ [0, 1], the max-marginal ratio: 1 on
 *                         the states of a best path (fb_viterbi's), < 1 elsewhere.
 * workspace ≥ fb_literal_fb_workspace_bytes(g, B, N_max) ((N_max + 3) batch vectors).
 */
size_t fb_literal_fb_workspace_bytes(fb_graph g, int32_t B, int32_t N_max);
fb_status fb_forward_backward_literal(fb_graph g, int32_t semiring, const float *log_emis, const int32_t *lengths,
                                      int32_t B, int32_t N_max, double *score, double *post, void *workspace,
                                      size_t workspace_bytes, void *stream);

/*
 * Kernel timing (tracing).  When enabled, every kernel the library launches is
 * bracketed by cudaEventRecord on the stream it is launched on.
 * fb_profile_collect synchronises those events and returns, per kernel name,
 * the number of launches and the summed device milliseconds since the last
 * reset: names[i] (static strings), counts[i], ms[i] for i < *n (≤ cap).
 */
void fb_profile_enable(int32_t on);
void fb_profile_reset(void);
fb_status fb_profile_collect(const char **names, int64_t *counts, double *ms, int32_t cap, int32_t *n);

/* Human-readable text for a status code / the last CUDA error string seen. */
const char *fb_status_str(fb_status s);
const char *fb_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FB_H */
