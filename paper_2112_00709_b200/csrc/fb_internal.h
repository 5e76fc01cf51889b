// fb_internal.h — device-side graph handle and kernel argument blocks shared by
// fb_graph.cpp (host preprocessing) and fb_kernels.cu (kernels + entry points).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/fb.h"

namespace fbx {

constexpr int kMaxSPT = 8;          // states per thread held in registers
constexpr int kMaxThreads = 1024;   // threads per CTA (one CTA per sequence)
constexpr int kSmemLimit = 227 * 1024;

enum Mode : int { MODE_FACTORED = 0, MODE_EXACT = 1,
                  MODE_RAW = 2,       // exact arithmetic, float64 lattices, no per-frame normalisation (lfmmi numerator)
                  MODE_VITERBI = 3 }; // schedule encoding of the tropical pass: natural-log weights, float64 gathers

// One direction's arc schedule in grouped sliced-ELL form (forward = in-arcs /
// CSC of T, backward = out-arcs / CSR; ledger L3).  A row (the state being
// produced) with d arcs gets g = the smallest power of two with ⌈d/g⌉ ≤ Lmax
// lanes; rows of equal g, sorted by ⌈d/g⌉, form slices of 32/g rows (one lane
// per row segment).  The g partial sums of a row are combined inside the slice
// by a uniform xor-shuffle, so every state receives exactly one value.  Slices
// are packed onto warps longest-first; every lane of a warp executes the same
// instruction stream with no per-arc control flow.
//
// Byte layout of one slice with L arcs per lane (L even, null-padded):
//   header  int32[32]        lane l: (row+1 if l leads a row else 0) | log2(g) << 16 | (L/2) << 19
//   index   uint32[L/2][32]  two u16 byte offsets of the other endpoints in the
//                            gathered array (p in factored mode, u in exact mode);
//                            slot 2i in the low half, 2i+1 in the high half
//   weight  float2[L/2][32]  e^{T} (factored) or T·log2(e) (exact) for slots 2i, 2i+1
// Member g's blob starts at byte rec_off[g] (rec_bytes[g] bytes); warp w's
// slices start at byte warp_off[g*W+w] of the blob, warp_nsl[g*W+w] of them.
struct Sched {
    const unsigned char *rec = nullptr;
    const int *rec_bytes = nullptr;     // [G]
    const long long *rec_off = nullptr; // [G]
    const int *warp_off = nullptr;      // [G*W]
    const int *warp_nsl = nullptr;      // [G*W]
    const int *warp_nsl0 = nullptr;     // [G*W] how many of them (first) have g = 1 (one-CTA schedules)
    int bytes_max = 0;                  // max rec_bytes
    int slots_max = 0;                  // max arc slots of one warp
};

// Inverse pdf map of each member: slots = distinct pdfs used by the graph, in
// ascending pdf order.  Member g: slots [slot_off[g], slot_off[g+1]); slot s is
// pdf slot_pdf[s] carried by states slot_states[slot_sptr[s] .. slot_sptr[s+1])
// (local ids, ascending).  pdf_slot[g*D + d] = local slot index or -1.
struct PdfMap {
    const int *slot_off = nullptr;
    const int *slot_pdf = nullptr;
    const int *slot_sptr = nullptr;
    const int *slot_states = nullptr;
    const int *pdf_slot = nullptr;
    const int *slot_pos = nullptr;    // [K_tot] position of a state in its member's slot-ordered list
    int U_max = 0;
    long long U_tot = 0;
    int spp_max = 0;                  // most states sharing one pdf in a member
};

// Cluster plan of a shared (G == 1) factored graph for k_fbc: a thread-block
// cluster of C CTAs runs S sequences in lockstep.  The K states are split into
// C parts along ascending pdf ranges (every state of a pdf lives in one part, so
// pdf-level posterior rows are part-local); part c owns the contiguous
// internal states [part_off[c], part_off[c+1]) (each part padded to a multiple
// of 4 with inert states) and computes their rows for all S sequences, reading
// the gathered vector p = 2^u of every state from its own shared memory.  After
// each frame a CTA ships its rows of u to the other C−1 CTAs with bulk
// shared→shared copies (DSMEM) that complete on the receivers' mbarriers.
// Schedules are the grouped sliced-ELL of Sched with S-float gathered elements
// (member c = part c's rows); index words are byte offsets into p[K_int][S].
struct CPlan {
    int ok = 0, C = 0, S = 0, T = 0, spt = 0, K_int = 0, Kc_max = 0, Dc_max = 0;
    int nop = 0;                        // no p = 2^u array: phase A applies ex2 to the gathered u (smem-bound configs)
    int split = 0;                      // bit 0 forward, bit 1 backward: members 2c / 2c+1 = part c's local-source /
                                        // remote-source arcs (phase A split around the exchange wait); else member
                                        // c = all of part c's arcs
    int emis16 = 0;                     // emission segments are 16-byte aligned (D % 4 == 0)
    const int *part_off = nullptr;      // [C+1] internal state offsets
    const int *pdf_lo = nullptr;        // [C+1] part c owns pdfs [pdf_lo[c], pdf_lo[c+1])
    const int *perm = nullptr;          // [K_int] original state id (−1: padding)
    const int *ipdf = nullptr;          // [K_int] pdf (0 for padding)
    const int *idist_fin = nullptr;     // [K_int] as Graph::dist_fin (kFar for padding)
    const int *idist_start = nullptr;   // [K_int]
    const float *iinit2 = nullptr;      // [K_int] π·log2(e) (−∞ for padding)
    const float *ifinal2 = nullptr;     // [K_int] ω·log2(e)
    const unsigned *pq = nullptr;       // [D] first local position of the pdf's states | count << 16
    Sched fwd, bwd;                     // member c: part c's rows (in-arcs / out-arcs)
    // exact fallback rows (internal ids, log2 weights): forward in-arcs, backward out-arcs
    const int *fptr = nullptr, *fsrc = nullptr, *bptr = nullptr, *bsrc = nullptr;
    const float *fw2 = nullptr, *bw2 = nullptr;
};

#ifdef __CUDACC__
#define FBX_HD2 __host__ __device__
#else
#define FBX_HD2
#endif
// The paper's literal batch matrix (fb_literal.cu): per member, the in-arc
// lists of its K_g states plus a phony state K_g (arcs s → phony weighted ω(s),
// a 1̄ self-loop; ledger L8).  Instance b (sequence b) owns rows
// [inst_off(b), inst_off(b) + K_b + 1) of the batch vector.
struct LitPlan {
    const int *row_off = nullptr;   // [G] member g's first row in ptr
    const int *ptr = nullptr;       // [Σ_g (K_g + 1) + 1]
    const int *src = nullptr;       // local source ids (K_g = the phony state)
    const double *w = nullptr;      // natural-log weights (ω for phony arcs, 0 for its self-loop)
    const int *inst_off = nullptr;  // G == B: [B + 1] = state_off[b] + b
    const int *optr = nullptr;      // out-arc lists of the same rows (backward pass): [Σ_g (K_g + 1) + 1]
    const int *odst = nullptr;      // local destination ids (K_g = the phony state)
    const double *ow = nullptr;     // natural-log weights (ω for arcs into phony, 0 for its self-loop)
    int g1 = 1, K1 = 0;             // G == 1: every instance has K + 1 rows
    long long inst_total = 0;       // G == B: Σ_b (K_b + 1)
    FBX_HD2 long long rows_per_batch(int B) const { return g1 ? (long long)B * K1 : inst_total; }
#ifdef __CUDACC__
    __device__ void locate(long long r, int B, int &b, int &j) const {
        if (g1) { b = (int)(r / K1); j = (int)(r - (long long)b * K1); return; }
        int lo = 0, hi = B;  // largest b with inst_off[b] <= r
        while (hi - lo > 1) { const int m = (lo + hi) >> 1; if (inst_off[m] <= r) lo = m; else hi = m; }
        b = lo; j = (int)(r - inst_off[lo]);
    }
#endif
};

struct Graph {
    int G = 0, K_tot = 0, D = 0, T = 0, W = 0, spt = 1, mode = 0;
    int mask_fwd = 0, mask_bwd = 0;  // any state ever masked by the viability distances
    long long nnz = 0;
    int K_max = 0;
    long long nnz_max = 0;
    // device arrays (all inside one allocation `block`)
    const int *state_off = nullptr;   // [G+1]
    const int *pdf = nullptr;         // [K_tot]
    const float *init2 = nullptr;     // [K_tot] π · log2(e)
    const float *final2 = nullptr;    // [K_tot] ω · log2(e)
    const float *init_nat = nullptr;  // [K_tot] π (natural log, as given)
    const float *final_nat = nullptr; // [K_tot] ω (natural log, as given)
    const int *dist_fin = nullptr;    // [K_tot] min #transitions to a final state (INT_MAX/2 if none)
    const int *dist_start = nullptr;  // [K_tot] min #transitions from an initial state
    const int *morder = nullptr;      // [G] members by descending arc count (persistent CTAs take the heavy ones first)
    Sched fwd, bwd;
    Sched vit;        // forward (in-arc) schedule with natural-log weights for fb_viterbi
    int vit_ok = 0;   // the Viterbi schedule was built (K ≤ 8192: 16-bit byte offsets into float64 u)
    int vit_global = 0; // ... but does not fit shared memory: k_viterbi streams it from global memory (L2)
    PdfMap pm;
    CPlan cp;         // cluster plan (k_fbc); cp.ok == 0: one CTA per sequence (k_fb)
    LitPlan lit;      // the paper's literal block-diagonal strategy (fb_literal.cu, N4)
    int legacy_ok = 1; // the one-CTA-per-sequence kernels fit (else only the cluster path runs)
    // diagnostic counters in the handle's device block (the only mutable device state of a
    // handle; atomics): [0] rows of the exp-factorised ⊕ that took the exact max-then-sum
    // fallback (k_fb, per row evaluation), [1] the same in the cluster kernel k_fbc (per
    // sequence-row).  Read / reset by fb_graph_counters.
    unsigned long long *ctr = nullptr;
    void *block = nullptr;
    size_t block_bytes = 0;
    bool dry = false;
    int device = 0;
};

#ifdef __CUDACC__
#define FBX_HD __host__ __device__
#else
#define FBX_HD
#endif

// Shared-memory carve-up of one forward/backward CTA (host and device agree):
// arc records | u (log2 values, V) | p = 2^u (factored) | segment partials (V)
// | γ row (pdf-level epilogue) | reductions + flags.
struct SmemLayout {
    size_t rec, u, p, part, gbuf, red, total;
};
FBX_HD inline size_t fbx_a16(size_t x) { return (x + 15) & ~size_t(15); }
// Per-state arrays hold K_pad = threads × states-per-thread entries.
FBX_HD inline SmemLayout smem_layout(int rec_bytes, int K_pad, bool exact, bool gbuf) {
    const size_t vsz = exact ? 8 : 4;
    SmemLayout L;
    size_t o = 0;
    L.rec = o; o += fbx_a16((size_t)rec_bytes);
    L.u = o; o += fbx_a16((size_t)K_pad * vsz);
    L.p = o; if (!exact) o += fbx_a16((size_t)K_pad * 4);
    L.part = o + 16; o += 16 + fbx_a16((size_t)K_pad * vsz);  // part[-1]: scratch cell of non-leader lanes
    L.gbuf = o; if (gbuf) o += fbx_a16((size_t)K_pad * 4);
    L.red = o; o += fbx_a16(8 * (2 * 32 + 2 * 64) + 64);
    L.total = o;
    return L;
}

// Output kinds of the backward posterior epilogue.
enum PostKind : int { POST_NONE = 0, POST_STATE = 1, POST_PDF_DENSE = 2, POST_PDF_COMPACT = 3, POST_GRAD = 4 };

// Shared-memory region of the pdf-level epilogue, placed after the reductions:
// ssp u16[U+1]  slot boundaries of the member's slot-ordered state list  (compact)
// pq  u32[D]    pdf → q0 | count << 16: its states' run in the slot-ordered
//               γ row (count 0: pdf unused)                          (dense / grad)
struct PdfRegion {
    size_t ssp, pq, bytes;
};
FBX_HD inline PdfRegion pdf_region(int kind, int U_max, int D) {
    PdfRegion R;
    size_t o = 0;
    R.ssp = o; if (kind == POST_PDF_COMPACT) o += fbx_a16((size_t)(U_max + 1) * 2);
    R.pq = o; if (kind == POST_PDF_DENSE || kind == POST_GRAD) o += fbx_a16((size_t)D * 4);
    R.bytes = (kind == POST_PDF_DENSE || kind == POST_PDF_COMPACT || kind == POST_GRAD) ? o : 0;
    return R;
}

// Shared-memory carve-up of one k_fbc CTA (host and device agree):
// rec (part schedule) | u[2] (per buffer: K_int·S floats, then C extras slots of
// S × 8 floats) | p (K_int·S) | part (Kc_max·S) | gbuf (Kc_max·S, pdf-level
// posteriors) | pq (Dc_max, pdf-level) | ebuf[2][S][Dc_max] emission segments
// | red (per warp × seq × 8 floats, + frame-0 and termination slots) | mbar[2].
constexpr int kCX = 8;  // floats per (part, sequence) extras slot
struct CLayout {
    size_t rec, u, ubytes, p, part, gbuf, xbuf, pq, ebuf, red, mbar, total;
};
FBX_HD inline CLayout cl_layout(int rec_bytes, int K_int, int Kc_max, int Dc_max, int S, int C, int W, bool pdfpost,
                                bool nop = false) {
    CLayout L;
    size_t o = 0;
    L.rec = o; o += fbx_a16((size_t)rec_bytes);
    L.ubytes = (size_t)K_int * S * 4 + (size_t)C * S * kCX * 4;
    L.u = o; o += 2 * fbx_a16(L.ubytes);
    L.p = o; if (!nop) o += fbx_a16((size_t)K_int * S * 4);  // nop: phase A exponentiates u on the fly
    L.part = o; o += fbx_a16((size_t)Kc_max * S * 4);
    L.gbuf = o; if (pdfpost && !nop) o += fbx_a16((size_t)Kc_max * S * 4);
    L.xbuf = o; if (pdfpost) o += fbx_a16((size_t)Kc_max * S * 4);  // nop: γ overwrites x in place (gbuf = xbuf)
    L.pq = o; if (pdfpost) o += fbx_a16((size_t)Dc_max * 4);
    L.ebuf = o; o += 2 * fbx_a16((size_t)S * Dc_max * 4);
    L.red = o; o += fbx_a16((size_t)(W + 2) * S * kCX * 4);
    L.mbar = o; o += 16;
    L.total = o;
    return L;
}

// Dynamic shared memory needed by a forward/backward launch over this graph.
size_t smem_bytes(const Graph &g, bool backward, bool pdf_level);
// ... and by a Viterbi launch (float64 u / best, int32 arg per state).
size_t viterbi_smem_bytes(const Graph &g, bool global_sched = false);

}  // namespace fbx

struct fb_graph_s {
    fbx::Graph g;
    // Shared factored graphs: the same graph with its states relabelled so that the
    // shared-memory gathers, part-row stores and emission gathers of the one-CTA
    // kernels hit distinct banks (fb_graph.cpp, bank_relabel).  lfmmi_loss_grad runs
    // its denominator passes on it (their α̂ lattice is private and the gradient is
    // pdf-level, so the labelling is invisible); the public lattice calls use g.
    fb_graph_s *perm = nullptr;
    // dry-run handles keep the host image of the compiled schedules for inspection
    std::vector<unsigned char> host_fwd, host_bwd;
    std::vector<int> host_fwd_meta, host_bwd_meta;  // per member: rec_off, rec_bytes; then W × (warp_off, warp_nsl)
};

namespace fbx {
void set_cuda_error(const char *what, int code);
}
