// fb_internal.h — device-side graph handle and kernel argument blocks shared by
// fb_graph.cpp (host preprocessing) and fb_kernels.cu (kernels + entry points).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

#include "../../include/fb.h"

namespace fbx {

constexpr int kMaxSPT = 8;          // states per thread held in registers
constexpr int kMaxThreads = 1024;   // threads per CTA (one CTA per sequence)
constexpr int kSmemLimit = 227 * 1024;

enum Mode : int { MODE_FACTORED = 0, MODE_EXACT = 1 };

// One direction's arc schedule in sliced-ELL form (forward = in-arcs / CSC of
// T, backward = out-arcs / CSR; ledger L3).  Rows are cut into segments of at
// most Lmax arcs; segments sorted by length are grouped 32 at a time into
// slices (one segment per lane, shorter ones padded with null arcs); slices
// are packed onto the W warps longest-first.  Every lane of a warp therefore
// executes the same number of slots with no per-arc control flow.
//   rec[r*32 + lane] = {byte offset of the other endpoint in the u / p arrays,
//                       weight: e^{T} (factored) or T·log2(e) (exact)}
//   member g: records start at rec_off[g]; warp w's slices are
//   sl_off[g] + warp_sl0[g*W+w] … + warp_nsl[g*W+w], its rows start at
//   warp_row[g*W+w]; slice q has sl_len[q] rows and lane l reduces into
//   segment sl_seg[q*32+l] (-1: idle lane).  Segments are numbered in row
//   order, so state j's segments are [segptr[j], segptr[j+1]).
struct Sched {
    const uint2 *rec = nullptr;
    const int *rec_rows = nullptr;      // [G]
    const long long *rec_off = nullptr; // [G]
    const int *warp_row = nullptr;      // [G*W]
    const int *warp_nsl = nullptr;      // [G*W]
    const int *warp_sl0 = nullptr;      // [G*W]
    const int *sl_off = nullptr;        // [G]
    const int *sl_len = nullptr;        // [Σ slices]
    const int *sl_seg = nullptr;        // [Σ slices * 32]
    const int *segptr = nullptr;        // member g at state_off[g] + g, K_g + 1 entries
    const int *nseg = nullptr;          // [G]
    int rows_max = 0;                   // max rec_rows
    int nseg_max = 0;
    int slots_max = 0;                  // max rows of one warp
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
    int U_max = 0;
    long long U_tot = 0;
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
    const int *dist_fin = nullptr;    // [K_tot] min #transitions to a final state (INT_MAX/2 if none)
    const int *dist_start = nullptr;  // [K_tot] min #transitions from an initial state
    Sched fwd, bwd;
    PdfMap pm;
    void *block = nullptr;
    size_t block_bytes = 0;
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
FBX_HD inline SmemLayout smem_layout(int rows_max, int K_max, int nseg_max, bool exact, bool gbuf) {
    const size_t vsz = exact ? 8 : 4;
    SmemLayout L;
    size_t o = 0;
    L.rec = o; o += fbx_a16((size_t)rows_max * 32 * 8);
    L.u = o; o += fbx_a16((size_t)K_max * vsz);
    L.p = o; if (!exact) o += fbx_a16((size_t)K_max * 4);
    L.part = o; o += fbx_a16((size_t)(nseg_max > 0 ? nseg_max : 1) * vsz);
    L.gbuf = o; if (gbuf) o += fbx_a16((size_t)K_max * 4);
    L.red = o; o += fbx_a16(8 * (2 * 32 + 2 * 64) + 64);
    L.total = o;
    return L;
}

// Dynamic shared memory needed by a forward/backward launch over this graph.
size_t smem_bytes(const Graph &g, bool backward, bool pdf_level);

}  // namespace fbx

struct fb_graph_s {
    fbx::Graph g;
};

namespace fbx {
void set_cuda_error(const char *what, int code);
}
