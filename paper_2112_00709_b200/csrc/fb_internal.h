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

// One direction's per-thread arc schedule (forward = in-arcs / CSC, backward =
// out-arcs / CSR).  Records are {meta, w}: meta = other-endpoint (16 bits) |
// (segment id + 1) << 16 on the last arc of a segment; w = e^{T} (factored) or
// T·log2(e) (exact).  Member g's records start at rec_off[g] (units of 32-record
// rows); warp w's slots start at row warp_row[g*W + w] (relative), it has
// warp_nslot[g*W + w] slots, and lane t has lane_cnt[g*T + t] real records.
struct Sched {
    const uint2 *rec = nullptr;
    const int *rec_rows = nullptr;   // [G] rows (of 32 records) of member g
    const long long *rec_off = nullptr; // [G] first record of member g
    const int *warp_row = nullptr;   // [G*W]
    const int *warp_nslot = nullptr; // [G*W]
    const int *lane_cnt = nullptr;   // [G*T]
    const int *segptr = nullptr;     // member g at state_off[g] + g, K_g + 1 entries
    const int *nseg = nullptr;       // [G]
    int rows_max = 0;                // max rec_rows
    int nseg_max = 0;
    int slots_max = 0;
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

// Dynamic shared memory needed by a forward/backward launch over this graph.
size_t smem_bytes(const Graph &g, bool backward, bool pdf_level);

}  // namespace fbx

struct fb_graph_s {
    fbx::Graph g;
};

namespace fbx {
void set_cuda_error(const char *what, int code);
}
