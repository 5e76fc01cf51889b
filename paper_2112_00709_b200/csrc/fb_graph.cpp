// fb_graph.cpp — host-side graph compiler for libfb (fb_graph_create/destroy/info).
//
// Turns G CSR automata (block-diagonal batch P:202-224) into what the
// one-CTA-per-sequence kernels consume:
//   • per direction (forward pulls over in-arcs = CSC of T, ledger L3; backward
//     pulls over out-arcs = CSR), an nnz-balanced per-thread arc schedule: rows
//     are split into segments of at most ⌈nnz/T⌉ arcs, segments are packed onto
//     the T threads longest-first (LPT), and each warp's arcs are laid out
//     slot-major so that every lane reads its record with one conflict-free
//     64-bit shared-memory load per slot;
//   • BFS viability distances (min #transitions to a final / from an initial
//     state) for exact masking of states that carry no posterior mass;
//   • the inverse state→pdf map (ledger L9) as ascending per-pdf state lists.
// Everything is computed once here and uploaded in a single allocation.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <new>
#include <numeric>
#include <queue>
#include <vector>

#include "fb_internal.h"

namespace fbx {

static const double kLog2e = 1.4426950408889634;
static const int kFar = INT_MAX / 4;

namespace {

struct HostSched {
    std::vector<unsigned char> blob;           // all members, 16-byte aligned each
    std::vector<int> rec_bytes, warp_off, warp_nsl, warp_nsl0;
    std::vector<long long> rec_off;
    int bytes_max = 0, slots_max = 0;
};

// Arc lists for one member graph in one direction: row r reduces over
// (other[a], w[a]) for a in [ptr[r], ptr[r+1]), ascending `other`.
struct RowLists {
    std::vector<int> ptr, other;
    std::vector<double> w;  // natural log
};

// Tie-break keys for slice formation while compiling a relabelled graph (the
// original state id of each new id), so that its slices hold the same rows as the
// original compile's; null otherwise.  Set only around the nested create.
thread_local const std::vector<int> *g_tie = nullptr;

// Grouped sliced-ELL schedule for one member graph (appends to hs); see Sched.
// esize = bytes per element of the gathered u / p arrays; index words hold byte
// offsets relative to the gathered array and are rebased to shared-memory
// offsets by the caller once the layout is known.
// vec: gathered elements are S-float vectors of the cluster kernel (esize = 4·S);
// slots are then placed by local search under the per-phase bank model only.
bool build_member_sched(const RowLists &rl, int K, int T, int mode, int esize, int Lmax, HostSched &hs,
                        bool vec = false) {
    const int W = T / 32;
    struct RowG { int row, len; };
    std::vector<RowG> cls[6];  // g = 1, 2, 4, 8, 16, 32
    for (int r = 0; r < K; ++r) {
        long long d = rl.ptr[r + 1] - rl.ptr[r];
        if (d == 0) continue;
        int lg = 0;
        while (lg < 5 && (d + (1LL << lg) - 1) / (1LL << lg) > Lmax) ++lg;
        cls[lg].push_back({r, (int)((d + (1LL << lg) - 1) / (1LL << lg))});
    }
    struct Slice { int lg, L; std::vector<int> rows; };
    std::vector<Slice> sl;
    for (int lg = 0; lg < 6; ++lg) {
        auto &c = cls[lg];
        if (g_tie)  // relabelled compile: ties in the original state order (same slices as the original)
            std::stable_sort(c.begin(), c.end(), [](const RowG &a, const RowG &b) {
                return a.len != b.len ? a.len > b.len : (*g_tie)[a.row] < (*g_tie)[b.row];
            });
        else
            std::stable_sort(c.begin(), c.end(), [](const RowG &a, const RowG &b) { return a.len > b.len; });
        const int per = 32 >> lg;
        for (size_t i = 0; i < c.size(); i += per) {
            Slice s;
            s.lg = lg;
            s.L = (c[i].len + 1) & ~1;
            if (s.L / 2 >= (1 << 13)) return false;
            for (size_t t = i; t < std::min(c.size(), i + per); ++t) s.rows.push_back(c[t].row);
            sl.push_back(std::move(s));
        }
    }
    // LPT: longest slice first onto the least-loaded warp (cost ≈ slots + slice overhead)
    std::vector<int> order(sl.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sl[a].L > sl[b].L; });
    using Item = std::pair<long long, int>;
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
    // warp 0 also reduces each frame's normaliser / posterior Z: start it with a little load
    for (int w = 0; w < W; ++w) heap.push({(w == 0 && W > 1) ? 6 : 0, w});
    std::vector<std::vector<int>> wsl(W);
    for (int q : order) {
        Item it = heap.top();
        heap.pop();
        wsl[it.second].push_back(q);
        heap.push({it.first + sl[q].L + 4, it.second});
    }
    auto slice_bytes = [](const Slice &s) { return (size_t)128 + (size_t)(s.L / 2) * 384; };
    // inside a warp, the slices of unsplit rows (g = 1) run first: phase A walks them in a
    // loop without the xor-combine (warp_nsl0 of them), then the split-row slices
    std::vector<int> warp_nsl0(W, 0);
    for (int w = 0; w < W; ++w) {
        std::stable_partition(wsl[w].begin(), wsl[w].end(), [&](int q) { return sl[q].lg == 0; });
        for (int q : wsl[w]) warp_nsl0[w] += sl[q].lg == 0;
    }
    std::vector<int> warp_off(W), warp_nsl(W);
    size_t bytes = 0;
    int slots_max = 0;
    for (int w = 0; w < W; ++w) {
        warp_off[w] = (int)bytes;
        warp_nsl[w] = (int)wsl[w].size();
        int slots = 0;
        for (int q : wsl[w]) { bytes += slice_bytes(sl[q]); slots += sl[q].L; }
        slots_max = std::max(slots_max, slots);
    }
    if (bytes >= (size_t)1 << 31) return false;
    const size_t off = hs.blob.size();
    hs.blob.resize(off + bytes, 0);
    unsigned char *base = hs.blob.data() + off;
    const float padw = (mode == MODE_FACTORED) ? 0.0f : -INFINITY;
    // shared-memory bank of a gathered element (32 banks of 4 bytes; an 8-byte
    // element is treated as one of 16 double-width banks)
    const int nbanks = esize == 4 ? 32 : (vec ? 128 / esize : 16);
    // a warp request of esize-byte elements is served in esize/4 phases of
    // 32/(esize/4) lanes (vec); each phase costs its most-loaded bank
    const int nphase = vec ? esize / 4 : 1, lpp = 32 / nphase;
    auto bank_of = [&](uint32_t boff) { return (int)((boff / (uint32_t)esize) % (uint32_t)nbanks); };
    std::vector<std::vector<long long>> rem(32);
    for (int w = 0; w < W; ++w) {
        size_t o = warp_off[w];
        for (int q : wsl[w]) {
            const Slice &s = sl[q];
            const int g = 1 << s.lg, L2 = s.L / 2;
            int32_t *hdr = (int32_t *)(base + o);
            uint32_t *idx = (uint32_t *)(base + o + 128);
            float *wt = (float *)(base + o + 128 + (size_t)L2 * 128);
            for (int l = 0; l < 32; ++l) {
                int ri = l >> s.lg, t = l & (g - 1);
                bool has = ri < (int)s.rows.size();
                uint32_t lead = (has && t == 0) ? (uint32_t)(s.rows[ri] + 1) : 0u;
                hdr[l] = (int32_t)(lead | ((uint32_t)s.lg << 16) | ((uint32_t)L2 << 19));
                rem[l].clear();
                if (has) {
                    const int r = s.rows[ri];
                    const long long d = rl.ptr[r + 1] - rl.ptr[r];
                    const long long len = (d + g - 1) / g;
                    const long long a0 = std::min<long long>(rl.ptr[r + 1], rl.ptr[r] + t * len);
                    const long long a1 = std::min<long long>(rl.ptr[r + 1], a0 + len);
                    for (long long a = a0; a < a1; ++a) rem[l].push_back(a);
                }
            }
            // Bank-aware slot assignment.  A lane's arcs may run in any order (a
            // fixed one, so results stay deterministic).  An arc-row costs as many
            // shared-memory wavefronts as the most distinct addresses falling in one
            // bank, so slots are assigned by bipartite edge colouring of the
            // (lane, bank) multigraph with L colours (Kempe-chain flips, König):
            // conflict-free whenever no bank carries more than L arcs of the slice;
            // excess arcs take a colour free at their lane.  Null slots finally copy
            // a live lane's address (a free broadcast).
            const int Ls = s.L;
            std::vector<long long> grid((size_t)Ls * 32, -1);  // arc index or -1 (null)
            auto addr_of = [&](long long arc) { return (uint32_t)rl.other[arc] * (uint32_t)esize; };
            if (vec) {
                for (int l = 0; l < 32; ++l)
                    for (size_t c0 = 0; c0 < rem[l].size(); ++c0) grid[c0 * 32 + l] = rem[l][c0];
            } else {
                // grid[c*32 + l] = arc of lane l in colour (slot) c; bank_c[b*Ls + c] =
                // lane whose arc of bank b has colour c (proper edges only)
                std::vector<int> bank_c((size_t)nbanks * Ls, -1);
                std::vector<char> over((size_t)Ls * 32, 0);
                auto G_ = [&](int l, int c) -> long long & { return grid[(size_t)c * 32 + l]; };
                auto free_lane = [&](int l) {
                    for (int c = 0; c < Ls; ++c) if (G_(l, c) < 0) return c;
                    return -1;
                };
                auto free_bank = [&](int bk) {
                    for (int c = 0; c < Ls; ++c) if (bank_c[(size_t)bk * Ls + c] < 0) return c;
                    return -1;
                };
                size_t maxlen = 0;
                for (int l = 0; l < 32; ++l) maxlen = std::max(maxlen, rem[l].size());
                for (size_t c0 = 0; c0 < maxlen; ++c0)
                    for (int l = 0; l < 32; ++l) {
                        if (c0 >= rem[l].size()) continue;
                        const long long arc = rem[l][c0];
                        const int bk = bank_of(addr_of(arc));
                        const int ca = free_lane(l);
                        const int cb = free_bank(bk);
                        bool placed = false;
                        if (cb >= 0) {
                            if (bank_c[(size_t)bk * Ls + ca] < 0) {
                                placed = true;
                            } else {
                                // alternating (ca, cb) path from bank bk: bank -ca- lane -cb- bank ...
                                std::vector<std::pair<int, int>> path;  // (lane, colour)
                                bool ok = true;
                                int vb = bk;
                                while (true) {
                                    const int ln = bank_c[(size_t)vb * Ls + ca];
                                    if (ln < 0) break;
                                    path.push_back({ln, ca});
                                    const long long nx = G_(ln, cb);
                                    if (nx < 0) break;
                                    if (over[(size_t)cb * 32 + ln]) { ok = false; break; }
                                    path.push_back({ln, cb});
                                    vb = bank_of(addr_of(nx));
                                }
                                if (ok) {
                                    std::vector<long long> arcs(path.size());
                                    for (size_t i = 0; i < path.size(); ++i) {
                                        arcs[i] = G_(path[i].first, path[i].second);
                                        G_(path[i].first, path[i].second) = -1;
                                        bank_c[(size_t)bank_of(addr_of(arcs[i])) * Ls + path[i].second] = -1;
                                    }
                                    for (size_t i = 0; i < path.size(); ++i) {
                                        const int nc = path[i].second == ca ? cb : ca;
                                        G_(path[i].first, nc) = arcs[i];
                                        bank_c[(size_t)bank_of(addr_of(arcs[i])) * Ls + nc] = path[i].first;
                                    }
                                    placed = G_(l, ca) < 0 && bank_c[(size_t)bk * Ls + ca] < 0;
                                }
                            }
                        }
                        if (placed) {
                            G_(l, ca) = arc;
                            bank_c[(size_t)bk * Ls + ca] = l;
                        } else {  // bank saturated (or blocked path): conflicting placement
                            const int cx = free_lane(l);
                            G_(l, cx) = arc;
                            over[(size_t)cx * 32 + l] = 1;
                        }
                    }
            }
            // local search on top of the colouring: swap two slots of one lane when
            // the two arc-rows' summed wavefront count does not grow (seeded, so the
            // schedule is deterministic)
            auto row_cost = [&](int r) {
                int total = 0;
                for (int ph = 0; ph < nphase; ++ph) {
                    uint32_t seen[32];
                    int ns = 0, cnt[32] = {0}, worst = 1;
                    for (int l = ph * lpp; l < (ph + 1) * lpp; ++l) {
                        const long long arc = grid[(size_t)r * 32 + l];
                        if (arc < 0) continue;
                        const uint32_t ad = addr_of(arc);
                        bool dup = false;
                        for (int x = 0; x < ns; ++x)
                            if (seen[x] == ad) { dup = true; break; }
                        if (dup) continue;
                        seen[ns++] = ad;
                        worst = std::max(worst, ++cnt[bank_of(ad)]);
                    }
                    total += worst;
                }
                return total;
            };
            if (Ls > 1 && mode == MODE_FACTORED) {
                std::vector<int> rc(Ls);
                for (int r = 0; r < Ls; ++r) rc[r] = row_cost(r);
                uint64_t rng = 0x9E3779B97F4A7C15ull ^ ((uint64_t)q << 17) ^ (uint64_t)Ls;
                auto next = [&]() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; };
                const int iters = 60 * Ls * 32;
                for (int it = 0; it < iters; ++it) {
                    const int l = (int)(next() % 32), r1 = (int)(next() % Ls), r2 = (int)(next() % Ls);
                    if (r1 == r2) continue;
                    long long &x1 = grid[(size_t)r1 * 32 + l], &x2 = grid[(size_t)r2 * 32 + l];
                    if (x1 < 0 && x2 < 0) continue;
                    std::swap(x1, x2);
                    const int c1 = row_cost(r1), c2 = row_cost(r2);
                    if (c1 + c2 <= rc[r1] + rc[r2]) { rc[r1] = c1; rc[r2] = c2; }
                    else std::swap(x1, x2);
                }
            }
            for (int sl2 = 0; sl2 < Ls; ++sl2) {
                uint32_t bcast = 0;
                for (int l = 0; l < 32; ++l)
                    if (grid[(size_t)sl2 * 32 + l] >= 0) { bcast = addr_of(grid[(size_t)sl2 * 32 + l]); break; }
                for (int l = 0; l < 32; ++l) {
                    const long long a = grid[(size_t)sl2 * 32 + l];
                    uint32_t boff = bcast;
                    float wf = padw;
                    if (a >= 0) {
                        boff = addr_of(a);
                        double wn = rl.w[a];
                        wf = (mode == MODE_FACTORED) ? (float)std::exp(wn)
                             : (mode == MODE_VITERBI) ? (float)wn : (float)(wn * kLog2e);
                        if (std::isinf(wn) && wn < 0) wf = padw;
                    }
                    uint32_t &word = idx[(sl2 / 2) * 32 + l];
                    word |= (sl2 & 1) ? (boff << 16) : boff;
                    wt[((sl2 / 2) * 32 + l) * 2 + (sl2 & 1)] = wf;
                }
            }
            o += slice_bytes(s);
        }
    }
    hs.rec_off.push_back((long long)off);
    hs.rec_bytes.push_back((int)bytes);
    hs.warp_off.insert(hs.warp_off.end(), warp_off.begin(), warp_off.end());
    hs.warp_nsl.insert(hs.warp_nsl.end(), warp_nsl.begin(), warp_nsl.end());
    hs.warp_nsl0.insert(hs.warp_nsl0.end(), warp_nsl0.begin(), warp_nsl0.end());
    hs.bytes_max = std::max<int>(hs.bytes_max, (int)bytes);
    hs.slots_max = std::max(hs.slots_max, slots_max);
    return (long long)K * esize <= 65536;  // byte offsets are 16-bit
}

int pow2ceil(long long x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

struct Packer {
    std::vector<unsigned char> buf;
    template <class T>
    size_t put(const std::vector<T> &v) {
        size_t off = align16(buf.size());
        buf.resize(off + v.size() * sizeof(T) + 16);
        if (!v.empty()) std::memcpy(buf.data() + off, v.data(), v.size() * sizeof(T));
        return off;
    }
};

bool bad(float x) { return std::isnan(x) || (std::isinf(x) && x > 0); }

// Host image of a CPlan (fb_internal.h).
struct HostCPlan {
    int C = 0, S = 0, T = 0, spt = 0, K_int = 0, Kc_max = 0, Dc_max = 0, emis16 = 0, nop = 0, split = 0;
    std::vector<int> part_off, pdf_lo, perm, ipdf, idf, ids;
    std::vector<float> ii2, if2;
    std::vector<unsigned> pq;
    HostSched hf, hb;
    std::vector<int> fptr, fsrc, bptr, bsrc;
    std::vector<float> fw2, bw2;
    size_t smem_fwd = 0, smem_bwd = 0;
};

// Cluster plan for one shared graph (G == 1, factored mode): C parts along
// ascending pdf ranges balanced on arcs (both directions) + a per-state phase-B
// cost, internal order (pdf, state id) inside a part, each part padded to a
// multiple of 4 states; per-part sliced-ELL schedules over S-float elements.
bool build_cluster_plan(const RowLists &in, const RowLists &out, int K, int D, const std::vector<int> &pdf,
                        const std::vector<int> &dist_fin, const std::vector<int> &dist_start,
                        const std::vector<float> &init2, const std::vector<float> &final2, int C, int S, int Lmax,
                        HostCPlan &cp, int Tforce = 0, bool nop = false) {
    // 1024 threads (≤ 4 owned states each) unless the part needs more states per thread
    int T = 1024;
    if (const char *e = std::getenv("FBX_CLUSTER_T")) T = std::atoi(e) == 512 ? 512 : 1024;
    if (Tforce) T = Tforce;
    const int W = T / 32;
    cp = HostCPlan();
    cp.C = C; cp.S = S; cp.T = T; cp.nop = nop;
    // local/remote split of phase A around the exchange wait: measured faster for the
    // no-p (4,4) paper-shape plan (N2 fwd 5.36 → 5.12 ms, bwd 8.72 → 8.36 ms), slower
    // for (2,2) on C3/C4 (6.52 → 6.94 ms); FBX_CLUSTER_SPLIT=0|1 overrides
    // bit 0: forward, bit 1: backward.  With p-exchange (round 2) the forward is faster
    // unsplit (N2 3.72 → 3.60 ms); after the lighter phase B of the IZ epilogue, interleaved
    // emissions and vector lattice accesses the backward is too (N2 bwd 4.27 → 4.19 ms, step
    // 7.57 → 7.49 ms), so no plan splits by default.
    cp.split = 0;
    if (const char *e = std::getenv("FBX_CLUSTER_SPLIT"))  // 0 none, 1 both, f forward only, b backward only
        cp.split = e[0] == 'f' ? 1 : e[0] == 'b' ? 2 : (std::atoi(e) != 0 ? 3 : 0);
    std::vector<double> cost(D, 0.0);
    for (int k = 0; k < K; ++k)
        cost[pdf[k]] += (in.ptr[k + 1] - in.ptr[k]) + (out.ptr[k + 1] - out.ptr[k]) + 8.0;
    double total = 0;
    for (double x : cost) total += x;
    cp.pdf_lo.assign(C + 1, 0);
    cp.pdf_lo[C] = D;
    {
        double acc = 0;
        int c = 1;
        for (int d = 0; d < D && c < C; ++d) {
            acc += cost[d];
            while (c < C && acc >= total * c / C) cp.pdf_lo[c++] = d + 1;
        }
        for (; c < C; ++c) cp.pdf_lo[c] = D;
    }
    std::vector<std::pair<int, int>> ps;
    for (int k = 0; k < K; ++k) ps.push_back({pdf[k], k});
    std::sort(ps.begin(), ps.end());
    cp.part_off.assign(C + 1, 0);
    std::vector<int> inv(K, -1);
    {
        size_t x = 0;
        for (int c = 0; c < C; ++c) {
            const int start = (int)cp.perm.size();
            while (x < ps.size() && ps[x].first < cp.pdf_lo[c + 1]) {
                inv[ps[x].second] = (int)cp.perm.size();
                cp.perm.push_back(ps[x].second);
                ++x;
            }
            if ((int)cp.perm.size() == start) return false;  // an empty part
            while (cp.perm.size() % 4) cp.perm.push_back(-1);
            cp.part_off[c + 1] = (int)cp.perm.size();
            cp.Kc_max = std::max(cp.Kc_max, cp.part_off[c + 1] - start);
        }
    }
    cp.K_int = (int)cp.perm.size();
    if ((long long)cp.K_int * S * 4 > 65536) return false;  // 16-bit gather offsets
    cp.spt = (cp.Kc_max + T - 1) / T;
    if (T == 1024 && (cp.spt > 4 || S == 4))  // S = 4 kernels need > 64 registers per thread
        return build_cluster_plan(in, out, K, D, pdf, dist_fin, dist_start, init2, final2, C, S, Lmax, cp, 512, nop);
    if (cp.spt > 8) return false;
    cp.spt = cp.spt <= 4 ? cp.spt : (cp.spt <= 6 ? 6 : 8);
    const int Ki = cp.K_int;
    cp.ipdf.assign(Ki, 0); cp.idf.assign(Ki, kFar); cp.ids.assign(Ki, kFar);
    cp.ii2.assign(Ki, -INFINITY); cp.if2.assign(Ki, -INFINITY);
    for (int i = 0; i < Ki; ++i) {
        const int o = cp.perm[i];
        if (o < 0) continue;
        cp.ipdf[i] = pdf[o]; cp.idf[i] = dist_fin[o]; cp.ids[i] = dist_start[o];
        cp.ii2[i] = init2[o]; cp.if2[i] = final2[o];
    }
    // pdf → (first local position, count) inside its part
    cp.pq.assign(D, 0u);
    for (int c = 0; c < C; ++c)
        for (int i = cp.part_off[c]; i < cp.part_off[c + 1]; ++i) {
            const int o = cp.perm[i];
            if (o < 0) continue;
            unsigned &w = cp.pq[pdf[o]];
            if ((w >> 16) == 0) w = (unsigned)(i - cp.part_off[c]);
            w += 1u << 16;
        }
    // emission segment of each part
    cp.emis16 = (D % 4) == 0;
    int dmax = 0;
    for (int c = 0; c < C; ++c) {
        int lo = cp.pdf_lo[c], hi = cp.pdf_lo[c + 1];
        if (cp.emis16) { lo &= ~3; hi = std::min(D, (hi + 3) & ~3); }
        dmax = std::max(dmax, hi - lo);
    }
    cp.Dc_max = std::max(4, (dmax + 3) & ~3);
    // per-part schedules and the exact-fallback arc lists (internal ids)
    auto lists = [&](const RowLists &rl, std::vector<int> &ptr, std::vector<int> &src, std::vector<float> &w2) {
        ptr.assign(Ki + 1, 0);
        for (int i = 0; i < Ki; ++i) {
            const int o = cp.perm[i];
            if (o >= 0)
                for (int a = rl.ptr[o]; a < rl.ptr[o + 1]; ++a) {
                    src.push_back(inv[rl.other[a]]);
                    w2.push_back((float)(rl.w[a] * kLog2e));
                }
            ptr[i + 1] = (int)src.size();
        }
    };
    lists(in, cp.fptr, cp.fsrc, cp.fw2);
    lists(out, cp.bptr, cp.bsrc, cp.bw2);
    for (int dir = 0; dir < 2; ++dir) {
        const RowLists &rl = dir ? out : in;
        HostSched &hs = dir ? cp.hb : cp.hf;
        const bool sp = (cp.split >> dir) & 1;
        for (int c = 0; c < C; ++c) {
            const int Kc = cp.part_off[c + 1] - cp.part_off[c];
            // split: member 2c = arcs from this part's own states (run before the
            // exchange wait), member 2c+1 = arcs from the other parts
            for (int pass = 0; pass < (sp ? 2 : 1); ++pass) {
                RowLists pl;
                pl.ptr.assign(Kc + 1, 0);
                for (int r = 0; r < Kc; ++r) {
                    const int o = cp.perm[cp.part_off[c] + r];
                    if (o >= 0)
                        for (int a = rl.ptr[o]; a < rl.ptr[o + 1]; ++a) {
                            const int si = inv[rl.other[a]];
                            const bool local = si >= cp.part_off[c] && si < cp.part_off[c + 1];
                            if (sp && local != (pass == 0)) continue;
                            pl.other.push_back(si);
                            pl.w.push_back(rl.w[a]);
                        }
                    pl.ptr[r + 1] = (int)pl.other.size();
                }
                if (!build_member_sched(pl, Kc, T, MODE_FACTORED, 4 * S, Lmax, hs, true)) return false;
            }
        }
        if (sp) {  // both members of a part sit back to back in shared memory
            hs.bytes_max = 0;
            for (int c = 0; c < C; ++c) hs.bytes_max = std::max(hs.bytes_max, hs.rec_bytes[2 * c] + hs.rec_bytes[2 * c + 1]);
        }
    }
    cp.smem_fwd = cl_layout(cp.hf.bytes_max, Ki, cp.Kc_max, cp.Dc_max, S, C, W, false, nop).total;
    cp.smem_bwd = cl_layout(cp.hb.bytes_max, Ki, cp.Kc_max, cp.Dc_max, S, C, W, true, nop).total;
    if (std::getenv("FBX_CLUSTER_DEBUG"))
        std::fprintf(stderr, "cluster plan C=%d S=%d nop=%d split=%d T=%d spt=%d K_int=%d Kc_max=%d rec_fwd=%d rec_bwd=%d smem_fwd=%zu smem_bwd=%zu\n",
                     C, S, (int)nop, cp.split, T, cp.spt, cp.K_int, cp.Kc_max, cp.hf.bytes_max, cp.hb.bytes_max, cp.smem_fwd,
                     cp.smem_bwd);
    return cp.smem_fwd <= (size_t)kSmemLimit && cp.smem_bwd <= (size_t)kSmemLimit;
}

}  // namespace

size_t viterbi_smem_bytes(const Graph &g, bool global_sched) {
    return smem_layout(global_sched ? 0 : g.vit.bytes_max, g.T * g.spt, true, false).total +
           fbx_a16((size_t)g.T * g.spt * 4);
}

size_t smem_bytes(const Graph &g, bool backward, bool post) {
    const Sched &s = backward ? g.bwd : g.fwd;
    return smem_layout(s.bytes_max, g.T * g.spt, g.mode == MODE_EXACT, backward && post).total;
}

// ---------------------------------------------------------------- bank-aware relabelling
//
// Shared-memory cost model of one frame of the one-CTA kernels (32 banks of 4
// bytes; a state's bank is its id mod 32):
//   • gathers: a slice with L slots per lane is conflict-free after the per-slice
//     edge colouring iff no bank holds more than L of its arcs (König), else it
//     costs about max_b(arcs in bank b) wavefronts: cost_g = max(L, max_b h[b]);
//   • part-row stores: the slice's row leaders write part[row]: max_b (rows in b);
//   • emission gathers of phase B: thread t owns ids t + kT, so each aligned block
//     of 32 ids gathers φ[pdf] from the staged row: max_b (states with pdf ≡ b).
// Both directions' slices (in-arcs / out-arcs) and the emission blocks (read in
// both) are summed.  A seeded local search over swaps of two ids accepts moves
// that do not raise the total; the slice membership (rows grouped by length, ties
// in original order) does not depend on the labelling.
struct RelabelDir {
    std::vector<int> L;                              // slots per lane of slice s
    std::vector<std::vector<std::pair<int, int>>> src;  // state → (slice, #arcs gathered from it)
    std::vector<int> lead;                           // state → slice it is a row of (−1 none)
};

static RelabelDir relabel_slices(const RowLists &rl, int K, int Lmax) {
    RelabelDir R;
    R.lead.assign(K, -1);
    R.src.assign(K, {});
    struct RowG { int row, len; };
    std::vector<RowG> cls[6];
    for (int r = 0; r < K; ++r) {
        long long d = rl.ptr[r + 1] - rl.ptr[r];
        if (d == 0) continue;
        int lg = 0;
        while (lg < 5 && (d + (1LL << lg) - 1) / (1LL << lg) > Lmax) ++lg;
        cls[lg].push_back({r, (int)((d + (1LL << lg) - 1) / (1LL << lg))});
    }
    for (int lg = 0; lg < 6; ++lg) {
        auto &c = cls[lg];
        std::stable_sort(c.begin(), c.end(), [](const RowG &a, const RowG &b) { return a.len > b.len; });
        const int per = 32 >> lg;
        for (size_t i = 0; i < c.size(); i += per) {
            const int sid = (int)R.L.size();
            R.L.push_back((c[i].len + 1) & ~1);
            std::vector<int> cnt;
            for (size_t t = i; t < std::min(c.size(), i + per); ++t) {
                const int r = c[t].row;
                R.lead[r] = sid;
                for (int a = rl.ptr[r]; a < rl.ptr[r + 1]; ++a) {
                    auto &v = R.src[rl.other[a]];
                    if (!v.empty() && v.back().first == sid) v.back().second++;
                    else v.push_back({sid, 1});
                }
            }
        }
    }
    return R;
}

// Returns pos[state] = new id (a permutation of 0 … K−1).
static std::vector<int> bank_relabel(const RowLists &in, const RowLists &outl, int K, int Lmax,
                                     const std::vector<int> &pdf, long long iters, bool verbose) {
    RelabelDir dir[2] = {relabel_slices(in, K, Lmax), relabel_slices(outl, K, Lmax)};
    const int NB = 32;
    std::vector<int> pos(K), at(K);
    std::iota(pos.begin(), pos.end(), 0);
    std::iota(at.begin(), at.end(), 0);
    // histograms
    std::vector<std::vector<int>> hg[2], hl[2];
    std::vector<int> cg[2], cl[2];
    for (int d = 0; d < 2; ++d) {
        const int ns = (int)dir[d].L.size();
        hg[d].assign(ns, std::vector<int>(NB, 0));
        hl[d].assign(ns, std::vector<int>(NB, 0));
        for (int x = 0; x < K; ++x) {
            for (auto &sc : dir[d].src[x]) hg[d][sc.first][pos[x] % NB] += sc.second;
            if (dir[d].lead[x] >= 0) hl[d][dir[d].lead[x]][pos[x] % NB]++;
        }
        cg[d].resize(ns);
        cl[d].resize(ns);
    }
    const int ng = (K + NB - 1) / NB;
    std::vector<std::vector<int>> he(ng, std::vector<int>(NB, 0));
    std::vector<int> ce(ng);
    for (int x = 0; x < K; ++x) he[pos[x] / NB][pdf[x] % NB]++;
    auto mx = [&](const std::vector<int> &h) { int m = 0; for (int v : h) m = std::max(m, v); return m; };
    long long total = 0;
    for (int d = 0; d < 2; ++d)
        for (size_t sl = 0; sl < dir[d].L.size(); ++sl) {
            cg[d][sl] = std::max(dir[d].L[sl], mx(hg[d][sl]));
            cl[d][sl] = mx(hl[d][sl]);
            total += cg[d][sl] + cl[d][sl];
        }
    for (int g = 0; g < ng; ++g) { ce[g] = mx(he[g]); total += 2 * ce[g]; }
    const long long start = total;
    uint64_t rng = 0x2545F4914F6CDD1Dull ^ (uint64_t)K;
    auto next = [&]() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; };
    std::vector<int> touched_s[2], touched_g;
    auto apply = [&](int x, int from, int to) {  // move state x from id `from` to id `to` (histograms only)
        for (int d = 0; d < 2; ++d) {
            for (auto &sc : dir[d].src[x]) {
                hg[d][sc.first][from % NB] -= sc.second;
                hg[d][sc.first][to % NB] += sc.second;
                touched_s[d].push_back(sc.first);
            }
            const int sl = dir[d].lead[x];
            if (sl >= 0) { hl[d][sl][from % NB]--; hl[d][sl][to % NB]++; touched_s[d].push_back(sl); }
        }
        he[from / NB][pdf[x] % NB]--;
        he[to / NB][pdf[x] % NB]++;
        touched_g.push_back(from / NB);
        touched_g.push_back(to / NB);
    };
    for (long long it = 0; it < iters; ++it) {
        const int p1 = (int)(next() % (uint64_t)K), p2 = (int)(next() % (uint64_t)K);
        if (p1 == p2 || (p1 % NB == p2 % NB && p1 / NB == p2 / NB)) continue;
        const int x = at[p1], y = at[p2];
        for (int d = 0; d < 2; ++d) touched_s[d].clear();
        touched_g.clear();
        apply(x, p1, p2);
        apply(y, p2, p1);
        long long delta = 0;
        std::vector<std::pair<int, int>> newc[2];
        for (int d = 0; d < 2; ++d) {
            auto &ts = touched_s[d];
            std::sort(ts.begin(), ts.end());
            ts.erase(std::unique(ts.begin(), ts.end()), ts.end());
            for (int sl : ts) {
                const int g2 = std::max(dir[d].L[sl], mx(hg[d][sl])), l2 = mx(hl[d][sl]);
                delta += (g2 - cg[d][sl]) + (l2 - cl[d][sl]);
                newc[d].push_back({g2, l2});
            }
        }
        std::sort(touched_g.begin(), touched_g.end());
        touched_g.erase(std::unique(touched_g.begin(), touched_g.end()), touched_g.end());
        std::vector<int> newe;
        for (int g : touched_g) { const int e2 = mx(he[g]); delta += 2 * (e2 - ce[g]); newe.push_back(e2); }
        if (delta <= 0) {
            for (int d = 0; d < 2; ++d)
                for (size_t i = 0; i < touched_s[d].size(); ++i) {
                    cg[d][touched_s[d][i]] = newc[d][i].first;
                    cl[d][touched_s[d][i]] = newc[d][i].second;
                }
            for (size_t i = 0; i < touched_g.size(); ++i) ce[touched_g[i]] = newe[i];
            total += delta;
            pos[x] = p2; pos[y] = p1; at[p1] = y; at[p2] = x;
        } else {
            for (int d = 0; d < 2; ++d) touched_s[d].clear();
            touched_g.clear();
            apply(x, p2, p1);
            apply(y, p1, p2);
        }
    }
    if (verbose) {
        long long lsum = 0;
        for (int d = 0; d < 2; ++d) for (int L : dir[d].L) lsum += L;
        std::fprintf(stderr, "[fbx] bank relabel K=%d: modelled smem wavefronts/frame %lld -> %lld (floor %lld)\n", K,
                     start, total, lsum + (long long)(dir[0].L.size() + dir[1].L.size()) + 2LL * ng);
    }
    return pos;
}

}  // namespace fbx

using namespace fbx;

static fb_status create_impl(fb_graph *out, int32_t G, const int32_t *state_offsets, const int32_t *row_ptr,
                             const int32_t *col, const float *log_w, const float *log_init, const float *log_final,
                             const int32_t *pdf_of, int32_t D, int32_t flags);

extern "C" fb_status fb_graph_create(fb_graph *out, int32_t G, const int32_t *state_offsets,
                                     const int32_t *row_ptr, const int32_t *col, const float *log_w,
                                     const float *log_init, const float *log_final,
                                     const int32_t *pdf_of, int32_t D, int32_t flags) {
    fb_status r = create_impl(out, G, state_offsets, row_ptr, col, log_w, log_init, log_final, pdf_of, D, flags);
    if (r != FB_OK) return r;
    fb_graph h = *out;
    const Graph &g = h->g;
    // relabelled twin for the lfmmi denominator passes (one CTA per sequence, factored)
    const bool stats_only = (flags & FB_GRAPH_DRY_RUN) && std::getenv("FBX_RELABEL_STATS");
    if (G != 1 || g.mode != MODE_FACTORED || !g.legacy_ok || g.cp.ok || ((flags & FB_GRAPH_DRY_RUN) && !stats_only) ||
        std::getenv("FBX_NO_RELABEL"))
        return FB_OK;
    const int K = g.K_tot;
    RowLists in, outl;
    in.ptr.assign(K + 1, 0);
    outl.ptr.assign(K + 1, 0);
    for (int i = 0; i < K; ++i) {
        for (int a = row_ptr[i]; a < row_ptr[i + 1]; ++a) { outl.other.push_back(col[a]); in.ptr[col[a] + 1]++; }
        outl.ptr[i + 1] = (int)outl.other.size();
    }
    for (int j = 0; j < K; ++j) in.ptr[j + 1] += in.ptr[j];
    in.other.resize(outl.other.size());
    {
        std::vector<int> fill(K, 0);
        for (int i = 0; i < K; ++i)
            for (int a = outl.ptr[i]; a < outl.ptr[i + 1]; ++a) in.other[in.ptr[outl.other[a]] + fill[outl.other[a]]++] = i;
    }
    std::vector<int> pdf(K);
    for (int i = 0; i < K; ++i) pdf[i] = pdf_of ? pdf_of[i] : i;
    int lmax = 24;
    if (const char *e = std::getenv("FBX_LMAX")) lmax = std::max(1, std::atoi(e));
    long long iters = 100LL * K;
    if (const char *e = std::getenv("FBX_RELABEL_ITERS")) iters = std::atoll(e);
    const std::vector<int> pos = bank_relabel(in, outl, K, lmax, pdf, iters, std::getenv("FBX_RELABEL_STATS") != nullptr);
    if (stats_only) return FB_OK;
    std::vector<int> inv(K);
    for (int i = 0; i < K; ++i) inv[pos[i]] = i;
    // the permuted graph: new id q is original state inv[q]
    std::vector<int32_t> rp(K + 1, 0), cl;
    std::vector<float> lw, li(K), lf(K);
    std::vector<int32_t> pd(K);
    cl.reserve(col ? row_ptr[K] : 0);
    for (int q = 0; q < K; ++q) {
        const int i = inv[q];
        for (int a = row_ptr[i]; a < row_ptr[i + 1]; ++a) { cl.push_back(pos[col[a]]); lw.push_back(log_w[a]); }
        rp[q + 1] = (int32_t)cl.size();
        li[q] = log_init[i];
        lf[q] = log_final[i];
        pd[q] = pdf[i];
    }
    fb_graph hp = nullptr;
    g_tie = &inv;
    r = create_impl(&hp, 1, state_offsets, rp.data(), cl.data(), lw.data(), li.data(), lf.data(), pd.data(), D,
                    flags | FB_GRAPH_FORCE_FACTORED);
    g_tie = nullptr;
    if (r == FB_OK) h->perm = hp;  // any failure: lfmmi simply runs on the original labelling
    return FB_OK;
}

static fb_status create_impl(fb_graph *out, int32_t G, const int32_t *state_offsets,
                                     const int32_t *row_ptr, const int32_t *col, const float *log_w,
                                     const float *log_init, const float *log_final,
                                     const int32_t *pdf_of, int32_t D, int32_t flags) {
    if (!out || G < 1 || !state_offsets || !row_ptr || !log_init || !log_final || D < 1)
        return FB_ERR_INVALID_ARG;
    if (D > (1 << 20)) return FB_ERR_UNSUPPORTED;  // pdf ids are packed in 20 bits on device
    *out = nullptr;
    if (state_offsets[0] != 0) return FB_ERR_INVALID_GRAPH;
    for (int g = 0; g < G; ++g)
        if (state_offsets[g + 1] <= state_offsets[g]) return FB_ERR_INVALID_GRAPH;
    const int K_tot = state_offsets[G];
    if (row_ptr[0] != 0) return FB_ERR_INVALID_GRAPH;
    for (int i = 0; i < K_tot; ++i)
        if (row_ptr[i + 1] < row_ptr[i]) return FB_ERR_INVALID_GRAPH;
    const long long nnz = row_ptr[K_tot];
    if (nnz > 0 && (!col || !log_w)) return FB_ERR_INVALID_ARG;

    Graph gr;
    gr.G = G;
    gr.K_tot = K_tot;
    gr.D = D;
    gr.nnz = nnz;
    std::vector<int> member(K_tot);
    for (int g = 0; g < G; ++g) {
        int K = state_offsets[g + 1] - state_offsets[g];
        if (K > 65536) return FB_ERR_UNSUPPORTED;
        gr.K_max = std::max(gr.K_max, K);
        gr.nnz_max = std::max<long long>(gr.nnz_max, row_ptr[state_offsets[g + 1]] - row_ptr[state_offsets[g]]);
        for (int k = state_offsets[g]; k < state_offsets[g + 1]; ++k) member[k] = g;
    }
    // validate arcs, weights, pdfs
    bool factored_ok = true;
    for (int i = 0; i < K_tot; ++i) {
        int g = member[i];
        for (int a = row_ptr[i]; a < row_ptr[i + 1]; ++a) {
            if (col[a] < state_offsets[g] || col[a] >= state_offsets[g + 1]) return FB_ERR_INVALID_GRAPH;
            if (bad(log_w[a])) return FB_ERR_INVALID_GRAPH;
            if (!(std::isinf(log_w[a]) && log_w[a] < 0) && (log_w[a] < -80.0f || log_w[a] > 80.0f))
                factored_ok = false;
        }
        if (bad(log_init[i]) || bad(log_final[i])) return FB_ERR_INVALID_GRAPH;
    }
    std::vector<int> pdf(K_tot);
    for (int i = 0; i < K_tot; ++i) {
        int p = pdf_of ? pdf_of[i] : i - state_offsets[member[i]];
        if (p < 0 || p >= D) return pdf_of ? FB_ERR_INVALID_GRAPH : FB_ERR_SHAPE;
        pdf[i] = p;
    }
    // ⊕ evaluation mode: exp-factorised rows pay off on large
    // ergodic graphs; small / left-to-right graphs use max-then-sum.
    if (flags & FB_GRAPH_FORCE_EXACT) {
        gr.mode = MODE_EXACT;
    } else if (flags & FB_GRAPH_FORCE_FACTORED) {
        if (!factored_ok) return FB_ERR_UNSUPPORTED;
        gr.mode = MODE_FACTORED;
    } else {
        long long nnz_min = LLONG_MAX;
        for (int g = 0; g < G; ++g)
            nnz_min = std::min<long long>(nnz_min, row_ptr[state_offsets[g + 1]] - row_ptr[state_offsets[g]]);
        gr.mode = (factored_ok && nnz_min >= 4096) ? MODE_FACTORED : MODE_EXACT;
    }
    // threads per CTA and states per thread: factored (large ergodic) graphs use
    // 1024 threads (~20 arcs per thread per frame); exact-mode graphs are short
    // dependent chains, so they get ~4 arcs per thread to cut per-frame latency.
    int T;
    if (gr.mode == MODE_FACTORED)
        T = gr.nnz_max >= 16384 ? 1024 : std::min(1024, std::max(128, pow2ceil((gr.nnz_max + 15) / 16)));
    else
        T = std::min(1024, std::max(128, pow2ceil((gr.nnz_max + 7) / 8)));
    // many small exact-mode members (a batch of numerator graphs): ≤ 256 threads per CTA
    // while ≤ 4 states per thread suffice, so more utterances run concurrently per SM
    if (gr.mode == MODE_EXACT && G > 1 && T > 256 && (gr.K_max + 255) / 256 <= 4) T = 256;
    // ... and 128 while ≤ 4 states per thread suffice (N2's 454-state numerators: 7 CTAs
    // per SM instead of 2, so every utterance of a 128-batch is resident on the idle SMs)
    if (gr.mode == MODE_EXACT && G > 1 && T > 128 && (gr.K_max + 127) / 128 <= 4) T = 128;
    if (const char *e = std::getenv("FBX_EXACT_T"); e && gr.mode == MODE_EXACT) T = std::max(128, std::atoi(e));
    if (const char *e = std::getenv("FBX_FACT_T"); e && gr.mode == MODE_FACTORED) T = std::max(128, std::atoi(e));
    T = std::max(T, std::min(1024, pow2ceil((gr.K_max + kMaxSPT - 1) / kMaxSPT)));
    T = std::min(1024, pow2ceil(T));  // T ∈ {128, 256, 512, 1024}: the kernels' compile-time CTA size
    int spt = (gr.K_max + T - 1) / T;
    spt = spt <= 4 ? spt : (spt <= 6 ? 6 : 8);  // instantiated: 1, 2, 3, 4, 6, 8
    if ((gr.K_max + T - 1) / T > kMaxSPT) return FB_ERR_UNSUPPORTED;
    gr.T = T;
    // longest row segment per lane before a row is split over 2, 4, … lanes
    int lmax = gr.mode == MODE_FACTORED ? 24 : 4;  // factored: 24 measured 2% faster than 12 on C4 (fewer slices)
    if (const char *e = std::getenv("FBX_LMAX")) lmax = std::max(1, std::atoi(e));
    gr.W = T / 32;
    gr.spt = spt;

    // per-member schedules, distances, pdf slots
    HostSched hf, hb, hv;
    bool vit_ok = true;
    std::vector<int> dist_fin(K_tot, kFar), dist_start(K_tot, kFar);
    std::vector<int> slot_off(G + 1, 0), slot_pdf, slot_sptr(1, 0), slot_states;
    std::vector<int> pdf_slot((size_t)G * D, -1);
    std::vector<int> slot_pos(K_tot, 0);
    std::vector<float> init2(K_tot), final2(K_tot);
    for (int i = 0; i < K_tot; ++i) {
        init2[i] = (float)((double)log_init[i] * kLog2e);
        final2[i] = (float)((double)log_final[i] * kLog2e);
    }
    RowLists in0, out0;  // member 0's arc lists (cluster plan of a shared graph)
    std::vector<int> lit_row_off(G), lit_ptr(1, 0), lit_src, lit_inst(G + 1, 0);
    std::vector<double> lit_w;
    std::vector<int> lit_optr(1, 0), lit_odst;  // out-arc lists (same row numbering as lit_ptr)
    std::vector<double> lit_ow;
    for (int g = 0; g < G; ++g) {
        const int s0 = state_offsets[g], K = state_offsets[g + 1] - s0;
        RowLists in, outl;
        in.ptr.assign(K + 1, 0);
        outl.ptr.assign(K + 1, 0);
        // out-arcs (CSR), sorted by destination within a row (stable for duplicates)
        std::vector<std::pair<int, int>> tmp;
        for (int i = 0; i < K; ++i) {
            tmp.clear();
            for (int a = row_ptr[s0 + i]; a < row_ptr[s0 + i + 1]; ++a) tmp.push_back({col[a] - s0, a});
            std::stable_sort(tmp.begin(), tmp.end(), [](auto &x, auto &y) { return x.first < y.first; });
            for (auto &pr : tmp) {
                outl.other.push_back(pr.first);
                outl.w.push_back(log_w[pr.second]);
                in.ptr[pr.first + 1]++;
            }
            outl.ptr[i + 1] = (int)outl.other.size();
        }
        // in-arcs (CSC) in ascending source order
        for (int j = 0; j < K; ++j) in.ptr[j + 1] += in.ptr[j];
        in.other.resize(outl.other.size());
        in.w.resize(outl.other.size());
        std::vector<int> fill(K, 0);
        for (int i = 0; i < K; ++i)
            for (int a = outl.ptr[i]; a < outl.ptr[i + 1]; ++a) {
                int j = outl.other[a];
                int p = in.ptr[j] + fill[j]++;
                in.other[p] = i;
                in.w[p] = outl.w[a];
            }
        const int esize = gr.mode == MODE_EXACT ? 8 : 4;
        if (!build_member_sched(in, K, T, gr.mode, esize, lmax, hf)) return FB_ERR_UNSUPPORTED;
        if (!build_member_sched(outl, K, T, gr.mode, esize, lmax, hb)) return FB_ERR_UNSUPPORTED;
        if (vit_ok && !build_member_sched(in, K, T, MODE_VITERBI, 8, lmax, hv)) vit_ok = false;
        // BFS over finite arcs: distance to a final state (reverse) / from an initial state
        std::deque<int> q;
        for (int k = 0; k < K; ++k)
            if (!(std::isinf(log_final[s0 + k]) && log_final[s0 + k] < 0)) { dist_fin[s0 + k] = 0; q.push_back(k); }
        while (!q.empty()) {
            int j = q.front(); q.pop_front();
            for (int a = in.ptr[j]; a < in.ptr[j + 1]; ++a) {
                if (std::isinf(in.w[a]) && in.w[a] < 0) continue;
                int i = in.other[a];
                if (dist_fin[s0 + i] == kFar) { dist_fin[s0 + i] = dist_fin[s0 + j] + 1; q.push_back(i); }
            }
        }
        for (int k = 0; k < K; ++k)
            if (!(std::isinf(log_init[s0 + k]) && log_init[s0 + k] < 0)) { dist_start[s0 + k] = 0; q.push_back(k); }
        while (!q.empty()) {
            int i = q.front(); q.pop_front();
            for (int a = outl.ptr[i]; a < outl.ptr[i + 1]; ++a) {
                if (std::isinf(outl.w[a]) && outl.w[a] < 0) continue;
                int j = outl.other[a];
                if (dist_start[s0 + j] == kFar) { dist_start[s0 + j] = dist_start[s0 + i] + 1; q.push_back(j); }
            }
        }
        // inverse pdf map: distinct pdfs ascending, states ascending
        std::vector<std::pair<int, int>> ps;
        for (int k = 0; k < K; ++k) ps.push_back({pdf[s0 + k], k});
        std::sort(ps.begin(), ps.end());
        int local = 0;
        for (size_t x = 0; x < ps.size(); ++x) {
            if (x == 0 || ps[x].first != ps[x - 1].first) {
                if (x) slot_sptr.push_back((int)slot_states.size());
                slot_pdf.push_back(ps[x].first);
                pdf_slot[(size_t)g * D + ps[x].first] = local++;
            }
            slot_pos[s0 + ps[x].second] = (int)(slot_states.size() - (size_t)slot_sptr[slot_off[g]]);
            slot_states.push_back(ps[x].second);
        }
        slot_sptr.push_back((int)slot_states.size());
        slot_off[g + 1] = slot_off[g] + local;
        gr.pm.U_max = std::max(gr.pm.U_max, local);
        for (int x = slot_off[g]; x < slot_off[g + 1]; ++x)
            gr.pm.spp_max = std::max(gr.pm.spp_max, slot_sptr[x + 1] - slot_sptr[x]);
        // literal batch matrix rows: in-arcs of every state, then the phony state's row
        lit_row_off[g] = (int)lit_ptr.size() - 1;
        for (int j = 0; j < K; ++j) {
            for (int a2 = in.ptr[j]; a2 < in.ptr[j + 1]; ++a2) { lit_src.push_back(in.other[a2]); lit_w.push_back(in.w[a2]); }
            lit_ptr.push_back((int)lit_src.size());
        }
        for (int k = 0; k < K; ++k)
            if (!(std::isinf(log_final[s0 + k]) && log_final[s0 + k] < 0)) {
                lit_src.push_back(k);
                lit_w.push_back(log_final[s0 + k]);
            }
        lit_src.push_back(K);
        lit_w.push_back(0.0);
        lit_ptr.push_back((int)lit_src.size());
        lit_inst[g + 1] = lit_inst[g] + K + 1;
        // out-arc lists of the same augmented block (backward pass, Eq. (14)): state
        // s → its successors, then s → phony weighted ω(s); phony → phony (1̄)
        for (int i = 0; i < K; ++i) {
            for (int a2 = outl.ptr[i]; a2 < outl.ptr[i + 1]; ++a2) {
                lit_odst.push_back(outl.other[a2]);
                lit_ow.push_back(outl.w[a2]);
            }
            if (!(std::isinf(log_final[s0 + i]) && log_final[s0 + i] < 0)) {
                lit_odst.push_back(K);
                lit_ow.push_back(log_final[s0 + i]);
            }
            lit_optr.push_back((int)lit_odst.size());
        }
        lit_odst.push_back(K);
        lit_ow.push_back(0.0);
        lit_optr.push_back((int)lit_odst.size());
        if (G == 1) { in0 = std::move(in); out0 = std::move(outl); }
    }
    gr.fwd.bytes_max = hf.bytes_max; gr.fwd.slots_max = hf.slots_max;
    gr.bwd.bytes_max = hb.bytes_max; gr.bwd.slots_max = hb.slots_max;
    gr.vit.bytes_max = hv.bytes_max; gr.vit.slots_max = hv.slots_max;
    // Viterbi schedules that exceed one SM's shared memory (the paper's 50,984-arc
    // denominator, N2) stay in global memory and are streamed through L2 each frame
    gr.vit_ok = vit_ok;
    gr.vit_global = vit_ok && viterbi_smem_bytes(gr) > (size_t)kSmemLimit;
    if (!gr.vit_ok) hv = HostSched();
    gr.pm.U_tot = slot_off[G];
    // cluster plan (k_fbc) for a shared factored graph: the first (C, S) that fits
    // shared memory, C CTAs per cluster, S sequences per cluster
    HostCPlan hcp;
    bool cp_ok = false;
    // one-CTA-per-sequence kernels: schedule, state arrays and i16 pdf maps in shared memory
    gr.legacy_ok = !(gr.pm.U_max >= 32768 || (long long)D * 2 > 65536 || smem_bytes(gr, false, false) > (size_t)kSmemLimit ||
                     smem_bytes(gr, true, true) + std::max(pdf_region(POST_GRAD, gr.pm.U_max, D).bytes,
                                                           pdf_region(POST_PDF_COMPACT, gr.pm.U_max, D).bytes) >
                         (size_t)kSmemLimit);
    const bool want_cluster = (flags & FB_GRAPH_CLUSTER) || std::getenv("FBX_CLUSTER") || !gr.legacy_ok;
    if (G == 1 && gr.mode == MODE_FACTORED && want_cluster) {
        // (C, S, no-p): single-wave shapes for B = 128 first ((2,2), (4,4): 128 CTAs), then wider clusters
        struct Cand { int C, S, nop; };
        std::vector<Cand> cand = {{2, 2, 0}, {4, 4, 0}, {4, 4, 1}, {4, 2, 0}, {8, 2, 0}, {8, 4, 0}, {8, 4, 1}};
        if (const char *e = std::getenv("FBX_CLUSTER")) {
            int c = 0, sq = 0, np = 0;
            if (std::sscanf(e, "%d,%d,%d", &c, &sq, &np) >= 2) cand = {{c, sq, np}};
        }
        for (auto cs : cand) {
            if (cs.C < 2 || cs.C > 8 || !(cs.S == 2 || cs.S == 4) || (cs.nop && cs.S != 4)) continue;
            const char *le = std::getenv("FBX_CLUSTER_LMAX");
            if (build_cluster_plan(in0, out0, K_tot, D, pdf, dist_fin, dist_start, init2, final2, cs.C, cs.S,
                                   le ? std::max(1, std::atoi(le)) : 32, hcp,  // N2 step: 12 -> 24 -> 32: 9.70 -> 9.55 -> 8.95 ms (48: 9.23)
                                   0, cs.nop != 0)) { cp_ok = true; break; }
        }
    }
    gr.pm.U_tot = slot_off[G];
    for (int i = 0; i < K_tot; ++i) {
        if (dist_fin[i] > 0) gr.mask_fwd = 1;
        if (dist_start[i] > 0) gr.mask_bwd = 1;
    }
    // index words hold byte offsets relative to the gathered array (p in factored
    // mode, u in exact mode), which the kernel addresses as [offset + base]
    if (!gr.legacy_ok && !cp_ok) return FB_ERR_UNSUPPORTED;

    // pack and upload
    Packer pk;
    std::vector<int> soff(state_offsets, state_offsets + G + 1);
    size_t o_soff = pk.put(soff), o_pdf = pk.put(pdf), o_i2 = pk.put(init2), o_f2 = pk.put(final2);
    size_t o_df = pk.put(dist_fin), o_ds = pk.put(dist_start);
    std::vector<int> morder(G);
    std::iota(morder.begin(), morder.end(), 0);
    std::stable_sort(morder.begin(), morder.end(), [&](int x, int y) {
        return row_ptr[state_offsets[x + 1]] - row_ptr[state_offsets[x]] > row_ptr[state_offsets[y + 1]] - row_ptr[state_offsets[y]];
    });
    size_t o_mo = pk.put(morder);
    std::vector<float> init_nat(log_init, log_init + K_tot), final_nat(log_final, log_final + K_tot);
    size_t o_in = pk.put(init_nat), o_fn = pk.put(final_nat);
    struct SO { size_t rec, rb, ro, wo, wn, wn0; };
    auto put_sched = [&](HostSched &h) {
        SO o;
        o.rec = pk.put(h.blob); o.rb = pk.put(h.rec_bytes); o.ro = pk.put(h.rec_off); o.wo = pk.put(h.warp_off);
        o.wn = pk.put(h.warp_nsl);
        o.wn0 = pk.put(h.warp_nsl0);
        return o;
    };
    SO of = put_sched(hf), ob = put_sched(hb), ov = put_sched(hv);
    size_t o_lro = pk.put(lit_row_off), o_lp = pk.put(lit_ptr), o_ls = pk.put(lit_src), o_lw = pk.put(lit_w),
           o_li = pk.put(lit_inst), o_lop = pk.put(lit_optr), o_lod = pk.put(lit_odst), o_low = pk.put(lit_ow);
    SO ocf{}, ocb{};
    size_t o_cpo = 0, o_cpl = 0, o_cpe = 0, o_cpd = 0, o_cdf = 0, o_cds = 0, o_ci2 = 0, o_cf2 = 0, o_cpq = 0,
           o_fp = 0, o_fs = 0, o_fw = 0, o_bp = 0, o_bs = 0, o_bw = 0;
    if (cp_ok) {
        ocf = put_sched(hcp.hf); ocb = put_sched(hcp.hb);
        o_cpo = pk.put(hcp.part_off); o_cpl = pk.put(hcp.pdf_lo); o_cpe = pk.put(hcp.perm); o_cpd = pk.put(hcp.ipdf);
        o_cdf = pk.put(hcp.idf); o_cds = pk.put(hcp.ids); o_ci2 = pk.put(hcp.ii2); o_cf2 = pk.put(hcp.if2);
        o_cpq = pk.put(hcp.pq);
        o_fp = pk.put(hcp.fptr); o_fs = pk.put(hcp.fsrc); o_fw = pk.put(hcp.fw2);
        o_bp = pk.put(hcp.bptr); o_bs = pk.put(hcp.bsrc); o_bw = pk.put(hcp.bw2);
        CPlan &c = gr.cp;
        c.ok = 1; c.C = hcp.C; c.S = hcp.S; c.T = hcp.T; c.spt = hcp.spt; c.K_int = hcp.K_int;
        c.Kc_max = hcp.Kc_max; c.Dc_max = hcp.Dc_max; c.emis16 = hcp.emis16; c.nop = hcp.nop; c.split = hcp.split;
        c.fwd.bytes_max = hcp.hf.bytes_max; c.fwd.slots_max = hcp.hf.slots_max;
        c.bwd.bytes_max = hcp.hb.bytes_max; c.bwd.slots_max = hcp.hb.slots_max;
    }
    size_t o_ctr = pk.put(std::vector<unsigned long long>(2, 0ull));
    size_t o_so = pk.put(slot_off), o_spd = pk.put(slot_pdf), o_ssp = pk.put(slot_sptr),
           o_sst = pk.put(slot_states), o_pds = pk.put(pdf_slot), o_spo = pk.put(slot_pos);
    if (flags & FB_GRAPH_DRY_RUN) {
        fb_graph h = new (std::nothrow) fb_graph_s;
        if (!h) return FB_ERR_NOMEM;
        gr.dry = true;
        gr.block_bytes = pk.buf.size();
        h->g = gr;
        auto meta = [&](HostSched &hs) {
            std::vector<int> m;
            for (int g2 = 0; g2 < G; ++g2) { m.push_back((int)hs.rec_off[g2]); m.push_back(hs.rec_bytes[g2]); }
            for (size_t w = 0; w < hs.warp_off.size(); ++w) { m.push_back(hs.warp_off[w]); m.push_back(hs.warp_nsl[w]); }
            return m;
        };
        h->host_fwd = hf.blob; h->host_bwd = hb.blob;
        h->host_fwd_meta = meta(hf); h->host_bwd_meta = meta(hb);
        *out = h;
        return FB_OK;
    }
    void *dev = nullptr;
    cudaGetDevice(&gr.device);
    cudaError_t e = cudaMalloc(&dev, pk.buf.size());
    if (e != cudaSuccess) { set_cuda_error("cudaMalloc(graph)", (int)e); return FB_ERR_NOMEM; }
    e = cudaMemcpy(dev, pk.buf.data(), pk.buf.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { cudaFree(dev); set_cuda_error("cudaMemcpy(graph)", (int)e); return FB_ERR_CUDA; }
    auto P = [&](size_t off) { return (const void *)((const unsigned char *)dev + off); };
    gr.block = dev;
    gr.block_bytes = pk.buf.size();
    gr.state_off = (const int *)P(o_soff);
    gr.pdf = (const int *)P(o_pdf);
    gr.init2 = (const float *)P(o_i2);
    gr.final2 = (const float *)P(o_f2);
    gr.dist_fin = (const int *)P(o_df);
    gr.dist_start = (const int *)P(o_ds);
    gr.morder = (const int *)P(o_mo);
    gr.init_nat = (const float *)P(o_in);
    gr.final_nat = (const float *)P(o_fn);
    auto set_sched = [&](Sched &d, const SO &o) {
        d.rec = (const unsigned char *)P(o.rec); d.rec_bytes = (const int *)P(o.rb);
        d.rec_off = (const long long *)P(o.ro); d.warp_off = (const int *)P(o.wo); d.warp_nsl = (const int *)P(o.wn);
        d.warp_nsl0 = (const int *)P(o.wn0);
    };
    set_sched(gr.fwd, of);
    set_sched(gr.bwd, ob);
    set_sched(gr.vit, ov);
    gr.lit.row_off = (const int *)P(o_lro); gr.lit.ptr = (const int *)P(o_lp); gr.lit.src = (const int *)P(o_ls);
    gr.lit.w = (const double *)P(o_lw); gr.lit.inst_off = (const int *)P(o_li);
    gr.lit.optr = (const int *)P(o_lop); gr.lit.odst = (const int *)P(o_lod); gr.lit.ow = (const double *)P(o_low);
    gr.lit.g1 = G == 1; gr.lit.K1 = gr.K_max + 1; gr.lit.inst_total = lit_inst[G];
    if (cp_ok) {
        CPlan &c = gr.cp;
        set_sched(c.fwd, ocf);
        set_sched(c.bwd, ocb);
        c.part_off = (const int *)P(o_cpo); c.pdf_lo = (const int *)P(o_cpl); c.perm = (const int *)P(o_cpe);
        c.ipdf = (const int *)P(o_cpd); c.idist_fin = (const int *)P(o_cdf); c.idist_start = (const int *)P(o_cds);
        c.iinit2 = (const float *)P(o_ci2); c.ifinal2 = (const float *)P(o_cf2); c.pq = (const unsigned *)P(o_cpq);
        c.fptr = (const int *)P(o_fp); c.fsrc = (const int *)P(o_fs); c.fw2 = (const float *)P(o_fw);
        c.bptr = (const int *)P(o_bp); c.bsrc = (const int *)P(o_bs); c.bw2 = (const float *)P(o_bw);
    }
    gr.ctr = (unsigned long long *)P(o_ctr);
    gr.pm.slot_off = (const int *)P(o_so); gr.pm.slot_pdf = (const int *)P(o_spd);
    gr.pm.slot_sptr = (const int *)P(o_ssp); gr.pm.slot_states = (const int *)P(o_sst);
    gr.pm.pdf_slot = (const int *)P(o_pds);
    gr.pm.slot_pos = (const int *)P(o_spo);
    fb_graph h = new (std::nothrow) fb_graph_s;
    if (!h) { cudaFree(dev); return FB_ERR_NOMEM; }
    h->g = gr;
    *out = h;
    return FB_OK;
}

extern "C" fb_status fb_graph_destroy(fb_graph g) {
    if (!g) return FB_OK;
    if (g->perm) fb_graph_destroy(g->perm);
    if (!g->g.dry) {
        cudaDeviceSynchronize();
        cudaFree(g->g.block);
    }
    delete g;
    return FB_OK;
}

extern "C" fb_status fb_graph_info(fb_graph h, int64_t *out) {
    if (!h || !out) return FB_ERR_INVALID_ARG;
    const Graph &g = h->g;
    int64_t v[16] = {g.G, g.K_tot, g.nnz, g.D, g.T, g.spt, g.mode,
                     (int64_t)smem_bytes(g, false, false), (int64_t)smem_bytes(g, true, true),
                     g.K_max, g.nnz_max, g.fwd.slots_max, g.bwd.slots_max, g.pm.U_max,
                     g.cp.ok ? g.cp.C : 0, g.cp.ok ? g.cp.S : 0};
    std::memcpy(out, v, sizeof v);
    return FB_OK;
}

extern "C" fb_status fb_graph_counters(fb_graph h, int64_t *out, int32_t reset) {
    if (!h || !out || h->g.dry) return FB_ERR_INVALID_ARG;
    // the handle's counters plus its relabelled twin's (lfmmi_loss_grad runs on the twin)
    out[0] = out[1] = 0;
    for (fb_graph x = h; x; x = x->perm) {
        unsigned long long v[2] = {0, 0};
        cudaError_t e = cudaMemcpy(v, x->g.ctr, sizeof v, cudaMemcpyDeviceToHost);  // synchronizes the device
        if (e != cudaSuccess) { set_cuda_error("fb_graph_counters", (int)e); return FB_ERR_CUDA; }
        out[0] += (int64_t)v[0];
        out[1] += (int64_t)v[1];
        if (reset) {
            e = cudaMemset(x->g.ctr, 0, sizeof v);
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { set_cuda_error("fb_graph_counters", (int)e); return FB_ERR_CUDA; }
        }
    }
    return FB_OK;
}

// Internal (not part of fb.h): copy a dry-run handle's compiled schedule to the
// caller for host-side verification.  which = 0 forward, 1 backward.
// Returns the number of bytes (blob) / ints (meta) available when buffers are NULL.
extern "C" long long fbx_debug_schedule(fb_graph h, int which, unsigned char *blob, int *meta) {
    if (!h || !h->g.dry) return -1;
    const auto &b = which ? h->host_bwd : h->host_fwd;
    const auto &m = which ? h->host_bwd_meta : h->host_fwd_meta;
    if (blob) std::memcpy(blob, b.data(), b.size());
    if (meta) std::memcpy(meta, m.data(), m.size() * sizeof(int));
    return blob ? (long long)b.size() : (meta ? (long long)m.size() : (long long)b.size() * 0 + (long long)b.size());
}

extern "C" long long fbx_debug_schedule_meta_len(fb_graph h, int which) {
    if (!h || !h->g.dry) return -1;
    return (long long)(which ? h->host_bwd_meta.size() : h->host_fwd_meta.size());
}
