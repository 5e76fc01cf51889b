"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This module draws graphs and emission tensors; it holds NONE of the method's
arithmetic (no forward/backward recursion, no path sums, no posteriors).  The
only arithmetic here is input construction: per-source normalisation of random
arc weights and a log-softmax of random logits for the "peaky" emission
variant.  Every array is produced in float32 from a
``numpy.random.Generator(PCG64(seed))`` so that the CUDA path and the float64
oracle read bit-identical inputs.

Graph convention (ledger L3 in DESIGN.md): T is stored as
CSR with row = source state i, column = destination state j, value
T_ij = log p(z_n = j | z_{n-1} = i).  An absent entry is 0̄ = -inf.

Workload recipes are those of SURVEY.md §8(d) (C1..C5 and the paper shape of
Table 1); DESIGN.md §"Input recipe" restates them.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np


@dataclass
class HostGraph:
    """One weighted automaton (T, π, ω) plus its state→pdf map (ledger L9)."""

    K: int
    row_ptr: np.ndarray  # int32 [K+1]
    col: np.ndarray  # int32 [nnz]   destination state
    logw: np.ndarray  # float32 [nnz] log arc weight T_ij (-inf allowed)
    log_init: np.ndarray  # float32 [K]  π
    log_final: np.ndarray  # float32 [K] ω
    pdf_of: np.ndarray  # int32 [K]    emission column of each state
    D: int  # number of emission columns

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def arcs(self):
        """(src, dst, logw) arrays in CSR order."""
        src = np.repeat(np.arange(self.K, dtype=np.int32), np.diff(self.row_ptr))
        return src, self.col, self.logw


def graph_from_arcs(K, src, dst, logw, log_init, log_final, pdf_of=None, D=None) -> HostGraph:
    """Build a CSR HostGraph from an arc list (stable sort by source, then destination)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    logw = np.asarray(logw, dtype=np.float32)
    if src.size:
        assert src.min() >= 0 and src.max() < K and dst.min() >= 0 and dst.max() < K
    order = np.lexsort((dst, src))
    src, dst, logw = src[order], dst[order], logw[order]
    row_ptr = np.zeros(K + 1, dtype=np.int32)
    np.add.at(row_ptr, src + 1, 1)
    row_ptr = np.cumsum(row_ptr).astype(np.int32)
    if pdf_of is None:
        pdf_of = np.arange(K, dtype=np.int32)
        D = K if D is None else D
    pdf_of = np.asarray(pdf_of, dtype=np.int32)
    assert D is not None and pdf_of.max(initial=0) < D
    return HostGraph(
        K=int(K),
        row_ptr=row_ptr,
        col=dst.astype(np.int32),
        logw=logw,
        log_init=np.asarray(log_init, dtype=np.float32),
        log_final=np.asarray(log_final, dtype=np.float32),
        pdf_of=pdf_of,
        D=int(D),
    )


@dataclass
class ComposedGraph:
    """G graphs concatenated block-diagonally: global state ids.

    Graph g owns states [state_offsets[g], state_offsets[g+1]) and only arcs
    inside that block.  This is the layout ``fb_graph_create`` consumes.
    """

    G: int
    state_offsets: np.ndarray  # int32 [G+1]
    row_ptr: np.ndarray  # int32 [K_tot+1]
    col: np.ndarray  # int32 [nnz], global ids
    logw: np.ndarray
    log_init: np.ndarray
    log_final: np.ndarray
    pdf_of: np.ndarray
    D: int
    members: List[HostGraph] = field(default_factory=list)

    @property
    def K_tot(self) -> int:
        return int(self.state_offsets[-1])

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])


def compose(graphs: List[HostGraph]) -> ComposedGraph:
    """Block-diagonal concatenation of member graphs."""
    assert len(graphs) >= 1
    D = graphs[0].D
    assert all(g.D == D for g in graphs)
    offs = np.zeros(len(graphs) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([g.K for g in graphs])
    aoffs = np.zeros(len(graphs) + 1, dtype=np.int64)
    aoffs[1:] = np.cumsum([g.nnz for g in graphs])
    row_ptr = np.concatenate(
        [g.row_ptr[:-1].astype(np.int64) + aoffs[i] for i, g in enumerate(graphs)] + [np.array([aoffs[-1]])]
    ).astype(np.int32)
    col = np.concatenate([g.col.astype(np.int64) + offs[i] for i, g in enumerate(graphs)]).astype(np.int32)
    return ComposedGraph(
        G=len(graphs),
        state_offsets=offs.astype(np.int32),
        row_ptr=row_ptr,
        col=col,
        logw=np.concatenate([g.logw for g in graphs]).astype(np.float32),
        log_init=np.concatenate([g.log_init for g in graphs]).astype(np.float32),
        log_final=np.concatenate([g.log_final for g in graphs]).astype(np.float32),
        pdf_of=np.concatenate([g.pdf_of for g in graphs]).astype(np.int32),
        D=D,
        members=list(graphs),
    )


# --------------------------------------------------------------------------- weights

def _uniform_open_low(rng, lo, size):
    """U(lo, 1] in float64."""
    return 1.0 - rng.random(size) * (1.0 - lo)


def _normalise_per_source(src, raw, K):
    """log(raw / Σ_{arcs from the same source} raw), float64 → float32."""
    tot = np.zeros(K, dtype=np.float64)
    np.add.at(tot, src, raw)
    return (np.log(raw) - np.log(tot[src])).astype(np.float32)


# --------------------------------------------------------------------------- graphs

def dense_graph(rng, K=3) -> HostGraph:
    """C1: dense K-state graph, rows = log Dirichlet(1), π = log Dirichlet(1), ω ≡ 0, identity map."""
    src, dst = np.meshgrid(np.arange(K), np.arange(K), indexing="ij")
    rows = rng.dirichlet(np.ones(K), size=K)
    logw = np.log(rows).astype(np.float32).ravel()
    pi = np.log(rng.dirichlet(np.ones(K))).astype(np.float32)
    return graph_from_arcs(K, src.ravel(), dst.ravel(), logw, pi, np.zeros(K, np.float32))


def random_small_graph(rng, K=None, max_K=6, D=None, p_arc=0.45, p_neg_inf=0.1, p_dup=0.1,
                       weighted_ends=True) -> HostGraph:
    """Tiny irregular graph for brute-force pins: sparse arcs, explicit -inf arcs,
    duplicate arcs, partially -inf π/ω, optional many-to-one pdf map."""
    if K is None:
        K = int(rng.integers(1, max_K + 1))
    src, dst, w = [], [], []
    for i in range(K):
        for j in range(K):
            if rng.random() < p_arc or (j == (i + 1) % K):
                src.append(i); dst.append(j)
                w.append(-np.inf if rng.random() < p_neg_inf else float(rng.normal(-1.0, 1.0)))
                if rng.random() < p_dup:
                    src.append(i); dst.append(j); w.append(float(rng.normal(-1.0, 1.0)))
    if weighted_ends:
        pi = rng.normal(-1.0, 1.0, K)
        om = rng.normal(-0.5, 1.0, K)
        pi[rng.random(K) < 0.3] = -np.inf
        om[rng.random(K) < 0.3] = -np.inf
        pi[int(rng.integers(K))] = float(rng.normal())
        om[int(rng.integers(K))] = float(rng.normal())
    else:
        pi = np.zeros(K); om = np.zeros(K)
    if D is None:
        pdf_of, Dv = None, None
    else:
        Dv = int(D)
        pdf_of = rng.integers(0, Dv, K)
    return graph_from_arcs(K, src, dst, w, pi.astype(np.float32), om.astype(np.float32), pdf_of, Dv)


def numerator_graph(rng, L, D, pdf_mode="identity", alt_p=0.15, k_max=300) -> HostGraph:
    """Left-to-right alignment graph (C2 recipe).

    2 states per phone: a_p (self-loop, -> b_p, -> a_{p+1}) and b_p (self-loop,
    -> a_{p+1}); minimum path = L frames.  Alternative-pronunciation branches
     with probability ``alt_p`` per phone span 2-4 phones in parallel
    with the main chain.  Weights = log U(0.05,1] normalised per source.  π = 1̄
    on a_0, ω = 1̄ on the last phone's two states.
    """
    K = 2 * L
    src, dst = [], []

    def chain(base, nph, entry_from, exit_to, final_list):
        for p in range(nph):
            a, b = base + 2 * p, base + 2 * p + 1
            src.extend([a, a, b]); dst.extend([a, b, b])
            if p + 1 < nph:
                src.extend([a, b]); dst.extend([base + 2 * (p + 1)] * 2)
        for s in entry_from:
            src.append(s); dst.append(base)
        last_a, last_b = base + 2 * (nph - 1), base + 2 * (nph - 1) + 1
        if exit_to is None:
            final_list.extend([last_a, last_b])
        else:
            src.extend([last_a, last_b]); dst.extend([exit_to, exit_to])

    finals: List[int] = []
    initials = [0]
    chain(0, L, [], None, finals)
    p = 0
    while p < L:
        if rng.random() < alt_p:
            m = int(rng.integers(2, 5))
            if p + m <= L and K + 2 * m <= k_max:
                base = K
                K += 2 * m
                entry = [] if p == 0 else [2 * (p - 1), 2 * (p - 1) + 1]
                if p == 0:
                    initials.append(base)
                chain(base, m, entry, None if p + m == L else 2 * (p + m), finals)
                p += m
                continue
        p += 1
    src = np.array(src); dst = np.array(dst)
    raw = _uniform_open_low(rng, 0.05, src.size)
    logw = _normalise_per_source(src, raw, K)
    pi = np.full(K, -np.inf, np.float32); pi[initials] = 0.0
    om = np.full(K, -np.inf, np.float32); om[finals] = 0.0
    if pdf_mode == "identity":
        assert K <= D
        pdf_of = np.arange(K)
    else:
        pdf_of = rng.integers(0, D, K)
    return graph_from_arcs(K, src, dst, logw, pi, om, pdf_of, D)


def denominator_graph(rng, K=3000, nnz=20000, hub_frac=0.02, hub_share=0.30, D=None,
                      pdf_mode="identity") -> HostGraph:
    """Ergodic n-gram-like denominator graph (C3/C4 recipe).

    K self-loops + ring i -> i+1 (reachability and co-reachability) + extra arcs
    with back-off-like skew: ``hub_frac`` of states take ``hub_share`` of the
    extra arcs as sources and (independently) as destinations.  Rows = log
    U(0.001,1] normalised per source; π = -log K; ω ≡ 1̄.
    """
    n_extra = nnz - 2 * K
    assert n_extra >= 0
    hubs = rng.choice(K, size=max(1, int(round(hub_frac * K))), replace=False)
    existing = set((i * K + i) for i in range(K)) | set((i * K + (i + 1) % K) for i in range(K))
    es, ed = [], []
    while len(es) < n_extra:
        m = (n_extra - len(es)) * 2
        s = np.where(rng.random(m) < hub_share, rng.choice(hubs, m), rng.integers(0, K, m))
        d = np.where(rng.random(m) < hub_share, rng.choice(hubs, m), rng.integers(0, K, m))
        for a, b in zip(s.tolist(), d.tolist()):
            key = a * K + b
            if key in existing:
                continue
            existing.add(key)
            es.append(a); ed.append(b)
            if len(es) == n_extra:
                break
    ar = np.arange(K)
    src = np.concatenate([ar, ar, np.array(es, dtype=np.int64)])
    dst = np.concatenate([ar, (ar + 1) % K, np.array(ed, dtype=np.int64)])
    raw = _uniform_open_low(rng, 0.001, src.size)
    logw = _normalise_per_source(src, raw, K)
    pi = np.full(K, -np.log(K), np.float32)
    om = np.zeros(K, np.float32)
    if pdf_mode == "identity":
        D = K if D is None else D
        pdf_of = np.arange(K)
    else:
        assert D is not None and K >= D
        pdf_of = random_surjection(rng, K, D)
    return graph_from_arcs(K, src, dst, logw, pi, om, pdf_of, D)


def random_surjection(rng, K, D) -> np.ndarray:
    """state -> pdf map using every pdf; the K-D extra states reuse distinct pdfs
    (C4: 3000 -> 2000, 1000 pdfs shared by 2 states)."""
    extra = K - D
    pdfs = np.concatenate([np.arange(D), rng.choice(D, size=extra, replace=extra > D)])
    return rng.permutation(pdfs).astype(np.int32)


# --------------------------------------------------------------------------- emissions

def emissions(rng, B, N, D, kind="uniform") -> np.ndarray:
    """φ [B, N, D] float32 read as log p(x_n | pdf).

    kind = "uniform": i.i.d. U[-10, 0) (ledger L15, primary);
    kind = "softmax4"/"softmax8": per-frame log-softmax of N(0, σ²) logits
    (TDNN-like peaky outputs, stress variants).
    """
    if kind == "uniform":
        out = rng.random((B, N, D), dtype=np.float32)
        out *= np.float32(-10.0)
        return out
    sigma = {"softmax4": 4.0, "softmax8": 8.0}[kind]
    z = rng.normal(0.0, sigma, (B, N, D))
    z -= z.max(axis=-1, keepdims=True)
    z -= np.log(np.exp(z).sum(axis=-1, keepdims=True))
    return z.astype(np.float32)


# --------------------------------------------------------------------------- configs

@dataclass
class Workload:
    name: str
    B: int
    N_max: int
    D: int
    lengths: np.ndarray  # int32 [B]
    emis: np.ndarray  # float32 [B, N_max, D]
    den: Optional[HostGraph] = None  # shared graph (G = 1)
    nums: Optional[List[HostGraph]] = None  # one graph per sequence (G = B)

    @property
    def seq_frames(self) -> int:
        return int(self.lengths.sum())


def make_c1(seed: int) -> Workload:
    rng = np.random.Generator(np.random.PCG64(seed))
    g = dense_graph(rng, 3)
    em = emissions(rng, 1, 6, 3)
    return Workload("C1", 1, 6, 3, np.array([6], np.int32), em, den=g)


def make_c2(seed: int = 2, B: int = 64, N_max: int = 180, D: int = 300, kind="uniform") -> Workload:
    rng = np.random.Generator(np.random.PCG64(seed))
    nums, lens = [], []
    for _ in range(B):
        L = int(rng.integers(50, 151))
        g = numerator_graph(rng, L, D, "identity")
        nums.append(g)
        lens.append(int(rng.integers(max(120, L), N_max + 1)))
    em = emissions(rng, B, N_max, D, kind)
    return Workload("C2", B, N_max, D, np.array(lens, np.int32), em, nums=nums)


def make_den(seed: int, K=3000, nnz=20000, D=None, pdf_mode="identity") -> HostGraph:
    rng = np.random.Generator(np.random.PCG64(seed))
    return denominator_graph(rng, K, nnz, D=D, pdf_mode=pdf_mode)


def make_c3(seed: int = 3, B: int = 128, N: int = 500, K: int = 3000, nnz: int = 20000,
            kind="uniform") -> Workload:
    den = make_den(seed, K, nnz)
    rng = np.random.Generator(np.random.PCG64(seed + 1000))
    em = emissions(rng, B, N, den.D, kind)
    return Workload("C3", B, N, den.D, np.full(B, N, np.int32), em, den=den)


def make_c4(seed: int = 4, B: int = 128, N: int = 500, K: int = 3000, nnz: int = 20000,
            D: int = 2000, kind="uniform", lengths=None, L_range=(50, 151)) -> Workload:
    den = make_den(seed, K, nnz, D=D, pdf_mode="surjection")
    rng = np.random.Generator(np.random.PCG64(seed + 1000))
    nums = [numerator_graph(rng, int(rng.integers(*L_range)), D, "random") for _ in range(B)]
    em = emissions(rng, B, N, D, kind)
    lens = np.full(B, N, np.int32) if lengths is None else np.asarray(lengths, np.int32)
    return Workload("C4", B, N, D, lens, em, den=den, nums=nums)


def c5_lengths(seed: int = 5, B: int = 1024) -> np.ndarray:
    """Clipped log-normal, median 250, range [50, 700] (700 = paper max)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = np.exp(rng.normal(np.log(250.0), 0.5, B))
    return np.clip(np.round(n), 50, 700).astype(np.int32)


def make_c5_utterances(seed: int = 5, B: int = 1024, D: int = 2000, K: int = 3000, nnz: int = 20000):
    """C5 pool: lengths, numerator graphs (L_b ~ U[N_b/3, N_b/2]) and the shared C4 den.
    Emissions are drawn per shard by ``c5_emissions`` so each rank draws only its own."""
    lens = c5_lengths(seed, B)
    rng = np.random.Generator(np.random.PCG64(seed + 1000))
    nums = [numerator_graph(rng, int(rng.integers(max(1, n // 3), max(2, n // 2) + 1)), D, "random",
                            k_max=10 ** 9) for n in lens.tolist()]
    den = make_den(4, K, nnz, D=D, pdf_mode="surjection")
    return lens, nums, den


def c5_emissions(seed: int, idx: np.ndarray, N_max: int, D: int) -> np.ndarray:
    """Per-utterance emissions for the C5 pool: utterance u draws from PCG64(seed, u)."""
    out = np.empty((len(idx), N_max, D), np.float32)
    for r, u in enumerate(np.asarray(idx).tolist()):
        rng = np.random.Generator(np.random.PCG64([seed, int(u)]))
        out[r] = emissions(rng, 1, N_max, D)[0]
    return out


def make_paper_shape(seed: int = 6, B: int = 128, N: int = 700, L_range=(190, 211)) -> Workload:
    """N2, the paper's Table 1 shape: den 3022 states / 50,984 arcs with
    a pdf surjection onto D = 84 outputs; B numerator graphs of ≈454 states / ≈1036
    arcs (C2 recipe with L ~ U[190, 210] phones, capped at 454 states); all N_b = N."""
    rng = np.random.Generator(np.random.PCG64(seed))
    den = denominator_graph(rng, 3022, 50984, D=84, pdf_mode="surjection")
    nums = [numerator_graph(rng, int(rng.integers(*L_range)), 84, "random", k_max=454) for _ in range(B)]
    em = emissions(rng, B, N, 84)
    return Workload("N2", B, N, 84, np.full(B, N, np.int32), em, den=den, nums=nums)
