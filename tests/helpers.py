"""Small test-only graph constructions (no method arithmetic).

These build graphs whose answers are fixed by closed forms or by library
routines: the 1-state chain, the symmetric 2-state graph, the CTC topology
(blank shared ⇒ a many-to-one pdf map), the paper's phony final state
(ledger L8) and a left-to-right chain for the stability test.
"""
from __future__ import annotations

import numpy as np

from paper_2112_00709_b200.synth import HostGraph, graph_from_arcs


def one_state(t=0.0, pi=0.0, om=0.0) -> HostGraph:
    return graph_from_arcs(1, [0], [0], [t], [pi], [om])


def symmetric_two_state() -> HostGraph:
    w = np.log(0.5)
    return graph_from_arcs(2, [0, 0, 1, 1], [0, 1, 0, 1], [w] * 4, [w, w], [0.0, 0.0])


def ctc_topology(labels, C) -> HostGraph:
    """CTC as a weighted automaton: states (blank, l1, blank, l2, …, blank),
    self-loops, s→s+1, s→s+2 when l_{s+2} ≠ l_s; all weights 1̄; start in the
    first blank or first label; finish in the last label or last blank.
    pdf_of = 0 (blank) for blank states, the label for label states."""
    ext = [0]
    for l in labels:
        ext += [int(l), 0]
    S = len(ext)
    src, dst = [], []
    for s in range(S):
        src.append(s); dst.append(s)
        if s + 1 < S:
            src.append(s); dst.append(s + 1)
        if s + 2 < S and ext[s + 2] != 0 and ext[s + 2] != ext[s]:
            src.append(s); dst.append(s + 2)
    pi = np.full(S, -np.inf); pi[0] = 0.0; pi[1] = 0.0
    om = np.full(S, -np.inf); om[S - 1] = 0.0; om[S - 2] = 0.0
    return graph_from_arcs(S, src, dst, np.zeros(len(src)), pi, om, np.array(ext), C)


def add_phony_final(g: HostGraph) -> HostGraph:
    """P:224-227 / SPEC S:270-276: a phony state with a 1̄ self-loop; an arc
    s→phony weighted ω(s) for every final s; new ω = 1̄ on the phony state only.
    The phony state emits through an extra pdf column D (so D' = D + 1)."""
    src, dst, w = g.arcs()
    K = g.K
    fin = np.flatnonzero(g.log_final != -np.inf)
    src = np.concatenate([src, fin, [K]])
    dst = np.concatenate([dst, np.full(fin.size, K), [K]])
    w = np.concatenate([w, g.log_final[fin], [0.0]])
    pi = np.concatenate([g.log_init, [-np.inf]])
    om = np.full(K + 1, -np.inf); om[K] = 0.0
    pdf = np.concatenate([g.pdf_of, [g.D]])
    return graph_from_arcs(K + 1, src, dst, w, pi, om, pdf, g.D + 1)


def pad_for_phony(emis, N_b, N_pad):
    """v(phony) = 0̄ for n < N_b and 1̄ after; real pdfs get 0̄ after N_b (ledger L8)."""
    N, D = emis.shape
    out = np.full((N_pad, D + 1), -np.inf)
    out[:N_b, :D] = emis[:N_b]
    out[N_b:, D] = 0.0
    return out


def left_to_right(K, stay=np.log(0.5)) -> HostGraph:
    src, dst, w = [], [], []
    for i in range(K):
        src.append(i); dst.append(i); w.append(stay if i + 1 < K else 0.0)
        if i + 1 < K:
            src.append(i); dst.append(i + 1); w.append(np.log(1 - np.exp(stay)))
    pi = np.full(K, -np.inf); pi[0] = 0.0
    om = np.full(K, -np.inf); om[K - 1] = 0.0
    return graph_from_arcs(K, src, dst, w, pi, om)


def relabel(g: HostGraph, perm) -> HostGraph:
    """State k → perm[k] (pdfs travel with their states)."""
    perm = np.asarray(perm)
    src, dst, w = g.arcs()
    pi = np.empty(g.K, np.float32); om = np.empty(g.K, np.float32); pdf = np.empty(g.K, np.int32)
    pi[perm] = g.log_init; om[perm] = g.log_final; pdf[perm] = g.pdf_of
    return graph_from_arcs(g.K, perm[src], perm[dst], w, pi, om, pdf, g.D)
