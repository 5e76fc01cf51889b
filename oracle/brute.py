"""Brute-force path enumeration — TEST INFRASTRUCTURE ONLY (pins the oracle).

The definition the method reaches exactly:

    logZ = log Σ_{z ∈ [K]^N} exp( π(z_0) + Σ_n v_n(z_n) + Σ_{n≥1} T(z_{n-1}, z_n) + ω(z_{N-1}) )
    γ_n(k) = Σ_{z : z_n = k} exp(score(z) − logZ)

with v_n(k) = φ[n, pdf_of[k]] (ledger L9) and duplicate arcs
combined with ⊕.  No recursion: every one of the K^N state sequences is
scored independently, so this shares no structure with oracle.c.

``brute_force`` sums with ``math.fsum`` (exactly rounded) over float64 path
scores; ``brute_force_mp`` scores and sums in mpmath at 50 digits (C1-sized
inputs only).  Guard: K^N ≤ 2e6.
"""
from __future__ import annotations

import itertools
import math

import numpy as np


def dense_T(g, semiring="log"):
    """K×K log-weight matrix with −∞ for absent arcs; duplicates ⊕-combined
    (log: logaddexp; tropical: max)."""
    K = g.K
    T = np.full((K, K), -np.inf)
    src = np.repeat(np.arange(K), np.diff(np.asarray(g.row_ptr)))
    for i, j, w in zip(src.tolist(), np.asarray(g.col).tolist(), np.asarray(g.logw, np.float64).tolist()):
        if T[i, j] == -np.inf:
            T[i, j] = w
        elif w != -np.inf and semiring == "tropical":
            T[i, j] = max(T[i, j], w)
        elif w != -np.inf:
            m = max(T[i, j], w)
            T[i, j] = m + math.log(math.exp(T[i, j] - m) + math.exp(w - m))
    return T


def _paths(K, N):
    if K ** N > 2_000_000:
        raise ValueError("brute force guard: K^N > 2e6")
    return np.array(list(itertools.product(range(K), repeat=N)), dtype=np.int64).reshape(-1, N)


def path_scores(g, emis, semiring="log"):
    """float64 score of every state sequence; emis is [N, D] (one sequence)."""
    emis = np.asarray(emis, np.float64)
    N = emis.shape[0]
    K = g.K
    T = dense_T(g, semiring)
    Z = _paths(K, N)
    pdf = np.asarray(g.pdf_of)
    s = np.asarray(g.log_init, np.float64)[Z[:, 0]] + np.asarray(g.log_final, np.float64)[Z[:, -1]]
    for n in range(N):
        s = s + emis[n, pdf[Z[:, n]]]
    for n in range(1, N):
        s = s + T[Z[:, n - 1], Z[:, n]]
    return Z, s


def brute_force(g, emis):
    """(logZ, γ [N,K], Γ [N,D], best_score, best_path) by enumerating all K^N paths."""
    Z, s = path_scores(g, emis)
    N = Z.shape[1]
    K = g.K
    D = g.D
    m = s.max()
    if m == -np.inf:
        return -np.inf, np.zeros((N, K)), np.zeros((N, D)), -np.inf, None
    e = np.exp(s - m)
    logZ = m + math.log(math.fsum(e.tolist()))
    p = np.exp(s - logZ)
    gam = np.zeros((N, K))
    for n in range(N):
        for k in range(K):
            sel = p[Z[:, n] == k]
            gam[n, k] = math.fsum(sel.tolist())
    Gam = np.zeros((N, D))
    pdf = np.asarray(g.pdf_of)
    for k in range(K):
        Gam[:, pdf[k]] += gam[:, k]
    # Viterbi: max score; ties → lowest final state, then lowest predecessor at each
    # step back (the DP tie-break read as "lowest index at every argmax").
    Z, s = path_scores(g, emis, "tropical")
    best = s.max()
    idx = np.flatnonzero(s == best)
    cands = Z[idx][:, ::-1]
    order = np.lexsort(cands.T[::-1])
    best_path = cands[order[0]][::-1].copy()
    return logZ, gam, Gam, best, best_path


def brute_force_mp(g, emis, dps=50):
    """logZ and γ with every path scored and summed in mpmath (C1-sized inputs)."""
    import mpmath as mp

    mp.mp.dps = dps
    emis = np.asarray(emis, np.float64)
    N = emis.shape[0]
    K = g.K
    T = dense_T(g)
    pdf = np.asarray(g.pdf_of)
    pi = np.asarray(g.log_init, np.float64)
    om = np.asarray(g.log_final, np.float64)
    terms = []
    paths = []
    for z in itertools.product(range(K), repeat=N):
        parts = [pi[z[0]], om[z[-1]]] + [emis[n, pdf[z[n]]] for n in range(N)] + [T[z[n - 1], z[n]] for n in range(1, N)]
        if any(x == -np.inf for x in parts):
            continue
        sc = mp.fsum([mp.mpf(float(x)) for x in parts])
        terms.append(mp.exp(sc))
        paths.append(z)
    tot = mp.fsum(terms)
    logZ = mp.log(tot)
    gam = np.zeros((N, K))
    for n in range(N):
        acc = [mp.mpf(0)] * K
        for z, t in zip(paths, terms):
            acc[z[n]] += t
        for k in range(K):
            gam[n, k] = float(acc[k] / tot)
    return float(logZ), gam
