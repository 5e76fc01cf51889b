"""T0: pin the float64 oracle to things other than itself.

Pins used (each chosen so a dropped term, wrong sign/index or transposed
operand in oracle.c fails at least one):
  * brute-force enumeration of all K^N paths (oracle/brute.py; mpmath for C1)
  * torch.nn.functional.ctc_loss on a CTC topology (many-to-one pdf map)
  * central finite differences of the LF-MMI loss
  * closed forms (1-state chain, symmetric 2-state, num = den, 1-state num/den)
  * invariants (Σγ = 1, α·β consistency, Σ grad = 0, relabelling, shifts)
  * the paper's phony-state batching vs per-length recursion
  * probability-domain matrix recursion Eq. (4)-(5) via numpy matmul
  * stability regression
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import brute
from paper_2112_00709_b200 import synth
from tests import helpers

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def run_fb(g, emis, N=None, **kw):
    emis = np.asarray(emis)
    if emis.ndim == 2:
        emis = emis[None]
    N = emis.shape[1] if N is None else N
    return oracle.fb_batch(g, emis, np.array([N], np.int32), alpha=True, beta=True, post=True,
                           post_pdf=True, **kw)


# ------------------------------------------------------------------ semiring

def test_logaddexp_examples():
    # S:60-63
    assert oracle.logaddexp(-math.inf, 3.0) == 3.0
    assert oracle.logaddexp(0.0, 0.0) == pytest.approx(math.log(2.0), abs=1e-16)
    assert oracle.logaddexp(1e8, 1e8) == pytest.approx(1e8 + math.log(2.0), abs=2e-8)
    assert oracle.logaddexp(-math.inf, -math.inf) == -math.inf
    rng = np.random.default_rng(0)
    for a, b in rng.uniform(-50, 50, (200, 2)):
        assert oracle.logaddexp(a, b) == pytest.approx(np.logaddexp(a, b), abs=1e-13)


# ------------------------------------------------------------------ brute force

def test_golden_c1_mpmath():
    """tests/golden/c1_mp50.json: C1 seeds brute-forced at 50 digits by
    tests/golden/make_golden.py (calls oracle.brute only)."""
    with open(os.path.join(GOLD, "c1_mp50.json")) as f:
        gold = json.load(f)
    for case in gold["cases"]:
        w = synth.make_c1(case["seed"])
        r = run_fb(w.den, w.emis[0])
        assert abs(r["logZ"][0] - case["logZ"]) <= 1e-10
        assert np.abs(r["post"][0] - np.array(case["post"])).max() <= 1e-10


@pytest.mark.parametrize("seed", range(100))
def test_c1_vs_brute(seed):
    w = synth.make_c1(seed)
    r = run_fb(w.den, w.emis[0])
    logZ, gam, Gam, _, _ = brute.brute_force(w.den, w.emis[0])
    assert abs(r["logZ"][0] - logZ) <= 1e-10
    assert abs(r["logZ_beta"][0] - logZ) <= 1e-10
    assert np.abs(r["post"][0] - gam).max() <= 1e-10
    assert np.abs(r["post_pdf"][0] - Gam).max() <= 1e-10


@pytest.mark.parametrize("seed", range(100))
def test_random_small_vs_brute(seed):
    rng = np.random.default_rng(1000 + seed)
    K = int(rng.integers(1, 7))
    D = None if rng.random() < 0.5 else int(rng.integers(1, K + 1))
    g = synth.random_small_graph(rng, K=K, D=D)
    N = int(rng.integers(1, 8))
    while K ** N > 300_000:
        N -= 1
    emis = rng.uniform(-5, 1, (N, g.D)).astype(np.float32)
    r = run_fb(g, emis)
    logZ, gam, Gam, _, _ = brute.brute_force(g, emis)
    if logZ == -math.inf:
        assert r["status"][0] == oracle.ST_EMPTY and r["logZ"][0] == -math.inf
        assert (r["post"][0] == 0).all()
        return
    assert r["status"][0] == 0
    assert abs(r["logZ"][0] - logZ) <= 1e-10 * max(1.0, abs(logZ))
    assert abs(r["logZ_beta"][0] - logZ) <= 1e-10 * max(1.0, abs(logZ))
    assert np.abs(r["post"][0] - gam).max() <= 1e-10
    assert np.abs(r["post_pdf"][0] - Gam).max() <= 1e-10
    # unreachable / dead states carry exactly zero mass
    assert (r["post"][0][gam == 0] == 0).all()


# ------------------------------------------------------------------ closed forms

def test_one_state_chain():
    # S:351
    g = helpers.one_state()
    e = np.array([[-1.0], [-2.0], [-3.0]], np.float32)
    r = run_fb(g, e)
    assert r["alpha"][0, :, 0].tolist() == [-1.0, -3.0, -6.0]
    assert r["beta"][0, :, 0].tolist() == [-5.0, -3.0, 0.0]
    assert r["logZ"][0] == -6.0
    assert (r["post"][0] == 1.0).all()


def test_symmetric_two_state():
    # S:376
    g = helpers.symmetric_two_state()
    rng = np.random.default_rng(3)
    row = rng.uniform(-3, 0, (7, 1)).astype(np.float32)
    e = np.repeat(row, 2, axis=1)
    r = run_fb(g, e)
    assert np.abs(r["post"][0] - 0.5).max() <= 1e-15


def test_shift_all_frames():
    w = synth.make_c1(7)
    r0 = run_fb(w.den, w.emis[0])
    r1 = run_fb(w.den, w.emis[0].astype(np.float64) + 2.5)
    assert r1["logZ"][0] == pytest.approx(r0["logZ"][0] + 6 * 2.5, abs=1e-12)
    assert np.abs(r1["post"] - r0["post"]).max() <= 1e-14


# ------------------------------------------------------------------ library routine: CTC

@pytest.mark.parametrize("seed", range(5))
def test_ctc_pin(seed):
    """CTC topology ⇒ logZ = −ctc_loss (float64) and Γ = exp(lp) − ∂ctc/∂lp
    (torch's CTC gradient assumes log-softmax input).  Pins the many-to-one pdf
    map (ledger L9) against an independent library implementation."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(seed)
    C, U, N = 6, 4, 14
    labels = rng.integers(1, C, U)
    labels[2] = labels[1]  # a repeated label exercises the s→s+2 exclusion
    lp = torch.log_softmax(torch.tensor(rng.normal(0, 2, (N, C))), dim=-1)
    g = helpers.ctc_topology(labels, C)
    r = run_fb(g, lp.numpy())
    lpt = lp.clone().unsqueeze(1).requires_grad_(True)
    loss = torch.nn.functional.ctc_loss(lpt, torch.tensor(labels)[None], torch.tensor([N]),
                                        torch.tensor([U]), blank=0, reduction="sum")
    loss.backward()
    assert abs(r["logZ"][0] + loss.item()) <= 1e-12
    Gam_torch = lp.exp().numpy() - lpt.grad[:, 0].numpy()
    assert np.abs(r["post_pdf"][0] - Gam_torch).max() <= 1e-12


# ------------------------------------------------------------------ LF-MMI

def _lfmmi1(num, den, emis):
    emis = np.asarray(emis, np.float64)
    return oracle.lfmmi_batch(synth.compose([num]), synth.compose([den]), emis[None],
                              np.array([emis.shape[0]], np.int32))


@pytest.mark.parametrize("seed", range(50))
def test_lfmmi_finite_difference(seed):
    """AC4: analytic gradient vs central differences, h = 1e-4."""
    rng = np.random.default_rng(5000 + seed)
    D = int(rng.integers(2, 6))
    num = synth.random_small_graph(rng, K=int(rng.integers(1, 6)), D=D)
    den = synth.random_small_graph(rng, K=int(rng.integers(1, 6)), D=D)
    N = int(rng.integers(1, 7))
    emis = rng.uniform(-3, 1, (N, D))
    r = _lfmmi1(num, den, emis)
    if r["status"][0] != 0:
        pytest.skip("empty lattice for this draw")
    h = 1e-4
    fd = np.zeros((N, D))
    for n in range(N):
        for d in range(D):
            ep = emis.copy(); ep[n, d] += h
            em = emis.copy(); em[n, d] -= h
            fd[n, d] = (_lfmmi1(num, den, ep)["loss"][0] - _lfmmi1(num, den, em)["loss"][0]) / (2 * h)
    g = r["grad"][0]
    assert np.abs(g - fd).max() <= 1e-5 * max(1.0, np.abs(g).max())
    # AC5: per-frame zero sum, bounded
    assert np.abs(g.sum(axis=1)).max() <= 1e-12
    assert g.min() >= -1 - 1e-12 and g.max() <= 1 + 1e-12


def test_lfmmi_num_equals_den():
    w = synth.make_c1(11)
    r = _lfmmi1(w.den, w.den, w.emis[0])
    assert r["loss"][0] == 0.0 and (r["grad"] == 0).all()


def test_lfmmi_one_state():
    # ℒ = (N−1)(t_n − t_d), grad = 0
    N = 9
    num = helpers.one_state(-0.3)
    den = helpers.one_state(-1.7)
    emis = np.random.default_rng(1).uniform(-4, 0, (N, 1))
    r = _lfmmi1(num, den, emis)
    tn, td = float(np.float32(-0.3)), float(np.float32(-1.7))  # graph weights are fp32
    assert r["loss"][0] == pytest.approx((N - 1) * (tn - td), abs=1e-12)
    assert (np.abs(r["grad"]) <= 1e-12).all()


def test_lfmmi_totals_closed_form_one_state():
    """All five totals on a batch of 1-state numerators / a 1-state denominator,
    where every quantity has a closed form: logZ_b = Σ_{n<N_b} v_{b,n}
    + (N_b − 1)·t + π + ω.  Pins totals[2] (Σ logZ_num) and totals[3] (Σ logZ_den)
    separately — a swap or a dropped term fails — and the exclusion of flagged
    sequences (NaN emission, bad length) from every total (§8(b))."""
    rng = np.random.default_rng(31)
    B, N_max = 6, 9
    tn = [float(np.float32(x)) for x in rng.uniform(-2, -0.1, B)]
    pin = [float(np.float32(x)) for x in rng.uniform(-1, 0, B)]
    td, pid, omd = float(np.float32(-1.3)), float(np.float32(-0.25)), float(np.float32(-0.5))
    nums = [helpers.one_state(tn[b], pin[b], 0.0) for b in range(B)]
    den = helpers.one_state(td, pid, omd)
    emis = rng.uniform(-4, 0, (B, N_max, 1)).astype(np.float32)
    lens = np.array([9, 1, 5, 9, 3, 10], np.int32)  # b = 5: N_b > N_max
    emis[3, 7, 0] = np.nan                            # b = 3: non-finite emission read
    r = oracle.lfmmi_batch(synth.compose(nums), synth.compose([den]), emis, lens)
    ok = np.array([True, True, True, False, True, False])
    assert ((r["status"] == 0) == ok).all()
    e64 = emis.astype(np.float64)
    zn = np.array([e64[b, : lens[b], 0].sum() + (lens[b] - 1) * tn[b] + pin[b] for b in range(B) if ok[b]])
    zd = np.array([e64[b, : lens[b], 0].sum() + (lens[b] - 1) * td + pid + omd for b in range(B) if ok[b]])
    t = r["totals"]
    assert t[2] == pytest.approx(zn.sum(), abs=1e-11)
    assert t[3] == pytest.approx(zd.sum(), abs=1e-11)
    assert t[0] == pytest.approx((zn - zd).sum(), abs=1e-11)
    assert t[1] == lens[ok].sum() and t[4] == 2
    assert r["logZ_num"][ok] == pytest.approx(zn, abs=1e-12)
    assert r["logZ_den"][ok] == pytest.approx(zd, abs=1e-12)


def test_lfmmi_shift_one_frame():
    # shifting one frame's φ row by c leaves ℒ and grad unchanged
    rng = np.random.default_rng(9)
    D = 4
    num = synth.random_small_graph(rng, K=4, D=D, weighted_ends=False)
    den = synth.random_small_graph(rng, K=5, D=D, weighted_ends=False)
    emis = rng.uniform(-3, 0, (6, D))
    r0 = _lfmmi1(num, den, emis)
    e1 = emis.copy(); e1[3] += 1.75
    r1 = _lfmmi1(num, den, e1)
    if r0["status"][0] == 0:
        assert abs(r1["loss"][0] - r0["loss"][0]) <= 1e-10
        assert np.abs(r1["grad"] - r0["grad"]).max() <= 1e-10


def test_lfmmi_totals_and_flags():
    rng = np.random.default_rng(2)
    D = 3
    nums = [synth.random_small_graph(rng, K=3, D=D) for _ in range(4)]
    den = synth.dense_graph(rng, 3)
    emis = rng.uniform(-3, 0, (4, 5, D))
    emis[2, 1, 0] = np.nan
    lens = np.array([5, 4, 5, 0], np.int32)
    r = oracle.lfmmi_batch(synth.compose(nums), synth.compose([den]), emis, lens)
    assert r["status"][2] & oracle.ST_NONFINITE and r["status"][3] & oracle.ST_BADLEN
    ok = r["status"] == 0
    assert r["totals"][4] == (~ok).sum()
    assert r["totals"][0] == pytest.approx(r["loss"][ok].sum(), abs=1e-12)
    assert r["totals"][1] == lens[ok].sum()
    assert (r["grad"][~ok] == 0).all()
    assert (r["grad"][1, 4:] == 0).all()  # padded frame (ledger L17)


# ------------------------------------------------------------------ invariants

def test_invariants_c2_small():
    w = synth.make_c2(seed=21, B=6, N_max=180)
    comp = synth.compose(w.nums)
    r = oracle.fb_batch(comp, w.emis, w.lengths, alpha=True, beta=True, post=True, post_pdf=True)
    assert (r["status"] == 0).all()
    assert np.abs(r["logZ"] - r["logZ_beta"]).max() <= 1e-9 * np.abs(r["logZ"]).max()
    assert r["gap"].max() <= 1e-9
    pp = r["post_pdf"]
    for b in range(6):
        s = pp[b, : w.lengths[b]].sum(axis=1)
        assert np.abs(s - 1).max() <= 1e-10
        assert (pp[b, w.lengths[b]:] == 0).all()


def test_relabelling_permutes_outputs():
    rng = np.random.default_rng(4)
    g = synth.random_small_graph(rng, K=6, D=4)
    emis = rng.uniform(-3, 0, (5, 4)).astype(np.float32)
    perm = rng.permutation(6)
    r0 = run_fb(g, emis)
    r1 = run_fb(helpers.relabel(g, perm), emis)
    assert r1["logZ"][0] == pytest.approx(r0["logZ"][0], abs=1e-12)
    assert np.abs(r1["post"][0][:, perm] - r0["post"][0]).max() <= 1e-13


def test_batch_equals_solo():
    w = synth.make_c2(seed=5, B=4, N_max=180)
    comp = synth.compose(w.nums)
    rb = oracle.fb_batch(comp, w.emis, w.lengths, post_pdf=True)
    for b in range(4):
        rs = oracle.fb_batch(w.nums[b], w.emis[b:b + 1], w.lengths[b:b + 1], post_pdf=True)
        assert rs["logZ"][0] == rb["logZ"][b]
        assert (rs["post_pdf"][0] == rb["post_pdf"][b]).all()


@pytest.mark.parametrize("Nb,Npad", [(4, 7), (6, 7), (2, 5)])
def test_phony_state_equivalence(Nb, Npad):
    """P:224-227 (ledger L8): the phony self-looping end state with 0̄/1̄ padding
    gives the same logZ and posteriors as running each sequence to its own length."""
    rng = np.random.default_rng(Nb * 10 + Npad)
    g = synth.random_small_graph(rng, K=3, D=3, p_neg_inf=0.2)
    emis = rng.uniform(-3, 0, (Npad, 3))
    r = run_fb(g, emis[:Nb])
    gp = helpers.add_phony_final(g)
    rp = run_fb(gp, helpers.pad_for_phony(emis, Nb, Npad))
    if r["status"][0] != 0:
        assert rp["status"][0] == oracle.ST_EMPTY
        return
    assert abs(rp["logZ"][0] - r["logZ"][0]) <= 1e-12
    assert np.abs(rp["post"][0][:Nb, :3] - r["post"][0]).max() <= 1e-12


def test_prob_domain_matrix_recursion():
    """Eq. (4)-(5) in the probability domain with numpy matmul
    (v_{n+1} inside the backward, ledger L2) on well-conditioned inputs (AC8)."""
    rng = np.random.default_rng(8)
    for _ in range(20):
        g = synth.random_small_graph(rng, K=int(rng.integers(2, 8)), D=None, p_neg_inf=0.0)
        N = int(rng.integers(2, 20))
        emis = rng.uniform(-3, 0, (N, g.D))
        T = np.exp(brute.dense_T(g))
        V = np.exp(emis[:, g.pdf_of])
        a = np.zeros((N, g.K)); b = np.zeros((N, g.K))
        a[0] = np.exp(g.log_init.astype(np.float64)) * V[0]
        for n in range(1, N):
            a[n] = V[n] * (T.T @ a[n - 1])
        b[N - 1] = np.exp(g.log_final.astype(np.float64))
        for n in range(N - 2, -1, -1):
            b[n] = T @ (b[n + 1] * V[n + 1])
        Z = (a[N - 1] * b[N - 1]).sum()
        if Z == 0:
            continue
        r = run_fb(g, emis)
        assert r["logZ"][0] == pytest.approx(math.log(Z), abs=1e-10)
        assert np.abs(r["post"][0] - a * b / Z).max() <= 1e-10


def test_stability_regression():
    """AC6: N = 1000, K = 10 left-to-right, φ ∈ [−100, −50]:
    the log-domain oracle stays finite and normalised while the probability
    domain underflows to 0."""
    g = helpers.left_to_right(10)
    rng = np.random.default_rng(6)
    emis = rng.uniform(-100, -50, (1000, 10))
    r = run_fb(g, emis)
    assert r["status"][0] == 0 and np.isfinite(r["logZ"][0])
    assert np.abs(r["post"][0].sum(axis=1) - 1).max() <= 1e-9
    T = np.exp(brute.dense_T(g))
    a = np.exp(g.log_init.astype(np.float64)) * np.exp(emis[0])
    for n in range(1, 1000):
        a = np.exp(emis[n]) * (T.T @ a)
    assert (a * np.exp(g.log_final.astype(np.float64))).sum() == 0.0


def test_status_flags():
    w = synth.make_c1(3)
    e = w.emis.copy(); e[0, 2, 1] = np.inf
    r = oracle.fb_batch(w.den, e, np.array([6], np.int32))
    assert r["status"][0] == oracle.ST_NONFINITE
    r = oracle.fb_batch(w.den, w.emis, np.array([7], np.int32))
    assert r["status"][0] == oracle.ST_BADLEN
    g = helpers.left_to_right(5)
    r = oracle.fb_batch(g, np.zeros((1, 3, 5), np.float32), np.array([3], np.int32))
    assert r["status"][0] == oracle.ST_EMPTY and r["logZ"][0] == -math.inf
    e = np.zeros((1, 3, 1), np.float32); e[0, 1, 0] = -np.inf  # −∞ emission is a legal 0̄
    r = oracle.fb_batch(helpers.one_state(), e, np.array([3], np.int32))
    assert r["status"][0] == oracle.ST_EMPTY


# ------------------------------------------------------------------ Viterbi (N1)

@pytest.mark.parametrize("seed", range(50))
def test_viterbi_vs_brute(seed):
    rng = np.random.default_rng(7000 + seed)
    K = int(rng.integers(1, 7))
    g = synth.random_small_graph(rng, K=K, D=int(rng.integers(1, K + 1)))
    N = int(rng.integers(1, 7))
    emis = rng.uniform(-5, 1, (N, g.D)).astype(np.float32)
    v = oracle.viterbi_batch(g, emis[None], np.array([N], np.int32))
    logZ, _, _, best, path = brute.brute_force(g, emis)
    if best == -math.inf:
        assert v["status"][0] == oracle.ST_EMPTY
        return
    assert v["score"][0] == pytest.approx(best, abs=1e-12)
    assert v["score"][0] <= logZ + 1e-12
    assert v["path"][0].tolist() == path.tolist()
