"""N4: the paper's literal execution strategy (block-diagonal batch SpMV per
frame with phony-state padding) in three semirings,
through the C-ABI, against the float64 oracle and against the fused kernels."""
import numpy as np
import pytest

import oracle
from paper_2112_00709_b200 import synth
from tests import helpers

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fbx():
    import torch

    assert torch.cuda.is_available(), "GPU tests need CUDA"
    from paper_2112_00709_b200 import build

    build.build()
    import paper_2112_00709_b200 as fbx

    fbx.lib()
    return fbx


def dev(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def literal(fbx, graph, emis, lengths, sr, flags=0):
    import torch

    g = fbx.Graph.from_host(graph, flags)
    s = fbx.fb_forward_literal(g, dev(emis.astype(np.float32)), dev(lengths.astype(np.int32)), sr)
    torch.cuda.synchronize()
    return s.cpu().numpy()


def test_log_semiring_c1_composed(fbx):
    """G = B block-diagonal batch of 100 dense K = 3 graphs (C1)."""
    ws = [synth.make_c1(s) for s in range(100)]
    g = synth.compose([w.den for w in ws])
    emis = np.concatenate([w.emis for w in ws])
    lens = np.full(100, 6, np.int32)
    lens[::7] = 3  # ragged: phony padding must reproduce the per-length result
    got = literal(fbx, g, emis, lens, fbx.SEMIRING_LOG)
    ref = oracle.fb_batch(g, emis, lens, post=False)["logZ"]
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_log_semiring_den_vs_oracle_and_fused(fbx):
    """G = 1 shared denominator (B copies in the block-diagonal batch)."""
    import torch

    w = synth.make_c3(seed=31, B=5, N=40, K=700, nnz=4000)
    lens = np.array([40, 1, 17, 40, 29], np.int32)
    got = literal(fbx, w.den, w.emis, lens, fbx.SEMIRING_LOG)
    ref = oracle.fb_batch(w.den, w.emis, lens, post=False)["logZ"]
    assert (np.abs(got - ref) / np.abs(ref)).max() <= 1e-12
    g = fbx.Graph.from_host(w.den)
    logZ, _, _, st = fbx.fb_forward(g, dev(w.emis), dev(lens))
    torch.cuda.synchronize()
    assert (np.abs(logZ.cpu().numpy() - got) / np.abs(got)).max() <= 1e-5


def test_log_semiring_numerators(fbx):
    w = synth.make_c2(seed=2, B=12)
    g = synth.compose(w.nums)
    got = literal(fbx, g, w.emis, w.lengths, fbx.SEMIRING_LOG)
    ref = oracle.fb_batch(g, w.emis, w.lengths, post=False)["logZ"]
    assert (np.abs(got - ref) / np.abs(ref)).max() <= 1e-12


def test_tropical_semiring_is_viterbi(fbx):
    w = synth.make_c2(seed=3, B=8)
    g = synth.compose(w.nums)
    got = literal(fbx, g, w.emis, w.lengths, fbx.SEMIRING_TROPICAL)
    ref = oracle.viterbi_batch(g, w.emis, w.lengths)["score"]
    assert np.abs(got - ref).max() <= 1e-9 * np.abs(ref).max()
    ws = [synth.make_c1(s) for s in range(20)]
    g1 = synth.compose([x.den for x in ws])
    e1 = np.concatenate([x.emis for x in ws])
    l1 = np.full(20, 6, np.int32)
    got1 = literal(fbx, g1, e1, l1, fbx.SEMIRING_TROPICAL)
    assert np.abs(got1 - oracle.viterbi_batch(g1, e1, l1)["score"]).max() <= 1e-12


def test_prob_semiring_equals_exp_logZ_and_underflows(fbx):
    """Probability domain: exp(logZ) on short inputs; on the AC6 input (N = 1000,
    φ ∈ [−100, −50]) it underflows to exactly 0 while the log semiring stays
    finite and matches the oracle — the paper's reason for the log domain."""
    ws = [synth.make_c1(s) for s in range(10)]
    g = synth.compose([w.den for w in ws])
    emis = np.concatenate([w.emis for w in ws])
    lens = np.full(10, 6, np.int32)
    got = literal(fbx, g, emis, lens, fbx.SEMIRING_PROB)
    ref = np.exp(oracle.fb_batch(g, emis, lens, post=False)["logZ"])
    assert (np.abs(got - ref) / ref).max() <= 1e-12
    lr = helpers.left_to_right(10)
    rng = np.random.default_rng(6)
    e = rng.uniform(-100, -50, (1, 1000, 10)).astype(np.float32)
    L = np.array([1000], np.int32)
    assert literal(fbx, lr, e, L, fbx.SEMIRING_PROB)[0] == 0.0
    lz = literal(fbx, lr, e, L, fbx.SEMIRING_LOG)[0]
    ref = oracle.fb_batch(lr, e, L, post=False)["logZ"][0]
    assert np.isfinite(lz) and abs(lz - ref) <= 1e-12 * abs(ref)


# ------------------------------------------------------------------ forward-backward + posteriors (N4)

def literal_fb(fbx, graph, emis, lengths, sr):
    import torch

    g = fbx.Graph.from_host(graph)
    score, post = fbx.fb_forward_backward_literal(g, dev(emis.astype(np.float32)), dev(lengths.astype(np.int32)), sr)
    torch.cuda.synchronize()
    return score.cpu().numpy(), post.cpu().numpy()


@pytest.mark.parametrize("which", ["c1", "small", "c2", "den"])
def test_literal_fb_log_posteriors_vs_oracle(fbx, which):
    """Log semiring: the literal backward over the augmented out-arc lists and the
    posteriors X ⊗ y ⊘ Z equal the oracle's γ (float64 both sides) on the C1 batch,
    the irregular brute-force family (−∞ / duplicate arcs, weighted π/ω, ragged
    lengths), numerator graphs (G = B) and a shared den (G = 1)."""
    if which == "c1":
        ws = [synth.make_c1(s) for s in range(30)]
        g = synth.compose([w.den for w in ws])
        emis = np.concatenate([w.emis for w in ws])
        lens = np.full(30, 6, np.int32)
        lens[::4] = 2
    elif which == "small":
        rng = np.random.Generator(np.random.PCG64(77))
        gs = [synth.random_small_graph(rng, K=int(rng.integers(1, 7)), D=6) for _ in range(60)]
        g = synth.compose(gs)
        emis = rng.uniform(-3, 0, (60, 7, 6)).astype(np.float32)
        lens = rng.integers(1, 8, 60).astype(np.int32)
    elif which == "c2":
        w = synth.make_c2(seed=4, B=6)
        g, emis, lens = synth.compose(w.nums), w.emis, w.lengths
    else:
        w = synth.make_c3(seed=35, B=3, N=30, K=700, nnz=4000)
        g, emis, lens = w.den, w.emis, np.array([30, 11, 30], np.int32)
    score, post = literal_fb(fbx, g, emis, lens, fbx.SEMIRING_LOG)
    ref = oracle.fb_batch(g, emis, lens, post=True)
    ok = ref["status"] == 0
    assert np.abs(score[ok] - ref["logZ"][ok]).max(initial=0) <= 1e-11 * max(1.0, np.abs(ref["logZ"][ok]).max())
    assert np.isneginf(score[~ok]).all()
    assert np.abs(post.reshape(ref["post"].shape) - ref["post"]).max() <= 1e-11


def test_literal_fb_prob_and_tropical(fbx):
    """Probability semiring: the same γ in the linear domain (short inputs).  Tropical:
    the max-marginal ratio is 1 exactly along fb_viterbi's best path (unique here) and
    ≤ 1 everywhere."""
    import torch

    w = synth.make_c2(seed=5, B=4, N_max=150)
    g, emis = synth.compose(w.nums), w.emis
    lens = np.minimum(w.lengths, 150)
    ref = oracle.fb_batch(g, emis, lens, post=True)
    ws = [synth.make_c1(s) for s in range(10)]
    g1 = synth.compose([x.den for x in ws])
    e1 = np.concatenate([x.emis for x in ws])
    l1 = np.full(10, 6, np.int32)
    sp, pp = literal_fb(fbx, g1, e1, l1, fbx.SEMIRING_PROB)
    r1 = oracle.fb_batch(g1, e1, l1, post=True)
    assert (np.abs(sp - np.exp(r1["logZ"])) / np.exp(r1["logZ"])).max() <= 1e-12
    assert np.abs(pp.reshape(r1["post"].shape) - r1["post"]).max() <= 1e-11
    st, pt = literal_fb(fbx, g, emis, lens, fbx.SEMIRING_TROPICAL)
    vit = oracle.viterbi_batch(g, emis, lens)
    assert np.abs(st - vit["score"]).max() <= 1e-9 * np.abs(vit["score"]).max()
    so = g.state_offsets
    N_max = emis.shape[1]
    for b in range(len(lens)):
        K = so[b + 1] - so[b]
        P = pt[N_max * so[b]: N_max * so[b + 1]].reshape(N_max, K)
        assert (P <= 1 + 1e-9).all() and (P[lens[b]:] == 0).all()
        path = vit["path"][b, : lens[b]]
        assert np.abs(P[np.arange(lens[b]), path] - 1).max() <= 1e-9
    torch.cuda.synchronize()


# ------------------------------------------------------------------ fused semiring-generic forward (N4)

@pytest.mark.parametrize("which", ["c1", "small", "c2", "c3", "n2"])
def test_fused_forward_semirings(fbx, which):
    """fb_forward_semiring: one fused kernel body instantiated for the log, tropical and
    probability semirings.  Log = the oracle's log Z, tropical = the oracle's
    Viterbi score, probability = exp(log Z) where it does not underflow; numerator batches
    (G = B), the irregular brute-force family, a shared den (G = 1) and the paper's den
    (schedule streamed from L2)."""
    import torch

    if which == "c1":
        ws = [synth.make_c1(s) for s in range(40)]
        g = synth.compose([w.den for w in ws])
        emis = np.concatenate([w.emis for w in ws])
        lens = np.full(40, 6, np.int32)
        lens[::5] = 2
    elif which == "small":
        rng = np.random.Generator(np.random.PCG64(88))
        gs = [synth.random_small_graph(rng, K=int(rng.integers(1, 7)), D=6) for _ in range(60)]
        g = synth.compose(gs)
        emis = rng.uniform(-3, 0, (60, 7, 6)).astype(np.float32)
        lens = rng.integers(1, 8, 60).astype(np.int32)
    elif which == "c2":
        w = synth.make_c2(seed=8, B=8)
        g, emis, lens = synth.compose(w.nums), w.emis, w.lengths
    elif which == "c3":
        w = synth.make_c3(seed=36, B=3, N=40, K=3000, nnz=20000)
        g, emis, lens = w.den, w.emis, np.array([40, 17, 40], np.int32)
    else:
        w = synth.make_paper_shape(seed=6, B=2, N=30, L_range=(5, 10))
        g, emis, lens = w.den, w.emis, np.array([30, 21], np.int32)
    G = fbx.Graph.from_host(g)
    e, L = dev(emis), dev(lens)
    out = {sr: fbx.fb_forward_semiring(G, e, L, sr) for sr in (fbx.SEMIRING_LOG, fbx.SEMIRING_TROPICAL,
                                                                fbx.SEMIRING_PROB)}
    torch.cuda.synchronize()
    ref = oracle.fb_batch(g, emis, lens, post=False)
    vit = oracle.viterbi_batch(g, emis, lens)
    ok = ref["status"] == 0
    zl, stl = (x.cpu().numpy() for x in out[fbx.SEMIRING_LOG])
    assert (stl == ref["status"]).all()
    assert np.abs(zl[ok] - ref["logZ"][ok]).max(initial=0) <= 1e-12 * max(1.0, np.abs(ref["logZ"][ok]).max(initial=1))
    zt, stt = (x.cpu().numpy() for x in out[fbx.SEMIRING_TROPICAL])
    assert (stt == vit["status"]).all()
    okv = vit["status"] == 0
    assert np.abs(zt[okv] - vit["score"][okv]).max(initial=0) <= 1e-12 * max(1.0, np.abs(vit["score"][okv]).max(initial=1))
    zp, stp = (x.cpu().numpy() for x in out[fbx.SEMIRING_PROB])
    lin = np.exp(ref["logZ"])
    fine = ok & (lin > 1e-280)
    assert (np.abs(zp[fine] - lin[fine]) / lin[fine]).max(initial=0) <= 1e-11
    assert (zp[ok & (lin == 0)] == 0).all() and (stp[ok & (lin == 0)] == fbx.SEQ_EMPTY_LATTICE).all()


def test_fused_prob_semiring_underflows_on_ac6(fbx):
    """AC6: the fused probability instance returns exactly 0 (flagged as an empty
    lattice) while the log instance matches the oracle's finite log Z."""
    import torch

    lr = helpers.left_to_right(10)
    e = np.random.default_rng(6).uniform(-100, -50, (1, 1000, 10)).astype(np.float32)
    L = np.array([1000], np.int32)
    G = fbx.Graph.from_host(lr)
    zp, sp = fbx.fb_forward_semiring(G, dev(e), dev(L), fbx.SEMIRING_PROB)
    zl, sl = fbx.fb_forward_semiring(G, dev(e), dev(L), fbx.SEMIRING_LOG)
    torch.cuda.synchronize()
    ref = oracle.fb_batch(lr, e, L, post=False)["logZ"][0]
    assert zp.item() == 0.0 and sp.item() == fbx.SEQ_EMPTY_LATTICE
    assert sl.item() == 0 and abs(zl.item() - ref) <= 1e-12 * abs(ref)
