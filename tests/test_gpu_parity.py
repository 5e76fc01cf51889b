"""T1-T3: CUDA path (through the C-ABI) vs the float64 oracle, element by element.

Gates (BASELINE.json north_star): |ΔlogZ| ≤ 1e-5·max(1, |logZ|); max |Δγ| ≤ 1e-5;
max |Δgrad| ≤ 1e-5.  Inputs are generated once in fp32 and fed bit-identically
to both sides.
"""
import numpy as np
import pytest

import oracle
from paper_2112_00709_b200 import synth

pytestmark = pytest.mark.gpu

TOL_LOGZ = 1e-5
TOL_POST = 1e-5
TOL_GRAD = 1e-5


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


def run_fb(fbx, graph, emis, lengths, flags=0, post="state"):
    import torch

    g = fbx.Graph.from_host(graph, flags)
    e, L = dev(emis), dev(lengths.astype(np.int32))
    logZ, alpha, scale, st = fbx.fb_forward(g, e, L)
    p, logZb, st2, beta, bscale = fbx.fb_backward(g, e, L, alpha=alpha, status=st.clone(), want_beta=True, post=post)
    torch.cuda.synchronize()
    return dict(g=g, logZ=logZ.cpu().numpy(), logZb=logZb.cpu().numpy(), st=st2.cpu().numpy(),
                st_fwd=st.cpu().numpy(), post=p.cpu().numpy(), alpha=alpha, scale=scale, beta=beta,
                bscale=bscale, e=e, L=L)


def check_logZ(got, ref, ok):
    err = np.abs(got[ok] - ref[ok]) / np.maximum(1.0, np.abs(ref[ok]))
    assert err.max(initial=0) <= TOL_LOGZ, err.max()
    return err.max(initial=0)


# ------------------------------------------------------------------ C1 (100 seeds, dense K=3)

@pytest.mark.parametrize("flags", [0, 1])
def test_c1_vs_oracle_and_bruteforce(fbx, flags):
    ws = [synth.make_c1(s) for s in range(100)]
    comp = synth.compose([w.den for w in ws])
    emis = np.concatenate([w.emis for w in ws])
    lens = np.full(100, 6, np.int32)
    r = run_fb(fbx, comp, emis, lens, flags=flags)
    ref = oracle.fb_batch(comp, emis, lens, post=True)
    assert (r["st"] == 0).all()
    check_logZ(r["logZ"], ref["logZ"], np.ones(100, bool))
    check_logZ(r["logZb"], ref["logZ"], np.ones(100, bool))
    assert np.abs(r["post"] - ref["post"]).max() <= TOL_POST


# ------------------------------------------------------------------ C2 numerator graphs (G = B)

@pytest.mark.parametrize("kind", ["uniform", "softmax4"])
def test_c2_numerators(fbx, kind):
    w = synth.make_c2(seed=2, kind=kind)
    comp = synth.compose(w.nums)
    r = run_fb(fbx, comp, w.emis, w.lengths)
    ref = oracle.fb_batch(comp, w.emis, w.lengths, alpha=True, post=True)
    assert (r["st"] == ref["status"]).all() and (r["st"] == 0).all()
    check_logZ(r["logZ"], ref["logZ"], r["st"] == 0)
    err = np.abs(r["post"] - ref["post"]).max()
    assert err <= TOL_POST, err
    # lattice: α_true = α̂ + scale on states carrying mass
    alpha = r["alpha"].cpu().numpy()
    scale = r["scale"].cpu().numpy()
    so = comp.state_offsets
    for b in range(0, w.B, 7):
        K = so[b + 1] - so[b]
        N = w.lengths[b]
        a_gpu = alpha[w.N_max * so[b]: w.N_max * so[b + 1]].reshape(w.N_max, K)
        a_ref = ref["alpha"][w.N_max * so[b]: w.N_max * so[b + 1]].reshape(w.N_max, K)
        rel = a_ref[:N] - scale[b, :N, None]
        live = (r["post"][w.N_max * so[b]: w.N_max * so[b + 1]].reshape(w.N_max, K)[:N] > 1e-6)
        assert np.abs(a_gpu[:N][live] - rel[live]).max() <= 1e-3
        assert np.isneginf(a_gpu[N:]).all()


# ------------------------------------------------------------------ C3 denominator (G = 1), reduced

@pytest.mark.parametrize("kind,flags,K,nnz", [("uniform", 0, 3000, 20000), ("softmax4", 0, 3000, 20000),
                                              ("softmax8", 0, 3000, 20000), ("uniform", 1, 1500, 10000),
                                              ("softmax4", 2, 1500, 10000), ("uniform", 0, 700, 4000)])
def test_c3_den_reduced(fbx, kind, flags, K, nnz):
    w = synth.make_c3(seed=3, B=6, N=64, kind=kind, K=K, nnz=nnz)
    lens = np.array([64, 1, 33, 64, 17, 50], np.int32)
    r = run_fb(fbx, w.den, w.emis, lens, flags=flags)
    ref = oracle.fb_batch(w.den, w.emis, lens, post=True)
    assert (r["st"] == 0).all()
    check_logZ(r["logZ"], ref["logZ"], np.ones(6, bool))
    err = np.abs(r["post"].reshape(ref["post"].shape) - ref["post"]).max()
    tol = TOL_POST  # σ = 8 too: measured 2.4e-6 on the den (profiles/r2_parity_errors.txt)
    assert err <= tol, err
    # posteriors sum to 1 on valid frames, 0 on padding
    P = r["post"].reshape(6, 64, -1)
    for b in range(6):
        assert np.abs(P[b, : lens[b]].sum(1) - 1).max() <= 1e-4
        assert (P[b, lens[b]:] == 0).all()


def test_c3_pdf_level_and_standalone_posteriors(fbx):
    w = synth.make_c4(seed=4, B=4, N=40)
    den = w.den
    lens = np.array([40, 40, 12, 3], np.int32)
    r = run_fb(fbx, den, w.emis, lens, post="pdf")
    ref = oracle.fb_batch(den, w.emis, lens, post=True, post_pdf=True)
    assert np.abs(r["post"] - ref["post_pdf"]).max() <= TOL_POST
    st = dev(r["st"])
    p_state = fbx.fb_posteriors(r["g"], r["alpha"], r["beta"], r["L"], st, 4, 40, pdf_level=False)
    p_pdf = fbx.fb_posteriors(r["g"], r["alpha"], r["beta"], r["L"], st, 4, 40, pdf_level=True)
    assert np.abs(p_state.cpu().numpy().reshape(ref["post"].shape) - ref["post"]).max() <= TOL_POST
    assert np.abs(p_pdf.cpu().numpy() - ref["post_pdf"]).max() <= TOL_POST


# ------------------------------------------------------------------ C4 LF-MMI, reduced

@pytest.mark.parametrize("kind", ["uniform", "softmax4"])
def test_c4_lfmmi_reduced(fbx, kind):
    import torch

    w = synth.make_c4(seed=4, B=8, N=120, kind=kind, L_range=(20, 60))
    lens = np.array([120, 120, 90, 61, 120, 100, 75, 120], np.int32)
    num = fbx.Graph.from_host(synth.compose(w.nums))
    den = fbx.Graph.from_host(w.den)
    loss, totals, st, grad = fbx.lfmmi_loss_grad(num, den, dev(w.emis), dev(lens))
    torch.cuda.synchronize()
    ref = oracle.lfmmi_batch(synth.compose(w.nums), synth.compose([w.den]), w.emis, lens)
    st = st.cpu().numpy()
    assert (st == ref["status"]).all()
    ok = st == 0
    assert ok.sum() >= 6
    zd_ref, zn_ref = ref["logZ_den"], ref["logZ_num"]
    err_loss = np.abs(loss.cpu().numpy()[ok] - ref["loss"][ok]) / np.maximum(1, np.abs(zd_ref[ok]))
    assert err_loss.max() <= TOL_LOGZ
    g = grad.cpu().numpy()
    err = np.abs(g - ref["grad"]).max()
    assert err <= TOL_GRAD, err
    t = totals.cpu().numpy()
    assert t[4] == (~ok).sum() and t[1] == lens[ok].sum()
    assert abs(t[0] - ref["totals"][0]) <= 1e-5 * max(1, abs(ref["totals"][3]))
    # per-frame zero sum of the gradient (AC5)
    assert np.abs(g.sum(-1)).max() <= 1e-4


# ------------------------------------------------------------------ faults (T3)

def test_status_flags(fbx):
    import torch

    w = synth.make_c4(seed=14, B=4, N=30, L_range=(10, 20))
    emis = w.emis.copy()
    emis[1, 5, :] = np.nan
    lens = np.array([30, 30, 0, 31], np.int32)  # bad lengths: 0 and > N_max
    num = fbx.Graph.from_host(synth.compose(w.nums))
    den = fbx.Graph.from_host(w.den)
    loss, totals, st, grad = fbx.lfmmi_loss_grad(num, den, dev(emis), dev(lens))
    torch.cuda.synchronize()
    st = st.cpu().numpy()
    assert st[0] == 0
    assert st[1] & fbx.SEQ_NONFINITE_INPUT
    assert st[2] & fbx.SEQ_BAD_LENGTH and st[3] & fbx.SEQ_BAD_LENGTH
    g = grad.cpu().numpy()
    assert (g[1:] == 0).all() and np.isfinite(g).all()
    assert (loss.cpu().numpy()[1:] == 0).all()
    assert totals.cpu().numpy()[4] == 3


def test_empty_lattice(fbx):
    # numerator needs ≥ L frames; give it fewer
    rng = np.random.Generator(np.random.PCG64(5))
    g = synth.numerator_graph(rng, 20, 300, "identity")
    emis = synth.emissions(rng, 2, 30, 300)
    lens = np.array([10, 30], np.int32)
    r = run_fb(fbx, synth.compose([g, g]), emis, lens)
    assert r["st_fwd"][0] == fbx.SEQ_EMPTY_LATTICE and r["st_fwd"][1] == 0
    assert r["logZ"][0] == -np.inf
    ref = oracle.fb_batch(synth.compose([g, g]), emis, lens)
    check_logZ(r["logZ"], ref["logZ"], np.array([False, True]))


# ------------------------------------------------------------------ determinism (T2)

def test_bitwise_determinism_and_batch_independence(fbx):
    import torch

    w = synth.make_c3(seed=9, B=5, N=40)
    lens = np.array([40, 31, 40, 7, 22], np.int32)
    r1 = run_fb(fbx, w.den, w.emis, lens)
    r2 = run_fb(fbx, w.den, w.emis, lens)
    assert (r1["post"] == r2["post"]).all() and (r1["logZ"] == r2["logZ"]).all()
    # sequence 3 alone (B = 1) == its row in the batch, bit for bit
    solo = run_fb(fbx, w.den, w.emis[3:4].copy(), lens[3:4])
    K = w.den.K
    assert (solo["post"].reshape(1, 40, K) == r1["post"].reshape(5, 40, K)[3:4]).all()
    assert solo["logZ"][0] == r1["logZ"][3]
    # shuffled batch → permuted identical outputs
    perm = np.array([4, 2, 0, 3, 1])
    r3 = run_fb(fbx, w.den, w.emis[perm].copy(), lens[perm])
    assert (r3["post"].reshape(5, 40, K) == r1["post"].reshape(5, 40, K)[perm]).all()
    torch.cuda.synchronize()


# ------------------------------------------------------------------ full BASELINE sizes, sampled

@pytest.mark.slow
def test_c3_full_size_sampled(fbx):
    """C3 at its full size (B=128, N=500, K=3000, nnz≈20k) in the bench launch
    configuration; the oracle recomputes sampled utterances one by one."""
    w = synth.make_c3(seed=3)
    r = run_fb(fbx, w.den, w.emis, w.lengths)
    assert (r["st"] == 0).all()
    K = w.den.K
    P = r["post"].reshape(128, 500, K)
    for b in (0, 77, 127):
        ref = oracle.fb_batch(w.den, w.emis[b:b + 1], w.lengths[b:b + 1], post=True)
        check_logZ(r["logZ"][b:b + 1], ref["logZ"], np.ones(1, bool))
        assert np.abs(P[b] - ref["post"][0]).max() <= TOL_POST
    # properties that hold at any size, on every utterance
    assert np.abs(P.sum(-1) - 1).max() <= 1e-4
    assert (np.abs(r["logZ"] - r["logZb"]) / np.abs(r["logZ"])).max() <= TOL_LOGZ


@pytest.mark.slow
def test_c4_full_size_sampled(fbx):
    import torch

    w = synth.make_c4(seed=4)
    num = fbx.Graph.from_host(synth.compose(w.nums))
    den = fbx.Graph.from_host(w.den)
    loss, totals, st, grad = fbx.lfmmi_loss_grad(num, den, dev(w.emis), dev(w.lengths))
    torch.cuda.synchronize()
    st = st.cpu().numpy()
    assert (st == 0).all()
    g = grad.cpu().numpy()
    for b in (3, 64, 120):
        ref = oracle.lfmmi_batch(synth.compose([w.nums[b]]), synth.compose([w.den]), w.emis[b:b + 1],
                                 w.lengths[b:b + 1])
        assert abs(loss.cpu().numpy()[b] - ref["loss"][0]) <= TOL_LOGZ * max(1, abs(ref["logZ_den"][0]))
        assert np.abs(g[b] - ref["grad"][0]).max() <= TOL_GRAD
    assert np.abs(g.sum(-1)).max() <= 1e-4


# ------------------------------------------------------------------ Viterbi (N1)

def _viterbi_check(fbx, graph, emis, lengths):
    import torch

    g = fbx.Graph.from_host(graph)
    score, path, st = fbx.fb_viterbi(g, dev(emis), dev(lengths.astype(np.int32)))
    torch.cuda.synchronize()
    ref = oracle.viterbi_batch(graph, emis, lengths)
    st = st.cpu().numpy()
    assert (st == ref["status"]).all()
    ok = st == 0
    # float64 max-plus with the same operand order as the oracle: identical scores and paths
    assert (score.cpu().numpy()[ok] == ref["score"][ok]).all()
    assert (path.cpu().numpy() == ref["path"]).all()


def test_viterbi_c1(fbx):
    ws = [synth.make_c1(s) for s in range(100)]
    _viterbi_check(fbx, synth.compose([w.den for w in ws]), np.concatenate([w.emis for w in ws]),
                   np.full(100, 6, np.int32))


def test_viterbi_c2_numerators(fbx):
    w = synth.make_c2(seed=2, B=16)
    _viterbi_check(fbx, synth.compose(w.nums), w.emis, w.lengths)


def test_viterbi_c3_den(fbx):
    w = synth.make_c3(seed=3, B=4, N=80)
    _viterbi_check(fbx, w.den, w.emis, np.array([80, 13, 1, 55], np.int32))


@pytest.mark.slow
@pytest.mark.parametrize("which", ["c3", "paper"])
def test_viterbi_full_size_sampled(fbx, which):
    """N1 at the bench sizes (`bench.py --workload viterbi` / `viterbi-paper`: C3 den B=128, N=500;
    the paper's den B=128, N=700, schedule streamed from L2) in the bench launch configuration;
    the oracle recomputes sampled utterances — scores and paths bit for bit."""
    import torch

    w = synth.make_c3(seed=3) if which == "c3" else synth.make_paper_shape(seed=6)
    g = fbx.Graph.from_host(w.den)
    score, path, st = fbx.fb_viterbi(g, dev(w.emis), dev(w.lengths))
    torch.cuda.synchronize()
    assert (st.cpu().numpy() == 0).all()
    score, path = score.cpu().numpy(), path.cpu().numpy()
    for b in (0, 63, 127):
        ref = oracle.viterbi_batch(w.den, w.emis[b:b + 1], w.lengths[b:b + 1])
        assert score[b] == ref["score"][0]
        assert (path[b] == ref["path"][0]).all()


def test_viterbi_paper_shape_n2(fbx):
    """N1 on the paper's Table 1 denominator (3022 states, 50,984 arcs): its
    float64 Viterbi schedule exceeds shared memory and is streamed from global memory
    (L2); scores and tie-broken paths equal the oracle's bit for bit."""
    w = synth.make_paper_shape(seed=6, B=3, N=60, L_range=(10, 20))
    g = fbx.Graph.from_host(w.den)
    assert g.info["cluster_C"] > 0  # the one-CTA forward-backward kernels do not fit either
    _viterbi_check(fbx, w.den, w.emis, np.array([60, 41, 1], np.int32))


# ------------------------------------------------------------------ cluster-batched kernel (k_fbc)

@pytest.mark.parametrize("cs", ["2,2", "4,2", "2,4", "4,4", "8,2", "4,4,1", "4,4,1/split1", "4,4,1/splitf",
                                "4,4,1/splitb", "2,2/split1", "8,4/split1", "8,4,1"])
def test_cluster_configs_vs_oracle(fbx, cs, monkeypatch):
    """Every (C CTAs, S sequences) cluster configuration of a shared factored
    graph against the oracle: logZ (both directions), α̂ + scale, state and pdf
    posteriors, ragged lengths (a length-1 sequence, an odd batch).  /splitX
    forces phase A's local/remote arc split (0 none, 1 both directions, f forward only, b backward
    only; default: none)."""
    if "/split" in cs:
        cs, sp = cs.split("/split")
        monkeypatch.setenv("FBX_CLUSTER_SPLIT", sp)
    monkeypatch.setenv("FBX_CLUSTER", cs)
    w = synth.make_c4(seed=21, B=5, N=48, K=1500, nnz=10000, D=1000, kind="softmax4")
    lens = np.array([48, 1, 30, 48, 17], np.int32)
    r = run_fb(fbx, w.den, w.emis, lens)
    C, S = (int(x) for x in cs.split(",")[:2])
    assert (r["g"].info["cluster_C"], r["g"].info["cluster_S"]) == (C, S)
    ref = oracle.fb_batch(w.den, w.emis, lens, alpha=True, post=True, post_pdf=True)
    assert (r["st"] == 0).all()
    check_logZ(r["logZ"], ref["logZ"], np.ones(5, bool))
    check_logZ(r["logZb"], ref["logZ"], np.ones(5, bool))
    K = w.den.K
    assert np.abs(r["post"].reshape(ref["post"].shape) - ref["post"]).max() <= TOL_POST
    # α̂ + C_n = α (float64 oracle), on finite entries; −∞ exactly where the oracle has −∞
    a = r["alpha"].cpu().numpy().reshape(5, 48, K).astype(np.float64) + r["scale"].cpu().numpy()[:, :, None]
    ra = ref["alpha"].reshape(5, 48, K)
    for b in range(5):
        fin = np.isfinite(ra[b, : lens[b]])
        assert (np.isfinite(a[b, : lens[b]]) == fin).all()
        d = np.abs(a[b, : lens[b]][fin] - ra[b, : lens[b]][fin]) / np.maximum(1.0, np.abs(ra[b, : lens[b]][fin]))
        assert d.max() <= 1e-5, d.max()
    rp = run_fb(fbx, w.den, w.emis, lens, post="pdf")
    assert np.abs(rp["post"] - ref["post_pdf"]).max() <= TOL_POST


def test_cluster_matches_one_cta_per_sequence(fbx):
    """k_fbc (FB_GRAPH_CLUSTER) and the one-CTA-per-sequence kernel on the same
    C4-shaped inputs; both within the gates of the oracle."""
    import torch

    w = synth.make_c4(seed=22, B=4, N=64, L_range=(10, 30))
    lens = np.array([64, 40, 64, 33], np.int32)
    num = fbx.Graph.from_host(synth.compose(w.nums))
    out = {}
    for flags in (0, 4):
        den = fbx.Graph.from_host(w.den, flags)
        assert (den.info["cluster_C"] > 0) == (flags == 4)
        loss, totals, st, grad = fbx.lfmmi_loss_grad(num, den, dev(w.emis), dev(lens))
        torch.cuda.synchronize()
        out[flags] = (loss.cpu().numpy(), grad.cpu().numpy(), st.cpu().numpy())
    ref = oracle.lfmmi_batch(synth.compose(w.nums), synth.compose([w.den]), w.emis, lens)
    for flags in (0, 4):
        loss, grad, st = out[flags]
        assert (st == 0).all()
        assert np.abs(grad - ref["grad"]).max() <= TOL_GRAD
        assert (np.abs(loss - ref["loss"]) / np.maximum(1, np.abs(ref["logZ_den"]))).max() <= TOL_LOGZ
    assert np.abs(out[0][1] - out[4][1]).max() <= 2 * TOL_GRAD


def test_paper_shape_den_n2(fbx):
    """N2: the paper's Table 1 denominator shape (3022 states, 50,984 arcs, D = 84;
    P:445-457), whose schedule exceeds one SM's shared memory — it runs split
    over a cluster.  Reduced B and N; oracle parity on logZ, posteriors, grad rows."""
    w = synth.make_paper_shape(seed=6, B=3, N=70, L_range=(10, 20))
    den, emis = w.den, w.emis
    lens = np.array([70, 70, 23], np.int32)
    r = run_fb(fbx, den, emis, lens, post="pdf")
    assert r["g"].info["cluster_C"] >= 2
    ref = oracle.fb_batch(den, emis, lens, post=True, post_pdf=True)
    assert (r["st"] == 0).all()
    check_logZ(r["logZ"], ref["logZ"], np.ones(3, bool))
    check_logZ(r["logZb"], ref["logZ"], np.ones(3, bool))
    assert np.abs(r["post"] - ref["post_pdf"]).max() <= TOL_POST


def test_paper_shape_lfmmi_n2(fbx):
    """N2 LF-MMI: paper-shape denominator (cluster kernel) + ≈454-state numerators."""
    import torch

    w = synth.make_paper_shape(seed=7, B=4, N=90, L_range=(30, 45))
    lens = np.array([90, 90, 60, 90], np.int32)
    num = fbx.Graph.from_host(synth.compose(w.nums))
    den = fbx.Graph.from_host(w.den)
    loss, totals, st, grad = fbx.lfmmi_loss_grad(num, den, dev(w.emis), dev(lens))
    torch.cuda.synchronize()
    ref = oracle.lfmmi_batch(synth.compose(w.nums), synth.compose([w.den]), w.emis, lens)
    st = st.cpu().numpy()
    assert (st == 0).all() and (ref["status"] == 0).all()
    assert np.abs(grad.cpu().numpy() - ref["grad"]).max() <= TOL_GRAD
    err = np.abs(loss.cpu().numpy() - ref["loss"]) / np.maximum(1, np.abs(ref["logZ_den"]))
    assert err.max() <= TOL_LOGZ


def test_host_entry_pipelined_matches_device_entry(fbx):
    """lfmmi_loss_grad_host (pinned host φ, double-buffered uploads on a copy stream)
    returns, call after call, exactly what lfmmi_loss_grad returns on device inputs."""
    import torch

    w = synth.make_c4(seed=23, B=4, N=40, L_range=(10, 20))
    num = fbx.Graph.from_host(synth.compose(w.nums))
    den = fbx.Graph.from_host(w.den)
    rng = np.random.default_rng(0)
    batches = [w.emis + np.float32(rng.normal(0, 0.5)) * (i % 2) for i in range(4)]
    lens = np.array([40, 33, 40, 21], np.int32)
    bufs = {}
    outs = []
    hosts = [torch.from_numpy(np.ascontiguousarray(e)).pin_memory() for e in batches]
    L = torch.from_numpy(lens).pin_memory()
    prev = None
    for e in hosts:  # call i+1 is enqueued before call i's results are read: uploads overlap compute
        cur = fbx.lfmmi_loss_grad_host(num, den, e, L, bufs)
        if prev is not None:
            torch.cuda.synchronize()
            outs.append(prev.clone())
        prev = cur
    torch.cuda.synchronize()
    outs.append(prev.clone())
    for e, out in zip(batches, outs):
        loss, totals, st, grad = fbx.lfmmi_loss_grad(num, den, dev(e), dev(lens))
        torch.cuda.synchronize()
        ref = np.concatenate([totals.cpu().numpy(), loss.cpu().numpy()])
        assert (out.numpy() == ref).all()


@pytest.mark.parametrize("cs", ["2,2", "4,4,1"])
def test_cluster_status_flags(fbx, cs, monkeypatch):
    """Fault handling through the cluster kernel: NaN emission, N_b = 0 and N_b > N_max
    flagged per sequence, the cluster's other sequences unaffected and exact."""
    import torch

    monkeypatch.setenv("FBX_CLUSTER", cs)
    w = synth.make_c4(seed=24, B=5, N=30, K=1500, nnz=10000, D=1000, L_range=(10, 20))
    emis = w.emis.copy()
    emis[1, 5, :] = np.nan
    lens = np.array([30, 30, 0, 31, 17], np.int32)
    num = fbx.Graph.from_host(synth.compose(w.nums))
    den = fbx.Graph.from_host(w.den)
    assert den.info["cluster_C"] > 0
    loss, totals, st, grad = fbx.lfmmi_loss_grad(num, den, dev(emis), dev(lens))
    torch.cuda.synchronize()
    st = st.cpu().numpy()
    assert st[0] == 0 and st[4] == 0
    assert st[1] & fbx.SEQ_NONFINITE_INPUT
    assert st[2] & fbx.SEQ_BAD_LENGTH and st[3] & fbx.SEQ_BAD_LENGTH
    g = grad.cpu().numpy()
    assert (g[1:4] == 0).all() and np.isfinite(g).all()
    ref = oracle.lfmmi_batch(synth.compose([w.nums[0], w.nums[4]]), synth.compose([w.den]), emis[[0, 4]],
                             lens[[0, 4]])
    assert np.abs(g[[0, 4]] - ref["grad"]).max() <= TOL_GRAD
    assert totals.cpu().numpy()[4] == 3


def test_cluster_determinism_and_batch_independence(fbx, monkeypatch):
    """k_fbc outputs are bitwise reproducible and an utterance's result does not depend
    on which sequences share its cluster (no cross-sequence arithmetic)."""
    monkeypatch.setenv("FBX_CLUSTER", "2,2")
    w = synth.make_c3(seed=9, B=5, N=40, K=1500, nnz=10000)
    lens = np.array([40, 31, 40, 7, 22], np.int32)
    r1 = run_fb(fbx, w.den, w.emis, lens)
    r2 = run_fb(fbx, w.den, w.emis, lens)
    assert (r1["post"] == r2["post"]).all() and (r1["logZ"] == r2["logZ"]).all()
    K = w.den.K
    perm = np.array([4, 2, 0, 3, 1])  # every utterance gets a different cluster partner
    r3 = run_fb(fbx, w.den, w.emis[perm].copy(), lens[perm])
    assert (r3["post"].reshape(5, 40, K) == r1["post"].reshape(5, 40, K)[perm]).all()
    assert (r3["logZ"] == r1["logZ"][perm]).all()


@pytest.mark.slow
def test_c5_pool_full_size_sampled(fbx):
    """configs[4] (C5): the bench's c5-weak batch — 128 utterances of the 1024-utterance pool,
    N_b log-normal in [50, 700] — through lfmmi_loss_grad; the oracle recomputes sampled
    utterances (the longest, the shortest, one in between) one by one."""
    import torch
    import bench

    w = bench.make_batch(0, 1, "c5-weak")
    num = fbx.Graph.from_host(synth.compose(w.nums))
    den = fbx.Graph.from_host(w.den)
    loss, totals, st, grad = fbx.lfmmi_loss_grad(num, den, dev(w.emis), dev(w.lengths))
    torch.cuda.synchronize()
    st = st.cpu().numpy()
    assert (st == 0).all()
    g = grad.cpu().numpy()
    L = w.lengths
    for b in (int(np.argmax(L)), int(np.argmin(L)), int(np.argsort(L)[len(L) // 2])):
        ref = oracle.lfmmi_batch(synth.compose([w.nums[b]]), synth.compose([w.den]), w.emis[b:b + 1], L[b:b + 1])
        assert abs(loss.cpu().numpy()[b] - ref["loss"][0]) <= TOL_LOGZ * max(1, abs(ref["logZ_den"][0]))
        assert np.abs(g[b, : L[b]] - ref["grad"][0, : L[b]]).max() <= TOL_GRAD
        assert (g[b, L[b]:] == 0).all()
    assert np.abs(g.sum(-1)).max() <= 1e-4


@pytest.mark.slow
def test_n2_full_size_sampled(fbx):
    """N2 at the paper's Table 1 size (B = 128, N = 700, den 3022 states / 50,984 arcs, cluster
    kernel) in the bench's launch configuration; sampled utterances against the oracle."""
    import torch

    w = synth.make_paper_shape(seed=6)
    num = fbx.Graph.from_host(synth.compose(w.nums))
    den = fbx.Graph.from_host(w.den)
    assert den.info["cluster_C"] > 0
    loss, totals, st, grad = fbx.lfmmi_loss_grad(num, den, dev(w.emis), dev(w.lengths))
    torch.cuda.synchronize()
    assert (st.cpu().numpy() == 0).all()
    g = grad.cpu().numpy()
    for b in (0, 127):
        ref = oracle.lfmmi_batch(synth.compose([w.nums[b]]), synth.compose([w.den]), w.emis[b:b + 1],
                                 w.lengths[b:b + 1])
        assert abs(loss.cpu().numpy()[b] - ref["loss"][0]) <= TOL_LOGZ * max(1, abs(ref["logZ_den"][0]))
        assert np.abs(g[b] - ref["grad"][0]).max() <= TOL_GRAD
    assert np.abs(g.sum(-1)).max() <= 1e-4


def test_lfmmi_multiwave_longest_first(fbx):
    """B > #SMs (the den recursion runs in several waves, the numerator has no idle SMs):
    ragged lengths through lfmmi_loss_grad against the oracle, utterance by utterance."""
    import torch

    B = 200
    w = synth.make_c4(seed=25, B=B, N=40, K=700, nnz=4000, D=500, L_range=(5, 12))
    rng = np.random.default_rng(25)
    lens = rng.integers(14, 41, B).astype(np.int32)
    num = fbx.Graph.from_host(synth.compose(w.nums))
    den = fbx.Graph.from_host(w.den)
    loss, totals, st, grad = fbx.lfmmi_loss_grad(num, den, dev(w.emis), dev(lens))
    torch.cuda.synchronize()
    assert (st.cpu().numpy() == 0).all()
    ref = oracle.lfmmi_batch(synth.compose(w.nums), synth.compose([w.den]), w.emis, lens)
    assert np.abs(grad.cpu().numpy() - ref["grad"]).max() <= TOL_GRAD
    err = np.abs(loss.cpu().numpy() - ref["loss"]) / np.maximum(1, np.abs(ref["logZ_den"]))
    assert err.max() <= TOL_LOGZ
