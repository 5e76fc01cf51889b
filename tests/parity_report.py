"""Measured GPU-vs-oracle errors against the BASELINE gates, per configuration
(the numbers behind the parity tests' pass/fail): max |ΔlogZ| /
max(1, |logZ|), max |Δγ| (state posteriors), max |ΔΓ| (pdf level), max |Δgrad|,
and the fallback-row counter of the exp-factorised ⊕, for the primary (U[−10, 0))
and stress (log-softmax σ = 4, 8) emissions on den and numerator graphs, LF-MMI,
the cluster kernel and the AC6 input.  Writes one table to stdout.

    python -m tests.parity_report > profiles/r2_parity_errors.txt   (test infrastructure: imports oracle/)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: this is a parity report)
from paper_2112_00709_b200 import synth  # noqa: E402
from tests import helpers  # noqa: E402


def main():
    import torch

    import paper_2112_00709_b200 as fbx

    def dev(x):
        return torch.from_numpy(np.ascontiguousarray(x)).cuda()

    rows = []

    def fb_case(name, graph, emis, lens, flags=0, env=None):
        if env:
            os.environ.update(env)
        g = fbx.Graph.from_host(graph, flags)
        g.counters(reset=True)
        e, L = dev(emis), dev(lens.astype(np.int32))
        logZ, alpha, _, st = fbx.fb_forward(g, e, L)
        post, _, st2, _, _ = fbx.fb_backward(g, e, L, alpha=alpha, status=st.clone())
        ppdf, _, _, _, _ = fbx.fb_backward(g, e, L, alpha=alpha, status=st.clone(), post="pdf")
        torch.cuda.synchronize()
        ctr = g.counters()
        if env:
            for k in env:
                os.environ.pop(k, None)
        ref = oracle.fb_batch(graph, emis, lens, post=True, post_pdf=True)
        ok = ref["status"] == 0
        lz = logZ.cpu().numpy()
        ez = (np.abs(lz[ok] - ref["logZ"][ok]) / np.maximum(1, np.abs(ref["logZ"][ok]))).max()
        ep = np.abs(post.cpu().numpy().reshape(ref["post"].shape) - ref["post"]).max()
        eP = np.abs(ppdf.cpu().numpy() - ref["post_pdf"]).max()
        rows.append((name, ez, ep, eP, None, ctr["fallback_rows"] + ctr["fallback_rows_cluster"],
                     bool((st2.cpu().numpy() == ref["status"]).all())))

    def lf_case(name, w, lens, env=None):
        if env:
            os.environ.update(env)
        num, den = fbx.Graph.from_host(synth.compose(w.nums)), fbx.Graph.from_host(w.den)
        loss, totals, st, grad = fbx.lfmmi_loss_grad(num, den, dev(w.emis), dev(lens))
        torch.cuda.synchronize()
        if env:
            for k in env:
                os.environ.pop(k, None)
        ref = oracle.lfmmi_batch(synth.compose(w.nums), synth.compose([w.den]), w.emis, lens)
        ok = ref["status"] == 0
        el = (np.abs(loss.cpu().numpy()[ok] - ref["loss"][ok]) / np.maximum(1, np.abs(ref["logZ_den"][ok]))).max()
        eg = np.abs(grad.cpu().numpy() - ref["grad"]).max()
        rows.append((name, el, None, None, eg, None, bool((st.cpu().numpy() == ref["status"]).all())))

    for kind in ("uniform", "softmax4", "softmax8"):
        w = synth.make_c3(seed=3, B=4, N=80, kind=kind, K=3000, nnz=20000)
        fb_case(f"C3 den (K=3000, 20k arcs) {kind}", w.den, w.emis, np.array([80, 80, 41, 80], np.int32))
    for kind in ("uniform", "softmax4", "softmax8"):
        w = synth.make_c2(seed=2, B=16, kind=kind)
        fb_case(f"C2 numerators (exact) {kind}", synth.compose(w.nums), w.emis, w.lengths)
    for kind in ("uniform", "softmax4", "softmax8"):
        w = synth.make_c4(seed=4, B=6, N=120, kind=kind, L_range=(20, 60))
        lf_case(f"C4 LF-MMI {kind}", w, np.array([120, 120, 90, 61, 120, 100], np.int32))
    w = synth.make_c4(seed=21, B=5, N=48, K=1500, nnz=10000, D=1000, kind="softmax4", L_range=(10, 20))
    fb_case("cluster (4,4) no-p, softmax4", w.den, w.emis, np.array([48, 1, 30, 48, 17], np.int32),
            env={"FBX_CLUSTER": "4,4,1"})
    w = synth.make_paper_shape(seed=7, B=4, N=90, L_range=(30, 45))
    lf_case("N2 LF-MMI (cluster den)", w, np.array([90, 90, 60, 90], np.int32))
    rng = np.random.Generator(np.random.PCG64(61))
    Ls = rng.integers(20, 60, 16)
    gs = [synth.numerator_graph(rng, int(L), 200, "random", alt_p=0.0) for L in Ls]
    for kind in ("uniform", "softmax8"):
        em = synth.emissions(rng, 16, int(Ls.max()), 200, kind=kind)
        fb_case(f"tight numerators N_b = L_b, forced factored, {kind}", synth.compose(gs), em, Ls.astype(np.int32),
                flags=fbx.GRAPH_FORCE_FACTORED)
    g10 = helpers.left_to_right(10)
    e10 = np.random.default_rng(71).uniform(-100, -50, (2, 1000, 10)).astype(np.float32)
    for flags, nm in ((0, "auto (exact)"), (2, "forced factored")):
        fb_case(f"AC6 N=1000 phi in [-100,-50], {nm}", g10, e10, np.array([1000, 777], np.int32), flags=flags)

    print("gates (BASELINE north_star): logZ rel 1e-5, gamma 1e-5, grad 1e-5; sigma=8 and forced-factored AC6 are "
          "reported stress cases (DESIGN.md L15, L20)")
    print(f"{'configuration':52s} {'logZ/loss rel':>13s} {'max|dγ|':>9s} {'max|dΓ|':>9s} {'max|dgrad|':>10s} "
          f"{'fallback rows':>13s} status==oracle")
    f = lambda v: "—" if v is None else f"{v:.2e}"
    for name, ez, ep, eP, eg, fb, sok in rows:
        print(f"{name:52s} {f(ez):>13s} {f(ep):>9s} {f(eP):>9s} {f(eg):>10s} {('—' if fb is None else str(fb)):>13s} {sok}")


if __name__ == "__main__":
    main()
