"""Small invocations of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck): C1 (dense K = 3, exact mode), C2-style
numerators (G = B, exact), a C3-shaped den (factored + TMA rows, 1024 threads),
lfmmi_loss_grad (den + k_fb_num + k_add_num + k_totals), the cluster kernel
k_fbc ((2,2) and (4,4) no-p with the split phase A), Viterbi, the literal
strategy, fb_posteriors and fb_gap.  Sizes are tiny (N ≤ 12) so racecheck
finishes; outputs are checked against nothing here (the parity tests do that).

    compute-sanitizer --tool memcheck python tools/sanitize.py [part ...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(parts):
    import torch

    import paper_2112_00709_b200 as fbx
    from paper_2112_00709_b200 import synth

    torch.cuda.set_device(0)

    def dev(x):
        return torch.from_numpy(np.ascontiguousarray(x)).cuda()

    def fb(graph, emis, lens, flags=0):
        g = fbx.Graph.from_host(graph, flags)
        e, L = dev(emis), dev(lens.astype(np.int32))
        logZ, alpha, ascale, st = fbx.fb_forward(g, e, L)
        post, _, st2, beta, bscale = fbx.fb_backward(g, e, L, alpha=alpha, status=st.clone(), want_beta=True)
        fbx.fb_backward(g, e, L, alpha=alpha, status=st.clone(), post="pdf")
        fbx.fb_posteriors(g, alpha, beta, L, st2, len(lens), emis.shape[1], pdf_level=True)
        fbx.fb_gap(g, alpha, ascale, beta, bscale, logZ, L, st2)
        torch.cuda.synchronize()
        return g

    if "c1" in parts:
        ws = [synth.make_c1(s) for s in range(4)]
        comp = synth.compose([w.den for w in ws])
        emis = np.concatenate([w.emis for w in ws])
        for flags in (0, 1, 2):
            fb(comp, emis, np.array([6, 1, 4, 6]), flags)
        g = fbx.Graph.from_host(comp)
        fbx.fb_viterbi(g, dev(emis), dev(np.array([6, 1, 4, 6], np.int32)))
        for sr in (0, 1, 2):
            fbx.fb_forward_literal(g, dev(emis), dev(np.array([6, 1, 4, 6], np.int32)), sr)
        torch.cuda.synchronize()
    if "c2" in parts:
        rng = np.random.Generator(np.random.PCG64(2))
        nums = [synth.numerator_graph(rng, int(L), 300, "identity") for L in (4, 6, 5, 3)]
        fb(synth.compose(nums), synth.emissions(rng, 4, 12, 300), np.array([12, 7, 12, 2], np.int32))
    if "c3" in parts:
        w = synth.make_c3(seed=3, B=2, N=8)
        fb(w.den, w.emis, np.array([8, 5], np.int32))
    if "lfmmi" in parts:
        w = synth.make_c4(seed=4, B=3, N=10, L_range=(3, 5))
        num = fbx.Graph.from_host(synth.compose(w.nums))
        den = fbx.Graph.from_host(w.den)
        fbx.lfmmi_loss_grad(num, den, dev(w.emis), dev(np.array([10, 7, 10], np.int32)))
        torch.cuda.synchronize()
    if "cluster" in parts:
        for cs in ("2,2", "4,4,1"):
            os.environ["FBX_CLUSTER"] = cs
            w = synth.make_c4(seed=21, B=5, N=8, K=1500, nnz=10000, D=1000, L_range=(2, 4))
            fb(w.den, w.emis, np.array([8, 1, 5, 8, 3], np.int32))
            num = fbx.Graph.from_host(synth.compose(w.nums))
            den = fbx.Graph.from_host(w.den)
            fbx.lfmmi_loss_grad(num, den, dev(w.emis), dev(np.array([8, 4, 5, 8, 3], np.int32)))
            torch.cuda.synchronize()
        os.environ.pop("FBX_CLUSTER", None)
    print("sanitize: done", parts, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "lfmmi", "cluster"])
