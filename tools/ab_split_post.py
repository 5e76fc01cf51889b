"""A/B: fused posterior epilogue in the backward vs backward-with-β̂ + standalone k_posteriors (C4 den, pdf level)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2112_00709_b200 as fbx
from paper_2112_00709_b200 import synth

def timeit(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))

w = synth.make_c4(seed=4)
g = fbx.Graph.from_host(w.den)
e = torch.from_numpy(w.emis).cuda(); L = torch.from_numpy(w.lengths).cuda()
B, N, K, D = 128, 500, w.den.K, w.D
logZ, alpha, sc, st = fbx.fb_forward(g, e, L)
post = torch.empty(B, N, D, device="cuda")
beta = torch.empty(B * N * K, device="cuda"); bsc = torch.empty(B, N, dtype=torch.float64, device="cuda")
t_fused = timeit(lambda: fbx.fb_backward(g, e, L, alpha=alpha, status=st.clone(), post="pdf", post_out=post))
t_bwd = timeit(lambda: fbx.fb_backward(g, e, L, alpha=alpha, status=st.clone(), want_beta=True, post=None))
p, zb, st2, beta, bsc = fbx.fb_backward(g, e, L, alpha=alpha, status=st.clone(), want_beta=True, post=None)
t_post = timeit(lambda: fbx.fb_posteriors(g, alpha, beta, L, st2, B, N, pdf_level=True, post=post))
print(f"fused bwd+pdf post {t_fused:.3f} ms | bwd (beta stored) {t_bwd:.3f} ms + k_posteriors(pdf) {t_post:.3f} ms = {t_bwd + t_post:.3f} ms")
