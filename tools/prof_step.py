"""Run a few C3 (den FB + posteriors) or C4 (LF-MMI) steps for ncu capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2112_00709_b200 as fbx
from paper_2112_00709_b200 import synth

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if which == "c3":
    w = synth.make_c3(seed=3)
    g = fbx.Graph.from_host(w.den)
    e = torch.from_numpy(w.emis).cuda(); L = torch.from_numpy(w.lengths).cuda()
    alpha = torch.empty(128 * 500 * w.den.K, device="cuda")
    sc = torch.empty(128, 500, dtype=torch.float64, device="cuda")
    post = torch.empty_like(alpha)
    for _ in range(steps):
        logZ, _, _, st = fbx.fb_forward(g, e, L, alpha=alpha, alpha_scale=sc)
        fbx.fb_backward(g, e, L, alpha=alpha, status=st, post="state", post_out=post)
else:
    w = synth.make_c4(seed=4)
    num = fbx.Graph.from_host(synth.compose(w.nums)); den = fbx.Graph.from_host(w.den)
    e = torch.from_numpy(w.emis).cuda(); L = torch.from_numpy(w.lengths).cuda()
    grad = torch.empty_like(e)
    ws = torch.empty(fbx.workspace_bytes(num, den, 128, 500), dtype=torch.uint8, device="cuda")
    for _ in range(steps):
        fbx.lfmmi_loss_grad(num, den, e, L, grad, ws)
torch.cuda.synchronize()
print("done")
