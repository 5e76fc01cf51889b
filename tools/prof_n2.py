"""A few N2 (paper-shape) den forward/backward launches for ncu capture / timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2112_00709_b200 as fbx
from paper_2112_00709_b200 import synth
w = synth.make_paper_shape(seed=6, B=int(os.environ.get("N2_B", "128")))
g = fbx.Graph.from_host(w.den)
print(g.info, flush=True)
e = torch.from_numpy(w.emis).cuda(); L = torch.from_numpy(w.lengths).cuda()
post = torch.empty(w.B, w.N_max, w.D, device="cuda")
def step():
    logZ, alpha, sc, st = fbx.fb_forward(g, e, L)
    fbx.fb_backward(g, e, L, alpha=alpha, status=st, post="pdf", post_out=post)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2): step()
torch.cuda.synchronize()
fbx.profile_enable(True); fbx.profile_reset()
for _ in range(3): step()
torch.cuda.synchronize()
print({k: round(v[1] / v[0], 3) for k, v in fbx.profile_collect().items()})
