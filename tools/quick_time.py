"""Quick device timing of the C3 (den FB + posteriors) and C4 (LF-MMI) full-size steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2112_00709_b200 as fbx
from paper_2112_00709_b200 import synth


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


which = sys.argv[1:] or ["c3", "c4"]
if "c3" in which:
    t0 = time.time()
    w = synth.make_c3(seed=3)
    print("gen c3", time.time() - t0, flush=True)
    g = fbx.Graph.from_host(w.den)
    print("graph", g.info, flush=True)
    e = torch.from_numpy(w.emis).cuda(); L = torch.from_numpy(w.lengths).cuda()
    B, N, K = 128, 500, w.den.K
    alpha = torch.empty(B * N * K, device="cuda"); sc = torch.empty(B, N, dtype=torch.float64, device="cuda")
    post = torch.empty(B * N * K, device="cuda")
    def step():
        logZ, _, _, st = fbx.fb_forward(g, e, L, alpha=alpha, alpha_scale=sc)
        fbx.fb_backward(g, e, L, alpha=alpha, status=st, post="state", post_out=post)
    ms = timeit(step)
    fbx.profile_enable(True); fbx.profile_reset()
    for _ in range(10): step()
    torch.cuda.synchronize()
    print("profile", {k: round(v[1] / v[0], 4) for k, v in fbx.profile_collect().items()}); fbx.profile_enable(False)
    print(f"C3 fwd+bwd+post: {ms:.3f} ms  -> {64000/ms*1e3:.3e} seq-frames/s", flush=True)
    del alpha, post, e
if "c4" in which:
    t0 = time.time()
    w = synth.make_c4(seed=4)
    print("gen c4", time.time() - t0, flush=True)
    num = fbx.Graph.from_host(synth.compose(w.nums), int(os.environ.get("FBX_NUM_FLAGS", "0")))
    den = fbx.Graph.from_host(w.den, int(os.environ.get("FBX_DEN_FLAGS", "0")))
    print("num", num.info, "\nden", den.info, flush=True)
    e = torch.from_numpy(w.emis).cuda(); L = torch.from_numpy(w.lengths).cuda()
    grad = torch.empty_like(e)
    ws = torch.empty(fbx.workspace_bytes(num, den, 128, 500), dtype=torch.uint8, device="cuda")
    loss = torch.empty(128, dtype=torch.float64, device="cuda"); tot = torch.empty(5, dtype=torch.float64, device="cuda")
    st = torch.empty(128, dtype=torch.int32, device="cuda")
    step = lambda: fbx.lfmmi_loss_grad(num, den, e, L, grad, ws, loss, tot, st)
    ms = timeit(step)
    fbx.profile_enable(True); fbx.profile_reset()
    for _ in range(10): step()
    torch.cuda.synchronize()
    print("profile", {k: round(v[1] / v[0], 4) for k, v in fbx.profile_collect().items()}); fbx.profile_enable(False)
    print(f"C4 lfmmi: {ms:.3f} ms  -> {64000/ms*1e3:.3e} seq-frames/s  totals {tot.cpu().numpy()}", flush=True)
