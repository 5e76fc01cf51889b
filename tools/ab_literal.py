"""A/B: the paper's literal strategy (fb_forward_literal, one block-diagonal batch
SpMV launch per frame, float64) vs the fused forward (fb_forward) on C3 / C4 / N2
denominators at full size.  Prints device ms per forward pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2112_00709_b200 as fbx
from paper_2112_00709_b200 import synth


def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for name in sys.argv[1:] or ["c3", "paper"]:
    w = synth.make_c3(seed=3) if name == "c3" else synth.make_paper_shape(seed=6)
    g = fbx.Graph.from_host(w.den)
    e = torch.from_numpy(w.emis).cuda(); L = torch.from_numpy(w.lengths).cuda()
    frames = float(w.lengths.sum())
    t_lit = timeit(lambda: fbx.fb_forward_literal(g, e, L, fbx.SEMIRING_LOG))
    t_fused = timeit(lambda: fbx.fb_forward(g, e, L))
    z_lit = fbx.fb_forward_literal(g, e, L, fbx.SEMIRING_LOG).cpu().numpy()
    z = fbx.fb_forward(g, e, L)[0].cpu().numpy()
    print(f"{name}: literal LOG forward {t_lit:.2f} ms ({frames / t_lit * 1e3:.3e} seq-frames/s) | "
          f"fused fb_forward {t_fused:.2f} ms ({frames / t_fused * 1e3:.3e} seq-frames/s) | "
          f"speedup {t_lit / t_fused:.1f}x | max rel logZ diff {np.max(np.abs(z - z_lit) / np.abs(z_lit)):.1e}",
          flush=True)
