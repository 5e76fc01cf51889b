"""Exact-fallback counters (fb_graph_counters) of one N2 LF-MMI call: how many (row, sequence)
evaluations of the exp-factorised ⊕ left [2^-80, 2^120] and took the exact max-then-sum."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2112_00709_b200 as fbx
from paper_2112_00709_b200 import synth

w = synth.make_paper_shape()
den = fbx.Graph.from_host(w.den)
num = fbx.Graph.from_host(synth.compose(w.nums))
e, L = torch.from_numpy(w.emis).cuda(), torch.from_numpy(w.lengths).cuda()
den.counters(reset=True)
fbx.lfmmi_loss_grad(num, den, e, L)
torch.cuda.synchronize()
print("N2 den counters", den.counters(), "row evaluations per pass:", 128 * 700 * w.den.K)
