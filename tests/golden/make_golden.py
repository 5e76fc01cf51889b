"""Writes tests/golden/c1_mp50.json: C1 (dense K=3, N=6, seeds
0..19) brute-forced over all 3^6 paths in mpmath at 50 digits
(P:79-83 definition).  Calls only oracle.brute and the shared
generator; run:  python tests/golden/make_golden.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import brute  # noqa: E402
from paper_2112_00709_b200 import synth  # noqa: E402

cases = []
for seed in range(20):
    w = synth.make_c1(seed)
    logZ, post = brute.brute_force_mp(w.den, w.emis[0])
    cases.append({"seed": seed, "logZ": logZ, "post": post.tolist()})
out = {"source": "brute-force path enumeration, mpmath 50 digits (P:79-83, S:400-403)",
       "generator": "paper_2112_00709_b200.synth.make_c1(seed)", "cases": cases}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c1_mp50.json"), "w") as f:
    json.dump(out, f, indent=1)
