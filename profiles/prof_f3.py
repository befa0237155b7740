"""Kernel-capture driver for the Alg. 4 sampler (next row f3) under ncu: config 8 (3D assignment
n = 64), fp32, two rounds of the customised sampler from a fixed p, then their evaluation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2510_27117_b200 as gf  # noqa: E402
from gen import instances as G  # noqa: E402

inst = G.make_config(8, 1)
s = gf.Solver(0)
s.load(inst)
s.preprocess(precision=32)
p = G.p_vectors(inst["n"], 1)["unif"]
for r in range(2):
    bits = s.sample_assign3d(p, 1, r, 0, 2, inst["a3_n"])
    s.eval(bits)
print("prof_f3 ok")
