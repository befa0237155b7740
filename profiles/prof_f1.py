"""Kernel-capture driver for the dense-Q kernels (next row f1) under ncu: config 6 (max cut n=20480),
fp32 iterates, two hook-mode PDHG steps (dense GEMV + primal) and one k_b=128 objective batch
(unpack + tcgen05 kernel).  Usage: ncu ... python profiles/prof_f1.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2510_27117_b200 as gf  # noqa: E402
from gen import instances as G  # noqa: E402

inst = G.make_config(6, 1)
s = gf.Solver(0)
s.load(inst)
s.preprocess(precision=int(os.environ.get("PREC", "32")), max_iter=20)
n = inst["n"]
rng = np.random.default_rng(0)
x = rng.random(n)
s.set_state(x, x, np.zeros(0))
s.step(2, 1e-3, 0.99 ** 0.5, 0.99 ** 0.5)
p = G.p_vectors(n, 1)["unif"]
bits = s.sample(p, 1, 0, 0, 2)
for _ in range(2):
    s.eval(bits)
print("prof_f1 ok")
