"""Indicator trace of facility location 64 x 256 with TUReformulate (fp64, halting off): how the
primal gap, dual gap and binary gap evolve, and how many rows the rounded x_k violates."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2510_27117_b200 as gf  # noqa: E402
from gen import instances as G  # noqa: E402
from oracle.tu import tu_reformulate  # noqa: E402

nf, nc = (int(v) for v in os.environ.get("SIZE", "64x256").split("x"))
inst = G.facility_location(nf, nc, 1)
for tu in (True, False):
    s = gf.Solver(0)
    s.load(inst)
    if tu:
        s.tu_reformulate(inst["tu_rows"], inst["tu_cols"])
    s.preprocess(precision=64)
    info = s.run(max_iters=int(os.environ.get("MAXIT", "50000")), tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0,
                 stall_rel=-1.0, trace_cap=100000)
    tr = s.trace()
    x = s.get_state()[0]
    print("TU" if tu else "noTU", "iters", info["iters"], "frac(0<x<1)", float(np.mean((x > 1e-6) & (x < 1 - 1e-6))))
    for k in (0, 9, 49, 99, 499, 999, 2999, len(tr) - 1):
        if k < len(tr):
            r = tr[k]
            print(f"  it {int(r[0]):6d} rho {r[1]:.4g} pgap {r[2]:.3e} sx {r[3]:.3e} sy {r[4]:.3e} bgap {r[5]:.3e} z {r[6]}")
    s.close()
