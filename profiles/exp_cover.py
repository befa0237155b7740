"""Per-class time of one Alg. 1 block on config 5 with the cover completion (eager replay)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_27117_b200 as gf  # noqa: E402
from gen import instances as G  # noqa: E402

s = gf.Solver(0)
s.load(G.make_config(5, 1))
s.preprocess(precision=32)
kw = dict(k_int=10, k_b=128, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0, complete=1)
for blocks in (5, 50):
    prof = s.profile_blocks(blocks, **kw)
    print(blocks, {k: round(v, 3) for k, v in prof.items() if v})
