"""Evaluator timing on config 5 (bench workload): per-kernel-class ms of the first 20 Alg. 1 blocks
from x0 (the window bench.py times) and of blocks 180-200, via gfors_profile_blocks (eager replay,
CUDA events around every launch).  Usage: python profiles/prof_eval.py [blocks]"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2510_27117_b200 as gf  # noqa: E402
from gen import instances as G  # noqa: E402

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 20
t = time.time()
inst = G.make_config(5, 1)
s = gf.Solver(0)
s.load(inst)
s.preprocess(precision=32)
print("load+prep", round(time.time() - t, 1), "s", flush=True)
kw = dict(k_int=10, k_b=128, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)
out = {}
for nb in (blocks,):
    ms = s.profile_blocks(nb, max_iters=10 * nb, **kw)
    act = s.profile_active()
    out[f"first_{nb}_blocks_ms_per_block"] = {k: round(v, 4) for k, v in ms.items() if v > 0}
    out[f"first_{nb}_blocks_active"] = {k: (round(a, 3), n) for k, (a, n) in act.items() if n}
print(json.dumps(out, indent=1))
