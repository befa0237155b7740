"""GEMV ring-depth / occupancy sweep (GFORS_QX_CFG) on config 6: per-product time of the fixed-point
dense GEMV from an eager replay (gfors_profile_blocks, class pdhg_qx)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os
sys.path.insert(0, %r)
import paper_2510_27117_b200 as gf
from gen import instances as G
inst = G.make_config(6, 1)
s = gf.Solver(0); s.load(inst); s.preprocess(precision=32, max_iter=30)
kw = dict(k_int=10, k_b=128, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)
s.profile_blocks(3, **kw)
s.profile_blocks(10, **kw)
act = s.profile_active()
ms, cnt = act["pdhg_qx"]
print(os.environ.get("GFORS_QX_CFG", "0"), "us per product (dense+final)", round(1000 * ms / (10 * 11), 2))
''' % ROOT
for cfg in ("0", "1", "2", "3"):
    env = dict(os.environ, GFORS_QX_CFG=cfg)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(out.stdout.strip() or out.stderr[-400:], flush=True)
