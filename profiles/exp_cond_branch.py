"""Graph-mode block time on config 5 (fp32, k_b = 128) with the mode branches as launched kernels that
exit early (cond_branch = 0, default) and as graph conditional nodes (cond_branch = 1): CUDA events
around one gfors_run of K blocks from x0, K = 20 and 200."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2510_27117_b200 as gf  # noqa: E402
from gen import instances as G  # noqa: E402
inst = G.make_config(5, 1)
kw = dict(k_int=10, k_b=128, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0, time_limit_s=1e9)
for cb in (0, 1, 0, 1):
    s = gf.Solver(0, options={"cond_branch": cb})
    s.load(inst)
    s.preprocess(precision=32)
    s.run(max_iters=50, **kw)
    for K in (20, 200):
        info = s.run(max_iters=10 * K, **kw)
        print(f"cond_branch={cb} K={K} ms/block={1e3 * info['elapsed_s'] / K:.3f} launches={info['launches']}", flush=True)
    s.close()
