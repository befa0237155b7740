"""Where the e2e time of config 5 goes: host->device load (gfors_load from pinned host arrays),
Preprocess (power iterations), run of K blocks, best_incumbent."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_27117_b200 as gf  # noqa: E402
from gen import instances as G  # noqa: E402

inst = G.make_config(5, 1)
host = {k: (torch.from_numpy(np.ascontiguousarray(v)).pin_memory().numpy() if isinstance(v, np.ndarray) else v)
        for k, v in inst.items()}
for rep in range(6):
    s = gf.Solver(0)
    s.set_option("load_timing", 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); s.load(host); torch.cuda.synchronize(); t1 = time.perf_counter()
    sc = s.preprocess(precision=32); torch.cuda.synchronize(); t2 = time.perf_counter()
    s.run(max_iters=2000, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0); torch.cuda.synchronize(); t3 = time.perf_counter()
    s.best_incumbent(); t4 = time.perf_counter()
    print(f"load {t1-t0:.3f} s, preprocess {t2-t1:.3f} s, run 200 blocks {t3-t2:.3f} s, best {t4-t3:.3f} s", flush=True)
    s.close()
