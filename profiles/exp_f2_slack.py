"""f2 experiment (reading R24 rev.): facility location (nf, nc) in the all-equality slack form with
TUReformulate (general, unit-triangular B_JI) against the inequality form without TU, fixed iteration
budgets, halting disabled.  Prints z_best, time to incumbent, candidates/s."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2510_27117_b200 as gf  # noqa: E402
from gen import instances as G  # noqa: E402

nf, nc = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (512, 2048)
for iters in (3000, 30000):
    for form in ("slack_tu", "ineq_no_tu", "ineq_tu_gub"):
        inst = G.facility_location_slack(nf, nc, 1) if form == "slack_tu" else G.facility_location(nf, nc, 1)
        s = gf.Solver(0)
        s.load(inst)
        t0 = time.time()
        if form != "ineq_no_tu":
            s.tu_reformulate(inst["tu_rows"], inst["tu_cols"])
        ttu = time.time() - t0
        s.preprocess(precision=32)
        info = s.run(max_iters=iters, k_b=128, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)
        z, x, meta = s.best_incumbent()
        print(f"{nf}x{nc} {form:12s} iters={iters} n={s.n} m={s.m} tu_s={ttu:.2f} z={z} "
              f"tti={meta['found_time_s'] if meta['has_incumbent'] else None} found_iter={meta['found_iter']} "
              f"loop_s={info['elapsed_s']:.3f} cand/s={info['candidates'] / info['elapsed_s']:.0f}", flush=True)
        s.close()
