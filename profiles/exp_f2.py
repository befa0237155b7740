"""Experiment driver (next row f2): facility location with and without TUReformulate on one GPU,
several sizes, SPEC default halting bounded by MAXIT iterations; prints one JSON line per run."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_27117_b200 as gf  # noqa: E402
from gen import instances as G  # noqa: E402

MAXIT = int(os.environ.get("MAXIT", "60000"))
sizes = [tuple(map(int, s.split("x"))) for s in os.environ.get("SIZES", "64x256,128x512,512x2048").split(",")]
for nf, nc in sizes:
    inst = G.facility_location(nf, nc, 1)
    for tu in (True, False):
        s = gf.Solver(0)
        s.load(inst)
        t0 = time.perf_counter()
        if tu:
            s.tu_reformulate(inst["tu_rows"], inst["tu_cols"])
        t_tu = time.perf_counter() - t0
        s.preprocess(precision=int(os.environ.get("PREC", "32")))
        kw = {} if os.environ.get("HALT", "1") == "1" else dict(tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0,
                                                                stall_rel=-1.0)
        if "SIGMA" in os.environ:
            kw["sigma"] = float(os.environ["SIGMA"])
        info = s.run(max_iters=MAXIT, k_b=int(os.environ.get("KB", "128")), **kw)
        z, x, meta = s.best_incumbent(want_x=False)
        print(json.dumps({"nf": nf, "nc": nc, "tu": tu, "sigma": kw.get("sigma", 0.99), "tu_s": round(t_tu, 3), "iters": info["iters"],
                          "halt": info["halt_reason"], "z": z if meta["has_incumbent"] else None,
                          "found_iter": meta["found_iter"], "tti_s": meta["found_time_s"] if meta["has_incumbent"] else None,
                          "loop_s": info["elapsed_s"]}), flush=True)
        s.close()
