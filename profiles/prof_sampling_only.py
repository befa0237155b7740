"""Sampling-only candidates/s on config 5 (RandSampleStep + EvalBest + argmin at fixed p, no PDHG) per
p-distribution and k_b (gfors_sample_eval_timed, device time of 10 rounds)."""
import json
import sys
sys.path.insert(0, ".")
import paper_2510_27117_b200 as gf  # noqa: E402
from gen import instances as G  # noqa: E402
inst = G.make_config(5, 1)
s = gf.Solver(0)
s.load(inst)
s.preprocess(precision=32)
pv = G.p_vectors(inst["n"], 5)
out = {}
for name in ("unif", "mix"):
    out[name] = {}
    for kb in (64, 128, 512, 1024, 4096):
        s.sample_eval_timed(pv[name], 20251030, kb // 64, 1)  # warm-up (lazy module loading of new instances)
        out[name][kb] = round(10 * kb / (s.sample_eval_timed(pv[name], 20251030, kb // 64, 10) * 1e-3))
    print(name, json.dumps(out[name]), flush=True)
