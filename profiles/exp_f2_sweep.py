"""f2 experiment: facility location 512x2048 (slack form + TUReformulate), 30000 iterations per ρ/σ
setting, halting disabled; prints the incumbent and the last trace row (iteration, ρ, primal gap,
dual gap parts, binary gap).  The stationary primal gap 0.00138 with binary gap 0 under every setting
is the fixed point the sampler cannot leave (profiles/r02_f2_rho_sweep.txt)."""
import sys, time, json
sys.path.insert(0, ".")
import paper_2510_27117_b200 as gf
from gen import instances as G
nf, nc = 512, 2048
iters = 30000
inst = G.facility_location_slack(nf, nc, 1)
s = gf.Solver(0)
s.load(inst)
s.tu_reformulate(inst["tu_rows"], inst["tu_cols"])
s.preprocess(precision=32)
for kw in (dict(rho_max=1.0), dict(rho_max=0.1), dict(rho_max=0.01), dict(growth_T=1000.0), dict(rho_min=1e-4, rho_max=0.1), dict(sigma=0.5),):
    info = s.run(max_iters=iters, k_b=128, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0, time_limit_s=30.0, **kw)
    z, x, meta = s.best_incumbent()
    tr = s.trace()
    print(json.dumps(kw), f"iters={info['iters']} z={z} tti={meta['found_time_s'] if meta['has_incumbent'] else None} found_iter={meta['found_iter']} loop_s={info['elapsed_s']:.1f}",
          "last:", [round(v, 5) for v in tr[-1].tolist()] if len(tr) else None, flush=True)
