"""f1 dense-K: config 3 (MKP n = 1e5, m = 50, density 0.5) per-class ms per Alg. 1 block with the
integer rows on tensor cores (option dense_k = 1, default here) and on the CUDA-core integer path
(dense_k = 0); eager replay with per-launch CUDA events (gfors_profile_blocks), 50 blocks from x0."""
import json
import sys

sys.path.insert(0, ".")
import paper_2510_27117_b200 as gf  # noqa: E402
from gen import instances as G  # noqa: E402

inst = G.make_config(3, 1)
for kb in (128, 1024):
    for dk in (1, 0):
        s = gf.Solver(0, options={"dense_k": dk})
        s.load(inst)
        s.preprocess(precision=32)
        ms = s.profile_blocks(50, k_int=10, k_b=kb, max_iters=500)
        act = s.profile_active()
        print(json.dumps({"k_b": kb, "dense_k": dk, "feas_ms_per_block": round(ms.get("feas", 0), 4),
                          "obj_tc_ms_per_block": round(ms.get("obj_tc", 0), 4),
                          "block_ms": round(sum(ms.values()), 4)}), flush=True)
        s.close()
