"""The linear objective over the sampler's list (k_obj_list: listed variables + the constant of the
p = 1 variables, sample_eval.cuh) equals the objective over every variable (k_obj_bits): whole runs
with option obj_list on and off produce the same incumbent sequence, bit for bit."""
import numpy as np
import pytest

from gen import instances as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gf():
    import paper_2510_27117_b200 as gf
    return gf


@pytest.mark.parametrize("fam,kw", [("setcover", dict(max_iters=800)), ("mis", dict(max_iters=600, sigma=0.5)),
                                    ("mkp", dict(max_iters=600)), ("setcover", dict(max_iters=400, k_b=1024)),
                                    ("setcover", dict(max_iters=400, k_b=64))])
def test_obj_list_same_runs(gf, fam, kw):
    inst = G.SMALL[fam](4)
    res = []
    for on in (1, 0):
        s = gf.Solver(0, options={"obj_list": on})
        s.load(inst)
        s.preprocess(precision=64)
        info = s.run(tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0, **kw)
        z, x, meta = s.best_incumbent()
        tr = s.trace()
        res.append((info["iters"], z, x, meta["found_iter"], meta["found_index"], tr[:, 6].copy()))
        s.close()
    a, b = res
    assert a[0] == b[0] and a[1] == b[1] and a[3] == b[3] and a[4] == b[4]
    assert (a[2] is None and b[2] is None) or np.array_equal(a[2], b[2])
    assert np.array_equal(a[5], b[5])
