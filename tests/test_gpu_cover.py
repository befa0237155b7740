"""Cover completion (reading R27; csrc/cover.cuh) against the oracle: bit-exact completion of a batch,
identical fp64 runs with complete = 1, and at full size (config 5) a feasible incumbent within a few
blocks, recomputed exactly by the oracle."""
import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gf():
    import paper_2510_27117_b200 as gf
    return gf


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("fam,nw", [("setcover", 1), ("setcover", 3), ("general", 2), ("bqp", 2)])
def test_cover_complete_bit_exact(gf, prec, fam, nw):
    inst = G.SMALL[fam](8)
    s = gf.Solver(0)
    s.load(inst)
    s.preprocess(precision=prec)
    o = O.Oracle(inst)
    rng = np.random.default_rng(nw)
    p = np.round(rng.random(inst["n"]) * 0.3, 2).astype(np.float32).astype(np.float64)
    bits = O.sample(p, 4, 2, 0, nw)
    a = s.cover_complete(p, bits)
    b = o.cover_complete(p, bits)
    assert np.array_equal(a, b)
    fg, zg = s.eval(a)
    fo, zo = o.eval(b)
    assert np.array_equal(fg, fo) and np.array_equal(zg, zo)
    if fam == "setcover":
        assert fg.all()


@pytest.mark.parametrize("graph", [1, 0])
def test_cover_run_parity_fp64(gf, graph):
    inst = G.SMALL["setcover"](9)
    s = gf.Solver(0)
    s.load(inst)
    s.preprocess()
    o = O.Oracle(inst)
    o.preprocess()
    kw = dict(max_iters=600, k_b=128, complete=1)
    ig = s.run(use_graph=graph, **kw)
    io = o.run(**kw)
    assert ig["iters"] == io["iters"] and ig["halt_reason"] == io["halt_reason"]
    zg, xg, mg = s.best_incumbent()
    zo, xo = o.best()
    assert zg == zo and np.array_equal(xg, xo)
    assert (mg["found_iter"], mg["found_index"]) == (io["found_iter"], io["found_index"])


def test_config5_cover_completion_incumbent(gf):
    """BASELINE config 5 (set cover 5M x 1M), bench launch configuration with complete = 1: an
    incumbent after the first sampling block, feasible with the reported objective (oracle)."""
    inst = G.make_config(5, 1)
    s = gf.Solver(0)
    s.load(inst)
    s.preprocess(precision=32)
    info = s.run(max_iters=50, k_int=10, k_b=128, complete=1, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0,
                 stall_rel=-1.0)
    z, x, meta = s.best_incumbent()
    assert meta["has_incumbent"] and meta["found_iter"] <= 50
    f, zz = O.Oracle(inst).eval_point(x)
    assert f and zz == z
