"""Dense integer rows of K on tensor cores ("int8 MMA for MKP's K.X"; knapsack rows,
PAPER L221-227; EvalBest "via matrix multiplications"): the general integer rows stored as
int8 and multiplied with the unpacked samples by the split-K instance of the tcgen05 kernel
(exact int32 sums).  Feasibility and objective bit-exact against the oracle; identical to the CUDA-core
integer path of the same library; MKP at full size (config 3) on sampled lanes."""
import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gf():
    import paper_2510_27117_b200 as gf
    return gf


def _solver(gf, inst, dense_k):
    s = gf.Solver(0, options={"dense_k": dense_k})
    s.load(inst)
    s.preprocess()
    return s


@pytest.mark.parametrize("fam", ["mkp", "general"])
@pytest.mark.parametrize("nw", [1, 2, 4, 8])
def test_dense_k_eval_bit_exact(gf, fam, nw):
    """k_b = 64..512 (N = 64..256 per pass, two passes at 512): feasibility masks and objectives equal
    the oracle's, with the tensor-core path forced and with it off."""
    inst = G.SMALL[fam](21)
    o = O.Oracle(inst)
    p = G.p_vectors(inst["n"], 4)["mix"]
    bits = O.sample(p, 9, 2, 0, nw)
    fo, zo = o.eval(bits)
    for dk in (1, 0):
        s = _solver(gf, inst, dk)
        fg, zg = s.eval(bits)
        assert np.array_equal(fg, fo) and np.array_equal(zg, zo)


def test_dense_k_near_capacity_rows(gf):
    """Lanes whose knapsack sums sit exactly at the capacity (feasible) and one unit above it
    (infeasible), on rows with negative canonical coefficients (LE rows negated to GE) and an EQ row:
    the int32 tensor-core sums decide the boundary exactly."""
    from tests.util import inst_from_dense
    n = 2000
    w = np.ones((3, n))
    w[1, ::2] = 2.0
    w[2, :] = 0.0
    w[2, :100] = 1.0
    inst = inst_from_dense(w, [1000.0, 1500.0, 50.0], [-1, -1, 0], np.arange(n) % 7 - 3.0)
    bits = np.zeros((n, 2), dtype=np.uint64)
    lanes = []
    for l, k in enumerate([1000, 1001, 999, 0, 50, 60]):
        x = np.zeros(n, dtype=np.uint64)
        x[:k] = 1
        bits[:, l // 64] |= x << np.uint64(l % 64)
        lanes.append(l)
    rng = np.random.default_rng(1)
    bits[:, 1] |= (rng.random((n,)) < 0.3).astype(np.uint64) * np.uint64(0xFFFF0000)
    o = O.Oracle(inst)
    fo, zo = o.eval(bits)
    s = _solver(gf, inst, 1)
    fg, zg = s.eval(bits)
    assert np.array_equal(fg, fo) and np.array_equal(zg, zo)
    assert fo[0] == 0 and fo[3] == 0 and fo[4] == 1  # row 2 is EQ 50: only the 50-lane holds it


def test_dense_k_run_parity(gf):
    """Whole fp64 runs on the MKP family: tensor-core feasibility gives the same incumbent sequence as
    the oracle."""
    inst = G.SMALL["mkp"](8)
    s = _solver(gf, inst, 1)
    o = O.Oracle(inst)
    o.preprocess()
    kw = dict(max_iters=1500, k_b=128)
    ig = s.run(**kw)
    io = o.run(**kw)
    assert ig["iters"] == io["iters"] and ig["halt_reason"] == io["halt_reason"]
    zg, xg, mg = s.best_incumbent()
    zo, xo = o.best()
    assert zg == zo and np.array_equal(xg, xo)


def test_dense_k_config3_full_size(gf):
    """Config 3 (MKP n = 1e5, m = 50, density 0.5) at full size: sampled lanes' feasibility and objective
    against the oracle evaluated one lane at a time; all 128 lanes against the CUDA-core path."""
    inst = G.make_config(3, 1)
    s1 = _solver(gf, inst, 1)
    s0 = _solver(gf, inst, 0)
    o = O.Oracle(inst)
    p = G.p_vectors(inst["n"], 6)["unif"] * 0.05  # sparse samples: some lanes fit the capacities
    bits = O.sample(p, 3, 1, 0, 2)
    f1, z1 = s1.eval(bits)
    f0, z0 = s0.eval(bits)
    assert np.array_equal(f1, f0) and np.array_equal(z1, z0)
    assert 0 < f1.sum() < 128 or f1.sum() == 128
    for lane in (0, 17, 64, 127):
        x = ((bits[:, lane // 64] >> np.uint64(lane % 64)) & np.uint64(1)).astype(np.uint8)
        f, z = o.eval_point(x)
        assert bool(f1[lane]) == f and z1[lane] == z
