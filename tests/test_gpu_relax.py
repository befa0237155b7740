"""Monotone relaxation + repair (csrc/repair.cuh; next row f4) against the oracle:
the repair of a batch is bit-exact, a relaxed PDHG step agrees to 1e-12 (fp64), and whole fp64 runs
with relax = repair = 1 are identical (iterations, incumbent, x); incumbents satisfy the ORIGINAL
equalities."""
import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gf():
    import paper_2510_27117_b200 as gf
    return gf


def _solver(gf, inst, precision=64, tight=False):
    s = gf.Solver(0)
    s.load(inst)
    tol, it = (1e-14, 100000) if tight else (1e-7, 500)
    s.preprocess(precision=precision, tol=tol, max_iter=it)
    o = O.Oracle(inst)
    o.preprocess(tol=tol, max_iter=it)
    return s, o


@pytest.mark.parametrize("n,dens,nw", [(3, 0.2, 1), (5, 0.05, 2), (6, 0.03, 3), (8, 0.01, 2)])
def test_repair_bit_exact(gf, n, dens, nw):
    inst = G.assignment3d(n, n)
    s, o = _solver(gf, inst)
    o.set_relax(1)
    rng = np.random.default_rng(n)
    bits = O.sample(np.where(rng.random(n ** 3) < 0.5, dens, 4 * dens).clip(0, 1), 3, 1, 0, nw)
    a = s.repair(bits)
    b = o.repair(bits)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, bits)  # something was dropped


def test_relaxed_step_parity(gf):
    inst = G.assignment3d(4, 2)
    s, o = _solver(gf, inst, tight=True)
    s.set_relax(1)
    o.set_relax(1)
    rng = np.random.default_rng(0)
    x = rng.random(64)
    y = rng.standard_normal(12) * 0.2
    s.set_state(x, x, y)
    o.set_state(x, x, y)
    s.step(1, 0.05, 0.9, 0.8)
    o.step(0.05, 0.9, 0.8)
    for a, b in zip(s.get_state(), o.get_state()):
        assert np.linalg.norm(a - b) <= 1e-12 * max(1.0, np.linalg.norm(b))
    ig, io = s.indicators(0.05, 0.9, 0.8), o.indicators(0.05, 0.9, 0.8)
    for k in ("primal_gap", "sx", "sy", "binary_gap"):
        assert abs(ig[k] - io[k]) <= 1e-11 * max(1.0, abs(io[k]))


@pytest.mark.parametrize("graph", [1, 0])
def test_relax_repair_run_parity_fp64(gf, graph):
    n = 5
    inst = G.assignment3d(n, 9)
    s, o = _solver(gf, inst)
    kw = dict(max_iters=1500, k_b=128, relax=1, repair=1)
    ig = s.run(use_graph=graph, **kw)
    io = o.run(**kw)
    assert ig["iters"] == io["iters"] and ig["halt_reason"] == io["halt_reason"]
    zg, xg, _ = s.best_incumbent()
    zo, xo = o.best()
    assert zg == zo and np.array_equal(xg, xo)
    if np.isfinite(zg):
        f, z = o.eval_point(xg)  # the ORIGINAL equalities hold
        assert f and z == zg


def test_relax_errors(gf):
    s, _ = _solver(gf, G.random_general(20, 4, 3, 4, 2))
    with pytest.raises(gf.GforsError, match="relax"):
        s.run(max_iters=20, relax=1)
    s2, _ = _solver(gf, G.assignment3d(3, 1))
    with pytest.raises(gf.GforsError, match="repair"):
        s2.run(max_iters=20, repair=1)


@pytest.mark.parametrize("n", [21, 26])
def test_repair_large_lanes_bit_exact(gf, n):
    """SPEC L354 repairs every lane: a lane holding all n^3 entries (n = 26: 17576 > the 16384 the
    kernel sorts in shared memory, so the ordered-scan path runs), a lane with ~half of them and
    sparse lanes are repaired bit-identically to the oracle."""
    inst = G.assignment3d(n, 4)
    s, o = _solver(gf, inst)
    o.set_relax(1)
    bits = O.sample(np.full(n ** 3, 0.02), 9, 1, 0, 2)
    bits[:, 0] |= np.uint64(1)  # lane 0: every entry
    half = np.random.default_rng(n).random(n ** 3) < 0.5
    bits[half, 1] |= np.uint64(1) << np.uint64(5)  # lane 69: ~n^3/2 entries
    a = s.repair(bits)
    b = o.repair(bits)
    assert np.array_equal(a, b)
    assert int(np.count_nonzero(a[:, 0] & np.uint64(1))) < n ** 3  # lane 0 was repaired


def test_repair_many_rows_bit_exact(gf):
    """m > 12288 rows: the per-lane row sums live in global scratch instead of shared memory."""
    inst = G.set_cover(13000, 600, 2, 6, 3)
    s, o = _solver(gf, inst)
    o.set_relax(1)
    rng = np.random.default_rng(2)
    bits = O.sample(rng.random(600) * 0.9 + 0.1, 4, 1, 0, 2)
    a = s.repair(bits)
    b = o.repair(bits)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, bits)
