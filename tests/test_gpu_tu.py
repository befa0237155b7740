"""TUReformulate in the library (gfors_tu_reformulate, csrc/tu_impl.inc; next row f2) against the
oracle's plain dense-numpy reformulation (oracle/tu.py): the two reduced problems are evaluated
bit-exactly alike (same samples -> same feasibility and objectives), whole fp64 runs agree (identical
iterations, incumbent and lifted x), lifted incumbents are feasible for the ORIGINAL problem with the
reported objective, and malformed index sets fail loudly."""
import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O
from oracle.tu import tu_reformulate
from tests.test_oracle_tu import _random_tu_instance

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gf():
    import paper_2510_27117_b200 as gf
    return gf


def _pair(gf, inst, J, I, precision=64):
    s = gf.Solver(0)
    s.load(inst)
    s.tu_reformulate(J, I)
    s.preprocess(precision=precision)
    red, lift = tu_reformulate(inst, J, I)
    o = O.Oracle(red)
    o.preprocess()
    return s, o, red, lift


@pytest.mark.parametrize("case", ["facility"] + [f"rand{k}" for k in range(6)])
def test_reduced_problem_evaluates_identically(gf, case):
    if case == "facility":
        inst = G.SMALL["facility"](2)
        J, I = inst["tu_rows"], inst["tu_cols"]
    else:
        inst, J, I = _random_tu_instance(int(case[4:]))
    s, o, red, _ = _pair(gf, inst, J, I)
    assert (s.n, s.m, s.n_orig) == (red["n"], red["m"], inst["n"])
    for pk in ("unif", "mix"):
        p = G.p_vectors(red["n"], 3)[pk]
        bits = O.sample(p, 7, 1, 0, 2)
        fg, zg = s.eval(bits)
        fo, zo = o.eval(bits)
        assert np.array_equal(fg, fo) and np.array_equal(zg, zo)


@pytest.mark.parametrize("seed", [1, 2])
def test_facility_run_parity_and_lift(gf, seed):
    inst = G.SMALL["facility"](seed)
    s, o, red, lift = _pair(gf, inst, inst["tu_rows"], inst["tu_cols"])
    kw = dict(max_iters=3000, k_b=128)
    ig = s.run(**kw)
    io = o.run(**kw)
    assert ig["iters"] == io["iters"] and ig["halt_reason"] == io["halt_reason"]
    zg, xg, _ = s.best_incumbent()
    zo, xo = o.best()
    assert zg == zo
    assert len(xg) == inst["n"] and np.array_equal(xg, lift(xo))
    f, z = O.Oracle(inst).eval_point(xg)  # feasible for the ORIGINAL problem, same objective
    assert f and z == zg


def test_tu_errors(gf):
    inst = G.SMALL["facility"](1)
    s = gf.Solver(0)
    s.load(inst)
    with pytest.raises(gf.GforsError, match="not an equality row"):
        s.tu_reformulate([30], [0])
    with pytest.raises(gf.GforsError, match="signed permutation"):
        # two customer rows, but the column of row 0 is given for row 1 too (it meets I twice)
        s.tu_reformulate([0, 1], [inst["tu_cols"][0], 6])
    s.load(inst)
    with pytest.raises(gf.GforsError, match="does not occur"):
        s.tu_reformulate([0], [inst["tu_cols"][1]])
