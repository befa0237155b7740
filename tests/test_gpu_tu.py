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
from tests.test_oracle_tu import _interval_tu_instance, _random_tu_instance

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


@pytest.mark.parametrize("case", ["facility", "facility_slack"] + [f"rand{k}" for k in range(6)]
                         + [f"interval{k}" for k in range(6)])
def test_reduced_problem_evaluates_identically(gf, case):
    """Signed-permutation B_JI (facility, rand*) and general B_JI eliminated with fill (facility_slack:
    unit triangular; interval*: overlapping consecutive-ones rows)."""
    if case == "facility":
        inst = G.SMALL["facility"](2)
        J, I = inst["tu_rows"], inst["tu_cols"]
    elif case == "facility_slack":
        inst = G.facility_location_slack(6, 24, 2)
        J, I = inst["tu_rows"], inst["tu_cols"]
    elif case.startswith("interval"):
        inst, J, I = _interval_tu_instance(int(case[8:]))
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


@pytest.mark.parametrize("seed", [1, 2])
def test_facility_slack_run_parity_and_lift(gf, seed):
    """The all-equality facility location (reading R24 rev.): the library's elimination (B_JI unit
    triangular, with fill) gives the oracle's reduced problem — identical fp64 runs — and the lifted
    incumbent is feasible for the ORIGINAL (inequality) facility-location problem."""
    inst = G.facility_location_slack(6, 24, seed)
    s, o, red, lift = _pair(gf, inst, inst["tu_rows"], inst["tu_cols"])
    assert s.m == red["m"] and np.all(red["sense"] == 1)
    kw = dict(max_iters=3000, k_b=128)
    ig = s.run(**kw)
    io = o.run(**kw)
    assert ig["iters"] == io["iters"] and ig["halt_reason"] == io["halt_reason"]
    zg, xg, _ = s.best_incumbent()
    zo, xo = o.best()
    assert zg == zo
    if np.isfinite(zg):
        assert np.array_equal(xg, lift(xo))
        fl = G.facility_location(6, 24, seed)
        f, z = O.Oracle(fl).eval_point(xg[: fl["n"]])
        assert f and z == zg


def test_tu_errors(gf):
    inst = G.SMALL["facility"](1)
    s = gf.Solver(0)
    s.load(inst)
    with pytest.raises(gf.GforsError, match="not an equality row"):
        s.tu_reformulate([30], [0])
    with pytest.raises(gf.GforsError, match="no \\+-1 pivot"):
        # customer row 0 does not contain the cheapest column of customer 1: B_JI = 0 is singular
        s.tu_reformulate([0], [inst["tu_cols"][1]])
    s.load(inst)
    with pytest.raises(gf.GforsError, match="repeated"):
        s.tu_reformulate([0, 0], [inst["tu_cols"][0], inst["tu_cols"][1]])
    # a non-TU B_J: rows x0 + x1 + x2 = 1, x0 - x1 + x2 = 1 with I = {0, 1}: eliminating leaves a 2
    from tests.util import inst_from_dense
    bad = inst_from_dense([[1, 1, 1, 0], [1, -1, 1, 1]], [1, 1], [0, 0], [1.0, 2.0, 3.0, 4.0])
    s.load(bad)
    with pytest.raises(gf.GforsError, match="not TU"):
        s.tu_reformulate([0, 1], [0, 1])
