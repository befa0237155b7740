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


def _canonical_pair(seed):
    """The same canonical problem given two ways: A with its rows already canonical (GE rows first,
    then EQ; no LE row), so the load keeps no host copy of K and TUReformulate downloads it from the
    device (ensure_host_k); B with every GE row negated into an LE row, so the load copies and negates
    on the host.  Integer values beyond +-1 (the int8 value class) and, for seed 1, a non-integer
    coefficient (the fp64 class)."""
    rng = np.random.default_rng(seed)
    n = 12
    K, r, sense, J, I = [], [], [], [], []
    for k in range(3):
        row = np.zeros(n)
        row[k * 4:(k + 1) * 4] = 1.0
        K.append(row); r.append(1.0); sense.append(0)
        J.append(k); I.append(k * 4 + int(rng.integers(0, 4)))
    ge = []
    for _ in range(4):
        row = np.zeros(n)
        idx = rng.choice(n, size=5, replace=False)
        row[idx] = rng.integers(1, 4, size=5) * rng.choice([-1, 1], size=5)
        if seed == 1:
            row[idx[0]] = 1.5
        ge.append((row, float(rng.integers(-2, 3))))
    c = rng.integers(-9, 10, size=n).astype(float)
    # A: GE rows first, then the EQ rows
    KA = [g[0] for g in ge] + K
    rA = [g[1] for g in ge] + r
    sA = [1] * len(ge) + sense
    JA = [len(ge) + j for j in J]
    # B: the GE rows as negated LE rows
    KB = [-g[0] for g in ge] + K
    rB = [-g[1] for g in ge] + r
    sB = [-1] * len(ge) + sense
    from tests.util import inst_from_dense
    return inst_from_dense(KA, rA, sA, c), inst_from_dense(KB, rB, sB, c), JA, I


@pytest.mark.parametrize("seed", [0, 1])
def test_host_k_download_matches_host_copy(gf, seed):
    """Host-side consumers see the same canonical K whether the load copied it (non-canonical input)
    or downloads it on demand (canonical input): the TU-reduced problems evaluate bit-identically."""
    A, B, J, I = _canonical_pair(seed)
    res = []
    for inst in (A, B):
        s = gf.Solver(0)
        s.load(inst)
        s.tu_reformulate(J, I)
        s.preprocess(precision=64)
        p = G.p_vectors(s.n, 3)["unif"]
        bits = O.sample(p, 5, 1, 0, 2)
        res.append((s.n, s.m) + s.eval(bits))
        s.close()
    assert res[0][:2] == res[1][:2]
    assert np.array_equal(res[0][2], res[1][2]) and np.array_equal(res[0][3], res[1][3])
