"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Bars (BASELINE.json north_star): sampling, feasibility and integer objectives bit-exact; PDHG
iterates / indicators within 1e-5 (fp64) or 1e-3 (fp32) relative after 1000 iterations.
"""
import math

import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O
from tests.util import brute_force, exhaustive_bits, inst_from_dense

pytestmark = pytest.mark.gpu

FAMILIES = ["setcover", "mis", "mkp", "bqp", "general", "real", "maxcut", "dense_psd"]
# families whose PDHG map is (up to the small -2 rho x term) non-expansive, where the 1000-iteration bar
# applies.  maxcut's Q is indefinite: the map expands free coordinates by up to 1 + 2 tau (||Q~|| + rho),
# so rounding-order differences grow geometrically (reading R21; test_gpu_dense_q.py pins that bound).
CONTRACTIVE = [f for f in FAMILIES if f != "maxcut"]


@pytest.fixture(scope="module")
def gf():
    import paper_2510_27117_b200 as gf
    return gf


def _pair(gf, inst, precision=64, tight=False, options=None):
    """tight: run both power iterations to 1e-14 so the scalings agree far below the PDHG tolerance
    (at the default 1e-7 stop they agree to ~1e-8 only).  options: gfors_set_option before
    the load (forced PDHG variants)."""
    tol, it = (1e-14, 100000) if tight else (1e-7, 500)
    s = gf.Solver(0, options=options)
    s.load(inst)
    sc = s.preprocess(precision=precision, tol=tol, max_iter=it)
    o = O.Oracle(inst)
    oc = o.preprocess(tol=tol, max_iter=it)
    return s, sc, o, oc


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# ------------------------------------------------------------------------------------ Preprocess
@pytest.mark.parametrize("fam", FAMILIES)
def test_preprocess_parity(gf, fam):
    inst = G.SMALL[fam](1)
    s, sc, o, oc = _pair(gf, inst)
    srow, r_sc, c_sc = s.scaled()
    assert np.allclose(srow, o.row_scales(), rtol=1e-14, atol=0)
    assert sc["zero_rows"] == oc["zero_rows"]
    # power iterations stop at relative change 1e-7 on both sides: agree to 1e-6
    assert abs(sc["obj_scale"] - oc["obj_scale"]) <= 1e-6 * oc["obj_scale"]
    assert abs(sc["k_scale"] - oc["k_scale"]) <= 1e-6 * oc["k_scale"]


# ------------------------------------------------------------------------------------ sampler
@pytest.mark.parametrize("fam", FAMILIES)
@pytest.mark.parametrize("pkind", ["unif", "mix", "traj"])
def test_sampler_bit_exact(gf, fam, pkind):
    inst = G.SMALL[fam](2)
    s, _, o, _ = _pair(gf, inst)
    if pkind == "traj":
        o.state_init()
        for _ in range(37):
            o.step(0.01, 0.99 ** 0.5, 0.99 ** 0.5)
        p = o.get_state()[0]
    else:
        p = G.p_vectors(inst["n"], 9)[pkind]
    for (seed, rnd, wb, nw) in [(1, 0, 0, 1), (20251030, 7, 3, 2), (2**63 + 5, 2**32 - 1, 1000, 5)]:
        a = s.sample(p, seed, rnd, wb, nw)
        b = O.sample(p, seed, rnd, wb, nw)
        assert np.array_equal(a, b), (seed, rnd, wb, nw)


def test_sampler_edge_probabilities(gf):
    n = 300
    inst = G.set_cover(10, n, 2, 5, 3)
    s, _, o, _ = _pair(gf, inst)
    p = np.zeros(n)
    p[0::5] = 1.0
    p[1::5] = 2.0 ** -32          # T = 1: only u == 0 samples 1
    p[2::5] = 1.0 - 2.0 ** -33    # T = 2^32 after ceil -> always 1
    p[3::5] = 0.5
    p[4::5] = np.nextafter(0.5, 0)
    a = s.sample(p, 77, 3, 0, 4)
    assert np.array_equal(a, O.sample(p, 77, 3, 0, 4))
    assert (a[0::5] == np.uint64(0xFFFFFFFFFFFFFFFF)).all()


# ------------------------------------------------------------------------------------ evaluator
@pytest.mark.parametrize("fam", FAMILIES)
def test_eval_bit_exact(gf, fam):
    inst = G.SMALL[fam](3)
    s, _, o, _ = _pair(gf, inst)
    for pk in ["unif", "mix"]:
        p = G.p_vectors(inst["n"], 4)[pk]
        bits = O.sample(p, 5, 1, 0, 3)
        fg, zg = s.eval(bits)
        fo, zo = o.eval(bits)
        assert np.array_equal(fg, fo)
        if o.integral:
            assert np.array_equal(zg, zo)
        else:
            assert np.allclose(zg, zo, rtol=1e-12, atol=1e-9)


def test_eval_exhaustive_vs_brute_force(gf):
    """All 2^20 points of config 1 through the GPU evaluator = enumeration."""
    inst = G.make_config(1, 1)
    s = gf.Solver(0)
    s.load(inst)
    s.preprocess()
    feas, z = s.eval(exhaustive_bits(20))
    zb, xb, ok, zu = brute_force(inst)
    assert np.array_equal(feas.astype(bool), ok)
    assert np.array_equal(z, zu)
    assert z[feas.astype(bool)].min() == zb


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_eval_exhaustive_mixed_rows(gf, seed):
    """GE/EQ/LE rows with +-1 patterns, general integers, Q and c0 (canonicalisation + all row classes)."""
    rng = np.random.default_rng(seed)
    n = 12
    K = np.zeros((9, n))
    K[0, :5] = 1                          # cover  >= 1
    K[1, 3:9] = -1                        # -sum >= -2  (<= 2)
    K[2, [0, 2, 4, 6]] = 1                # == 2
    K[3, 5:] = rng.integers(-5, 6, n - 5) # general int
    K[3, 5] = 3
    K[4, :] = 1                           # sum <= 7 (LE)
    K[5, [1, 7]] = [2, -3]                # general
    K[6, [8, 9, 10]] = 1                  # >= 2 (count, B=2)
    K[7, [2, 3, 11]] = -1                 # == -1 (count EQ with negative sign)
    K[8, :] = 0                           # empty row, 0 >= -1
    K[8, 0] = 1
    r = [1, -2, 2, 1, 7, -1, 2, -1, 0]
    sense = [1, 1, 0, 1, -1, 1, 1, 0, 1]
    Q = rng.integers(-3, 4, (n, n)).astype(float)
    Q = Q + Q.T
    inst = inst_from_dense(K, r, sense, rng.integers(-9, 10, n).astype(float), Q=Q, c0=3.0, maximize=seed == 2)
    s = gf.Solver(0)
    s.load(inst)
    s.preprocess()
    o = O.Oracle(inst)
    bits = exhaustive_bits(n)
    fg, zg = s.eval(bits)
    fo, zo = o.eval(bits)
    assert np.array_equal(fg, fo) and np.array_equal(zg, zo)
    _, _, ok, zu = brute_force(inst)
    assert np.array_equal(fg.astype(bool), ok)


# ------------------------------------------------------------------------------------ PDHG
@pytest.mark.parametrize("fam", FAMILIES)
@pytest.mark.parametrize("prec,tol", [(64, 1e-12), (32, 1e-6)])
def test_one_step_parity(gf, fam, prec, tol):
    inst = G.SMALL[fam](4)
    s, _, o, _ = _pair(gf, inst, prec, tight=True)
    rng = np.random.default_rng(0)
    n, m = inst["n"], inst["m"]
    x = rng.random(n); xb = rng.random(n); y = rng.random(m) * 0.1 - 0.02
    y[: o.m1] = np.abs(y[: o.m1])
    if prec == 32:  # start both from the fp32-representable state
        x, xb, y = (v.astype(np.float32).astype(np.float64) for v in (x, xb, y))
    s.set_state(x, xb, y)
    o.set_state(x, xb, y)
    s.step(1, 0.3, 0.9, 0.8)
    o.step(0.3, 0.9, 0.8)
    xg, xbg, yg = s.get_state()
    xo, xbo, yo = o.get_state()
    assert _rel(xg, xo) <= tol and _rel(xbg, xbo) <= tol and _rel(yg, yo) <= tol


@pytest.mark.parametrize("fam", CONTRACTIVE)
@pytest.mark.parametrize("prec,tol", [(64, 1e-5), (32, 1e-3)])
def test_1000_iteration_parity(gf, fam, prec, tol):
    """1000 iterations under the default rho schedule, sampling off."""
    inst = G.SMALL[fam](5)
    s, _, o, _ = _pair(gf, inst, prec)
    tau = math.sqrt(0.99)
    rho = O.rho_schedule(1e-3, 10.0, 100.0, 2.0, 1e-6, 100)
    o.state_init()
    x0, xb0, y0 = o.get_state()
    s.set_state(x0, xb0, y0)
    for b in range(100):
        s.step(10, rho[b], tau, tau)
        for _ in range(10):
            o.step(rho[b], tau, tau)
    xg, xbg, yg = s.get_state()
    xo, xbo, yo = o.get_state()
    assert _rel(xg, xo) <= tol, _rel(xg, xo)
    assert _rel(yg, yo) <= tol, _rel(yg, yo)
    ig = s.indicators(rho[99], tau, tau)
    io = o.indicators(rho[99], tau, tau)
    for k in ("primal_gap", "dual_gap", "binary_gap"):
        assert abs(ig[k] - io[k]) <= tol * max(abs(io[k]), 1e-3), (k, ig[k], io[k])


@pytest.mark.parametrize("fam", FAMILIES)
def test_indicators_parity(gf, fam):
    inst = G.SMALL[fam](6)
    s, _, o, _ = _pair(gf, inst, tight=True)
    rng = np.random.default_rng(1)
    n, m = inst["n"], inst["m"]
    x = rng.random(n); xb = rng.random(n); y = np.abs(rng.random(m))
    s.set_state(x, xb, y); o.set_state(x, xb, y)
    s.step(1, 0.7, 0.5, 0.6); o.step(0.7, 0.5, 0.6)
    ig = s.indicators(0.7, 0.5, 0.6)
    io = o.indicators(0.7, 0.5, 0.6)
    for k in ("primal_gap", "sx", "sy", "binary_gap"):
        assert abs(ig[k] - io[k]) <= 1e-11 * max(1.0, abs(io[k])), (k, ig[k], io[k])


# ------------------------------------------------------------------------------------ Alg. 1
def _compare_runs(gf, inst, prec=64, graph=1, **kw):
    s, _, o, _ = _pair(gf, inst, prec)
    ig = s.run(use_graph=graph, **kw)
    io = o.run(trace_max=100000, **kw)
    zg, xg, mg = s.best_incumbent()
    zo, xo = o.best()
    return s, o, ig, io, (zg, xg, mg), (zo, xo)


@pytest.mark.parametrize("fam", ["setcover", "bqp", "mkp", "general", "dense_psd"])
@pytest.mark.parametrize("graph", [1, 0])
def test_run_parity_fp64(gf, fam, graph):
    """fp64 trajectories agree, so the incumbent sequence is identical."""
    inst = G.SMALL[fam](7)
    s, o, ig, io, (zg, xg, mg), (zo, xo) = _compare_runs(gf, inst, graph=graph, max_iters=600, k_b=128)
    assert ig["iters"] == io["iters"] and ig["halt_reason"] == io["halt_reason"]
    assert ig["rounds"] == io["rounds"]
    assert zg == zo or (math.isinf(zg) and math.isinf(zo))
    if not math.isinf(zo):
        assert np.array_equal(xg, xo)
        assert (mg["found_iter"], mg["found_round"], mg["found_index"]) == (
            io["found_iter"], io["found_round"], io["found_index"])
    tg = s.trace()
    to = io["trace"]
    assert tg.shape == to.shape
    assert np.array_equal(tg[:, [0, 1, 6, 7]], to[:, [0, 1, 6, 7]])
    assert np.allclose(tg[:, 2:6], to[:, 2:6], rtol=1e-6, atol=1e-9)


def test_run_parity_config1_and_quality(gf):
    inst = G.make_config(1, 4)
    s, o, ig, io, (zg, xg, mg), (zo, xo) = _compare_runs(gf, inst, max_iters=5000)
    assert zg == zo and np.array_equal(xg, xo) and ig["iters"] == io["iters"]
    zb, _, _, _ = brute_force(inst)
    assert zg >= zb
    f, zz = o.eval_point(xg)
    assert f and zz == zg


def test_run_fp32_incumbent_feasible(gf):
    """fp32 iterates: the trajectory differs from the fp64 oracle at the 1e-3 level, so the incumbent
    is checked for feasibility and objective by oracle recomputation, and for quality."""
    for seed in (5, 6):
        inst = G.make_config(1, seed)
        s, o, ig, io, (zg, xg, mg), (zo, xo) = _compare_runs(gf, inst, prec=32, max_iters=3000)
        assert not math.isinf(zg) and not math.isinf(zo)
        f, zz = o.eval_point(xg)
        assert f and zz == zg
        zb, _, _, _ = brute_force(inst)
        assert zg <= 1.25 * zb


@pytest.mark.parametrize("case", ["tail", "short", "kr3", "kb1024", "kb512", "maximize_mis", "mis_kb1024", "no_constraints",
                                  "infeasible"])
def test_run_edge_cases(gf, case):
    kw = dict(max_iters=203)
    inst = G.SMALL["setcover"](9)
    if case == "short":
        kw = dict(max_iters=7)
    elif case == "kr3":
        kw = dict(max_iters=100, k_r=3, k_int=7)
    elif case == "kb1024":
        kw = dict(max_iters=60, k_b=1024)
    elif case == "kb512":  # 8-word feasibility units (one-plane rows, one thread per row and word)
        kw = dict(max_iters=60, k_b=512)
    elif case == "maximize_mis":
        inst = G.max_independent_set(300, 0.02, 3, weighted=True)
        kw = dict(max_iters=500, sigma=0.5)
    elif case == "mis_kb1024":  # 8-word units of two-plane packing rows (per-row lane groups)
        inst = G.max_independent_set(300, 0.02, 3, weighted=True)
        kw = dict(max_iters=300, sigma=0.5, k_b=1024)
    elif case == "no_constraints":
        inst = inst_from_dense([], [], [], np.random.default_rng(0).integers(-5, 6, 50).astype(float))
        kw = dict(max_iters=100)
    elif case == "infeasible":
        inst = inst_from_dense([[1, 1], [-1, -1]], [2, -1], [1, 1], [1.0, 1.0])
        kw = dict(max_iters=50)
    s, o, ig, io, (zg, xg, mg), (zo, xo) = _compare_runs(gf, inst, **kw)
    assert ig["iters"] == io["iters"] and ig["rounds"] == io["rounds"] and ig["halt_reason"] == io["halt_reason"]
    assert zg == zo or (math.isinf(zg) and math.isinf(zo))
    if not math.isinf(zo):
        assert np.array_equal(xg, xo)
        assert mg["found_index"] == io["found_index"] and mg["found_round"] == io["found_round"]


def test_run_deterministic(gf):
    inst = G.SMALL["bqp"](2)
    s = gf.Solver(0)
    s.load(inst)
    s.preprocess()
    a = s.run(max_iters=300); ta = s.trace(); za = s.best_incumbent()
    b = s.run(max_iters=300); tb = s.trace(); zb = s.best_incumbent()
    assert np.array_equal(ta, tb) and za[0] == zb[0] and np.array_equal(za[1], zb[1])


def test_errors_fail_loudly(gf):
    s = gf.Solver(0)
    with pytest.raises(gf.GforsError):
        s.preprocess()  # before load
    inst = G.SMALL["setcover"](1)
    bad = dict(inst, k_val=inst["k_val"].copy())
    bad["k_val"][3] = 0.0
    with pytest.raises(gf.GforsError, match="explicit zero"):
        s.load(bad)
    s.load(inst)
    s.preprocess()
    with pytest.raises(gf.GforsError, match="k_b"):
        s.run(k_b=100)
    with pytest.raises(gf.GforsError, match="sigma"):
        s.run(sigma=1.5)


@pytest.mark.parametrize("fam", ["setcover", "general", "bqp"])
def test_sparse_primal_variant_parity(gf, fam):
    """The zero-dual-skipping primal (forced on small instances) against the oracle: 1000 fp64
    iterations within 1e-5, and a full run with identical incumbent sequence."""
    inst = G.SMALL[fam](11)
    s, _, o, _ = _pair(gf, inst, 64, options={"sparse_primal": 1})
    tau = math.sqrt(0.99)
    rho = O.rho_schedule(1e-3, 10.0, 100.0, 2.0, 1e-6, 100)
    o.state_init()
    x0, xb0, y0 = o.get_state()
    s.set_state(x0, xb0, y0)
    for b in range(100):
        s.step(10, rho[b], tau, tau)
        for _ in range(10):
            o.step(rho[b], tau, tau)
    xg, _, yg = s.get_state()
    xo, _, yo = o.get_state()
    assert _rel(xg, xo) <= 1e-5 and _rel(yg, yo) <= 1e-5
    ig = s.run(max_iters=400)
    io = o.run(max_iters=400)
    assert ig["iters"] == io["iters"] and ig["rounds"] == io["rounds"]
    zg, xbest, mg = s.best_incumbent()
    zo, xo2 = o.best()
    assert zg == zo or (math.isinf(zg) and math.isinf(zo))


@pytest.mark.parametrize("fam", ["setcover", "mis", "bqp"])
def test_push_dual_variant_parity(gf, fam):
    """Sparse-xbar dual (fixed-point scatter, forced on) against the oracle: 1000 fp64 iterations
    within 1e-5; a run keeps the same incumbent and iteration accounting."""
    inst = G.SMALL[fam](12)
    s, _, o, _ = _pair(gf, inst, 64, options={"push_dual": 1})
    tau = math.sqrt(0.99)
    rho = O.rho_schedule(1e-3, 10.0, 100.0, 2.0, 1e-6, 100)
    o.state_init()
    x0, xb0, y0 = o.get_state()
    s.set_state(x0, xb0, y0)
    for b in range(100):
        s.step(10, rho[b], tau, tau)
        for _ in range(10):
            o.step(rho[b], tau, tau)
    xg, _, yg = s.get_state()
    xo, _, yo = o.get_state()
    assert _rel(xg, xo) <= 1e-5 and _rel(yg, yo) <= 1e-5
    ig = s.run(max_iters=400)
    io = o.run(max_iters=400)
    assert ig["iters"] == io["iters"] and ig["rounds"] == io["rounds"]
    zg, _, _ = s.best_incumbent()
    zo, _ = o.best()
    assert zg == zo or (math.isinf(zg) and math.isinf(zo))


@pytest.mark.parametrize("fam", ["setcover", "mis", "bqp"])
@pytest.mark.parametrize("prec,tol", [(64, 1e-5), (32, 1e-3)])
def test_push_primal_variant_parity(gf, fam, prec, tol):
    """Sparse-dual primal (fixed-point column scatter, forced on together with the push dual) against
    the oracle: 1000 iterations within the north_star tolerance, same run accounting."""
    inst = G.SMALL[fam](13)
    s, _, o, _ = _pair(gf, inst, prec, options={"push_dual": 1, "push_primal": 1})
    tau = math.sqrt(0.99)
    rho = O.rho_schedule(1e-3, 10.0, 100.0, 2.0, 1e-6, 100)
    o.state_init()
    x0, xb0, y0 = o.get_state()
    s.set_state(x0, xb0, y0)
    for b in range(100):
        s.step(10, rho[b], tau, tau)
        for _ in range(10):
            o.step(rho[b], tau, tau)
    xg, _, yg = s.get_state()
    xo, _, yo = o.get_state()
    assert _rel(xg, xo) <= tol and _rel(yg, yo) <= tol
    ig = s.run(max_iters=400)
    io = o.run(max_iters=400)
    assert ig["iters"] == io["iters"] and ig["rounds"] == io["rounds"]
    if prec == 64:
        zg, _, _ = s.best_incumbent()
        zo, _ = o.best()
        assert zg == zo or (math.isinf(zg) and math.isinf(zo))


@pytest.mark.parametrize("switch", ["delta_dual", "xskip", "cond_branch"])
@pytest.mark.parametrize("fam", ["setcover", "mis"])
@pytest.mark.parametrize("prec", [64, 32])
def test_exact_shortcuts_bit_identical(gf, switch, fam, prec):
    """Shortcuts that must reproduce the plain computation BIT FOR BIT (push modes forced on):
    delta_dual — the delta push of the dual adds exact integer differences instead of a fresh
    fixed-point sum; xskip — the push primal skips columns whose update provably returns the value
    already stored; cond_branch — graph conditional nodes run only the chosen mode's kernels
    instead of launching both with early exits.  Same iterates after hook steps, same run trace and
    incumbent."""
    inst = G.SMALL[fam](14)
    tau = math.sqrt(0.99)
    rho = O.rho_schedule(1e-3, 10.0, 100.0, 2.0, 1e-6, 60)
    out = []
    for on in (0, 1):
        s = gf.Solver(0, options={"push_dual": 1, "push_primal": 1, switch: on})
        s.load(inst)
        s.preprocess(precision=prec, tol=1e-10, max_iter=5000)
        s.set_state(np.zeros(inst["n"]), np.zeros(inst["n"]), np.zeros(inst["m"]))
        for b in range(60):
            s.step(10, rho[b], tau, tau)
        st = s.get_state()
        info = s.run(max_iters=2000, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)
        out.append((st, s.trace(), s.best_incumbent(), info["iters"]))
        assert info["launches"] > 0
    (sa, ta, za, ia), (sb, tb, zb, ib) = out
    for u, v in zip(sa, sb):
        assert np.array_equal(u, v)
    assert ia == ib and np.array_equal(ta, tb)
    assert za[0] == zb[0] or (math.isinf(za[0]) and math.isinf(zb[0]))
