"""Dense-Q path (csrc/dense_q.cuh): the int8 dense GEMV in the PDHG step and
the tcgen05 int8 objective kernel, against the CPU oracle (integer objectives bit-exact) and against
the CSR path of the same library (option dense_q = 0).  One-step / 1000-iteration / whole-run parity
of the dense path runs in test_gpu_parity.py (family "maxcut", which loads as dense Q)."""

import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gf():
    import paper_2510_27117_b200 as gf
    return gf


def _solver(gf, inst, precision=64, dense=None, tight=False, options=None):
    opts = dict(options or {})
    if dense is not None:
        opts["dense_q"] = 1 if dense else 0
    s = gf.Solver(0, options=opts)
    s.load(inst)
    tol, it = (1e-14, 100000) if tight else (1e-7, 500)
    sc = s.preprocess(precision=precision, tol=tol, max_iter=it)
    return s, sc


def _lane_bits(bits, lane):
    return ((bits[:, lane // 64] >> np.uint64(lane % 64)) & np.uint64(1)).astype(np.uint8)


@pytest.mark.parametrize("n", [300, 1000, 1500])
@pytest.mark.parametrize("words", [1, 2, 3, 5, 8])
def test_dense_objective_bit_exact(gf, n, words):
    """x_l'Qx_l + c'x_l on 64*words lanes (1-2 tcgen05 passes of N <= 256, ragged N = 64/192/...;
    n not a multiple of 128) equals the oracle's exact integer objective lane by lane."""
    inst = G.max_cut(n, 0.5, n + words)
    s, _ = _solver(gf, inst)
    o = O.Oracle(inst)
    for pk in ("unif", "mix"):
        p = G.p_vectors(n, words)[pk]
        bits = O.sample(p, 3, words, 0, words)
        fg, zg = s.eval(bits)
        fo, zo = o.eval(bits)
        assert fg.all() and fo.all()
        assert np.array_equal(zg, zo), np.flatnonzero(zg != zo)[:10]


def test_dense_objective_equals_cut_definition(gf):
    """Property at any size: z = -(cut weight) computed from the edge weights by definition."""
    n = 700
    inst = G.max_cut(n, 0.5, 11)
    Wd = -G.dense_Q(inst)
    s, _ = _solver(gf, inst)
    bits = O.sample(np.full(n, 0.5), 9, 2, 0, 2)
    _, zg = s.eval(bits)
    for lane in (0, 1, 63, 64, 100, 127):
        x = _lane_bits(bits, lane).astype(bool)
        assert zg[lane] == -Wd[np.ix_(x, ~x)].sum()


def test_dense_and_csr_paths_agree(gf):
    """The dense int8 storage and the CSR storage of the same Q give the same objectives (bit-exact),
    the same Preprocess scale and the same PDHG step (1e-13 relative; the sums run in different
    orders, so equality holds to rounding only)."""
    inst = G.max_cut(400, 0.5, 5)
    sd, scd = _solver(gf, inst, dense=True, tight=True)
    sc_, scc = _solver(gf, inst, dense=False, tight=True)
    assert abs(scd["obj_scale"] - scc["obj_scale"]) <= 1e-12 * scc["obj_scale"]
    bits = O.sample(G.p_vectors(400, 1)["unif"], 1, 1, 0, 4)
    assert np.array_equal(sd.eval(bits)[1], sc_.eval(bits)[1])
    rng = np.random.default_rng(2)
    x = rng.random(400)
    for s_ in (sd, sc_):
        s_.set_state(x, x, np.zeros(0))
        s_.step(1, 0.05, 0.99 ** 0.5, 0.99 ** 0.5)
    xd, xbd, _ = sd.get_state()
    xc, xbc, _ = sc_.get_state()
    assert np.linalg.norm(xd - xc) <= 1e-13 * np.linalg.norm(xc)
    assert np.linalg.norm(xbd - xbc) <= 1e-13 * np.linalg.norm(xbc)


def test_maxcut_short_horizon_parity(gf):
    """Reading R21: for indefinite Q the PDHG map expands free coordinates by at most
    L = 1 + 2 tau (||Q~||_2 + rho) per iteration, so GPU-vs-oracle differences of one step (<= 1e-12,
    test_one_step_parity) can grow at most like L^k.  Pins that bound over the first 25 iterations
    from x0 (fp64, SPEC default sigma)."""
    inst = G.SMALL["maxcut"](4)
    s, sc = _solver(gf, inst, 64, tight=True)
    o = O.Oracle(inst)
    oc = o.preprocess(tol=1e-14, max_iter=100000)
    Qc = -G.dense_Q(inst)  # canonical (minimisation) Q of the maximize instance
    tau, rho = 0.99 ** 0.5, 1e-3
    L = 1.0 + 2.0 * tau * (np.linalg.norm(Qc, 2) / oc["obj_scale"] + rho)
    o.state_init()
    x0, xb0, y0 = o.get_state()
    s.set_state(x0, xb0, y0)
    errs = []
    for k in range(1, 26):
        s.step(1, rho, tau, tau)
        o.step(rho, tau, tau)
        xg = s.get_state()[0]
        xo = o.get_state()[0]
        e = np.linalg.norm(xg - xo) / max(1.0, np.linalg.norm(xo))
        errs.append(e)
        assert e <= 1e-12 * L ** k, (k, e, L)


def test_maxcut_run_incumbent_exact(gf):
    """Whole Alg. 1 on max cut (graph, fp64 and fp32): the incumbent's objective equals the oracle's
    exact evaluation of the returned x, z_best never worsens, and the cut is at least the cut of
    the best of the first round's samples (monotone incumbent)."""
    inst = G.max_cut(256, 0.5, 8)
    o = O.Oracle(inst)
    Wd = -G.dense_Q(inst)
    for prec in (64, 32):
        s, _ = _solver(gf, inst, prec)
        info = s.run(max_iters=1500, k_b=128)
        z, x, meta = s.best_incumbent()
        f, zz = o.eval_point(x)
        xb = x.astype(bool)
        assert f and z == -zz == Wd[np.ix_(xb, ~xb)].sum()  # user sense: the cut weight
        tr = s.trace()
        zt = tr[:, 6][np.isfinite(tr[:, 6])]
        assert (np.diff(zt) <= 0).all()
        assert info["iters"] <= 1500


def test_config6_fullsize_sampled(gf):
    """BASELINE-scale max cut (n = 20480, density 0.5), bench launch configuration
    (fp32, k_int = 10, k_b = 128, graph): invariants, and sampled candidates checked one by one
    against the cut definition and the oracle's point evaluation."""
    inst = G.make_config(6, 1)
    s, sc = _solver(gf, inst, 32)
    info = s.run(max_iters=100, k_int=10, k_b=128, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)
    assert info["iters"] == 100 and info["rounds"] == 10
    x, _, _ = s.get_state()
    assert np.all(np.isfinite(x)) and (x >= 0).all() and (x <= 1).all()
    bits = s.sample(x, 20251030, 9, 0, 2)
    _, zg = s.eval(bits)
    n = inst["n"]
    Wd = np.zeros((n, n), dtype=np.int16)
    rows = np.repeat(np.arange(n), np.diff(inst["q_rowptr"]))
    Wd[rows, inst["q_col"]] = -inst["q_val"].astype(np.int16)
    o = O.Oracle(inst)
    for lane in (0, 77, 100, 127):
        xl = _lane_bits(bits, lane)
        xb = xl.astype(bool)
        assert zg[lane] == -Wd[np.ix_(xb, ~xb)].sum(dtype=np.int64)
        f, zz = o.eval_point(xl)
        assert f and zg[lane] == zz
    z, _, _ = s.best_incumbent(want_x=False)
    assert np.isfinite(z)


@pytest.mark.parametrize("kint", [10, 3, 1])
def test_gemv_reuse_across_blocks(gf, kint):
    """fp32 loop: the trigger's product of x_k serving the next block's first primal (option qx_reuse)
    gives the same trajectory as recomputing it (the first primal's product is bit-identical; the
    s^x term of the indicators differs only in how the fixed-point difference is formed), and the
    same incumbent."""
    inst = G.max_cut(400, 0.5, 21)
    res = []
    for reuse in (1, 0):
        s, _ = _solver(gf, inst, 32, options={"qx_reuse": reuse})
        kw = dict(k_int=kint, k_b=128, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)
        s.run(max_iters=30 * kint, **kw)
        x = s.get_state()[0]
        z, xb, _ = s.best_incumbent()
        tr = s.trace()
        res.append((x, z, xb, tr))
    assert np.array_equal(res[0][0], res[1][0])
    assert res[0][1] == res[1][1] and np.array_equal(res[0][2], res[1][2])
    t0, t1 = res[0][3], res[1][3]
    assert np.array_equal(t0[:, [0, 1, 2, 4, 5, 6, 7]], t1[:, [0, 1, 2, 4, 5, 6, 7]])
    assert np.allclose(t0[:, 3], t1[:, 3], rtol=1e-6, atol=1e-9)  # ||s^x||


def test_dense_objective_max_batch(gf):
    """k_b = 4096 per rank (the dense objective's limit): 16 tcgen05 passes of N = 256, a 4-stage ring
    next to the 32 KB of lane sums; bit-exact against the oracle."""
    inst = G.max_cut(300, 0.5, 99)
    s, _ = _solver(gf, inst)
    o = O.Oracle(inst)
    bits = O.sample(G.p_vectors(300, 7)["unif"], 2, 5, 0, 64)
    fg, zg = s.eval(bits)
    fo, zo = o.eval(bits)
    assert np.array_equal(zg, zo)
    with pytest.raises(gf.GforsError, match="4096"):
        s.eval(np.zeros((300, 65), dtype=np.uint64))
