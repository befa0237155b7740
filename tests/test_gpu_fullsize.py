"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (fp32 iterates,
k_int = 10, k_b = 128, CUDA graph), on sampled outputs the oracle can compute one by one and on
properties that hold at any size."""
import math

import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu

BENCH = dict(k_int=10, k_b=128, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)


@pytest.fixture(scope="module")
def gf():
    import paper_2510_27117_b200 as gf
    return gf


@pytest.fixture(scope="module")
def cfg5(gf):
    inst = G.make_config(5, 1)
    s = gf.Solver(0)
    s.load(inst)
    sc = s.preprocess(precision=32)
    o = O.Oracle(inst)
    return inst, s, sc, o


def test_config5_run_invariants_and_sampled_parity(gf, cfg5):
    inst, s, sc, o = cfg5
    info = s.run(max_iters=300, **BENCH)
    assert info["iters"] == 300 and info["rounds"] == 30 and info["halt_reason"] == 2
    x, xb, y = s.get_state()
    m1 = int(np.sum(inst["sense"] != 0))
    assert (x >= 0).all() and (x <= 1).all() and (y[:m1] >= 0).all()
    assert np.all(np.isfinite(xb))
    tr = s.trace()
    assert (np.diff(tr[:, 6][np.isfinite(tr[:, 6])]) <= 0).all()  # z_best never increases
    # sampler on x_k: GPU batch vs oracle draws for 3000 random variables (bit-exact)
    bits = s.sample(x, 20251030, 29, 0, 2)
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(inst["n"], 3000, replace=False))
    ob = O.sample_subset(x[idx], idx, 20251030, 29, 0, 2)
    assert np.array_equal(bits[idx], ob)
    # evaluator: 4 candidate lanes evaluated one by one by the oracle on the full instance
    feas, z = s.eval(bits)
    for lane in (0, 37, 64, 127):
        xl = ((bits[:, lane // 64] >> np.uint64(lane % 64)) & np.uint64(1)).astype(np.uint8)
        f, zz = o.eval_point(xl)
        assert bool(feas[lane]) == f and z[lane] == zz
    # a feasible lane exists only if it is also feasible for the oracle; the all-ones point is feasible
    f1, z1 = o.eval_point(np.ones(inst["n"], dtype=np.uint8))
    ones = np.full((inst["n"], 1), np.uint64(0xFFFFFFFFFFFFFFFF), dtype=np.uint64)
    fg, zg = s.eval(ones)
    assert f1 and fg.all() and zg[0] == z1 == inst["c"].sum()


@pytest.fixture(scope="module")
def cfg5_tight(cfg5):
    inst, _, _, o = cfg5
    oc = o.preprocess(tol=1e-12, max_iter=2000)
    return inst, o, oc


def test_config5_one_step_parity_full_size(gf, cfg5_tight):
    """One Alg. 2 step at full size from an identical state (oracle preprocess to 1e-12)."""
    inst, o, oc = cfg5_tight
    s = gf.Solver(0)
    s.load(inst)
    s.preprocess(precision=64, tol=1e-12, max_iter=2000)
    rng = np.random.default_rng(3)
    x = rng.random(inst["n"]); xb = rng.random(inst["n"]); y = rng.random(inst["m"]) * 1e-3
    s.set_state(x, xb, y)
    o.set_state(x, xb, y)
    s.step(1, 0.01, 0.99 ** 0.5, 0.99 ** 0.5)
    o.step(0.01, 0.99 ** 0.5, 0.99 ** 0.5)
    xg, _, yg = s.get_state()
    xo, _, yo = o.get_state()
    assert np.linalg.norm(xg - xo) <= 1e-10 * np.linalg.norm(xo)
    assert np.linalg.norm(yg - yo) <= 1e-10 * max(np.linalg.norm(yo), 1e-30)
    assert oc["zero_rows"] == 0
    d = np.abs(xg - xo) / np.maximum(np.abs(xo), 1e-3)
    assert d.max() <= 1e-10, d.max()


def test_config5_one_step_parity_full_size_fp32(gf, cfg5_tight):
    """The bench's precision: one fp32 step at full size (multi-block row kernels, 2.4e4 row blocks)
    from an fp32-representable state; every element within 1e-6 of the oracle's fp64 step."""
    inst, o, _ = cfg5_tight
    s = gf.Solver(0)
    s.load(inst)
    s.preprocess(precision=32, tol=1e-12, max_iter=2000)
    rng = np.random.default_rng(4)
    f32 = lambda v: v.astype(np.float32).astype(np.float64)  # noqa: E731
    x = f32(rng.random(inst["n"])); xb = f32(rng.random(inst["n"])); y = f32(rng.random(inst["m"]) * 1e-3)
    s.set_state(x, xb, y)
    o.set_state(x, xb, y)
    s.step(1, 0.01, 0.99 ** 0.5, 0.99 ** 0.5)
    o.step(0.01, 0.99 ** 0.5, 0.99 ** 0.5)
    xg, xbg, yg = s.get_state()
    xo, xbo, yo = o.get_state()
    for g, v in ((xg, xo), (xbg, xbo), (yg, yo)):
        d = np.abs(g - v) / np.maximum(np.abs(v), 1e-3)
        assert d.max() <= 1e-6, d.max()


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_configs_2_3_4_full_size(gf, cfg):
    """Full-size configs 2-4: 100 fp64 iterations against the oracle (1e-5), sampler and evaluator
    bit-exact on the resulting x_k, incumbent feasibility recomputed by the oracle."""
    inst = G.make_config(cfg, 1)
    s = gf.Solver(0)
    s.load(inst)
    s.preprocess(precision=64, tol=1e-12, max_iter=5000)
    o = O.Oracle(inst)
    o.preprocess(tol=1e-12, max_iter=5000)
    tau = math.sqrt(0.99)
    rho = O.rho_schedule(1e-3, 10.0, 100.0, 2.0, 1e-6, 10)
    o.state_init()
    x0, xb0, y0 = o.get_state()
    s.set_state(x0, xb0, y0)
    for b in range(10):
        s.step(10, rho[b], tau, tau)
        for _ in range(10):
            o.step(rho[b], tau, tau)
    xg, _, yg = s.get_state()
    xo, _, yo = o.get_state()
    assert np.linalg.norm(xg - xo) <= 1e-5 * np.linalg.norm(xo)
    assert np.linalg.norm(yg - yo) <= 1e-5 * max(np.linalg.norm(yo), 1e-12)
    bits = s.sample(xo, 7, 3, 5, 2)
    assert np.array_equal(bits, O.sample(xo, 7, 3, 5, 2))
    fg, zg = s.eval(bits)
    fo, zo = o.eval(bits)
    assert np.array_equal(fg, fo) and np.array_equal(zg, zo)
    info = s.run(max_iters=500, k_b=256)
    z, xbest, meta = s.best_incumbent()
    if not math.isinf(z):
        f, zz = o.eval_point(xbest)
        assert f and zz == (-z if inst["maximize"] else z)


def test_config7_tu_fullsize_lift_consistency(gf):
    """Facility location 512 x 2048 (next row f2) with TUReformulate at full size: for sampled lanes of
    the reduced problem, the GPU's feasibility and objective equal the oracle's evaluation of the
    lifted point x_I = 1 - sum_{i != i_j} y_ij on the ORIGINAL rows (exactness of the theorem)."""
    inst = G.make_config(7, 1)
    s = gf.Solver(0)
    s.load(inst)
    s.tu_reformulate(inst["tu_rows"], inst["tu_cols"])
    s.preprocess(precision=32)
    n = inst["n"]
    keep = np.setdiff1d(np.arange(n), inst["tu_cols"])
    assert s.n == keep.size
    rng = np.random.default_rng(3)
    p = np.where(rng.random(keep.size) < 0.999, 0.0, 1.0)  # sparse assignments: some lanes feasible
    p[: 512] = 1.0  # open every facility
    bits = O.sample(p, 5, 0, 0, 2)
    feas, z = s.eval(bits)
    o = O.Oracle(inst)
    nf, nc = 512, 2048
    for lane in (0, 1, 77, 127):
        xr = ((bits[:, lane // 64] >> np.uint64(lane % 64)) & np.uint64(1)).astype(np.uint8)
        x = np.zeros(n, dtype=np.int64)
        x[keep] = xr
        y = x[nf:].reshape(nc, nf)
        for j, col in enumerate(inst["tu_cols"]):
            x[col] = 1 - (y[j].sum() - y[j, col - nf - j * nf])
        f, zz = o.eval_point(np.clip(x, 0, 1).astype(np.uint8))
        ok_bin = np.all((x >= 0) & (x <= 1))
        assert bool(feas[lane]) == (f and ok_bin)
        if feas[lane]:
            assert z[lane] == zz


def test_config8_assign3d_fullsize_bit_exact(gf):
    """3D assignment n = 64 (next row f3): one Alg. 4 batch at full size is bit-identical to the
    oracle's, and every lane is feasible."""
    inst = G.make_config(8, 1)
    s = gf.Solver(0)
    s.load(inst)
    s.preprocess(precision=32)
    o = O.Oracle(inst)
    p = G.p_vectors(inst["n"], 2)["mix"]
    a = s.sample_assign3d(p, 20251030, 17, 0, 2, 64)
    b = O.sample_assign3d(p, 64, o.canonical_c(), 20251030, 17, 0, 2)
    assert np.array_equal(a, b)
    assert s.eval(a)[0].all()
