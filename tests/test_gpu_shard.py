"""Sample sharding on one GPU: (1) independent shards (nccl_id NULL) cover disjoint Philox word ranges,
so the best of two ranks equals one rank with twice the batch; (2) the in-loop NCCL exchange path
(world = 1 communicator, the same kernels and collective call as world = N) reproduces the
unsharded run exactly."""
import math

import numpy as np
import pytest

from gen import instances as G

pytestmark = pytest.mark.gpu
FIXED = dict(tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)


@pytest.fixture(scope="module")
def gf():
    import paper_2510_27117_b200 as gf
    return gf


def _solve(gf, inst, **kw):
    ctor = {k: kw.pop(k) for k in ("rank", "world", "nccl_id") if k in kw}
    s = gf.Solver(0, **ctor)
    s.load(inst)
    s.preprocess()
    info = s.run(**kw)
    return s, info, s.best_incumbent()


@pytest.mark.parametrize("seed", [1, 2])
def test_two_independent_shards_equal_one_rank_double_batch(gf, seed):
    inst = G.make_config(1, seed)
    _, _, (z1, _, _) = _solve(gf, inst, max_iters=300, k_b=128, **FIXED)
    zs = []
    for r in range(2):
        _, info, (z, x, meta) = _solve(gf, inst, max_iters=300, k_b=64, rank=r, world=2, **FIXED)
        zs.append(z)
        if meta["found_index"] >= 0:
            assert 64 * r <= meta["found_index"] % 128 < 64 * (r + 1)  # rank r owns words [r, r+1)
    assert min(zs) == z1


@pytest.mark.parametrize("graph", [1, 0])
def test_nccl_exchange_path_matches_unsharded(gf, graph):
    try:
        nid = gf.nccl_unique_id()
    except gf.GforsError:
        pytest.skip("libnccl.so.2 not loadable")
    inst = G.SMALL["setcover"](3)
    _, i0, (z0, x0, m0) = _solve(gf, inst, max_iters=400, use_graph=graph)
    s, i1, (z1, x1, m1) = _solve(gf, inst, max_iters=400, use_graph=graph, rank=0, world=1, nccl_id=nid)
    assert i0["iters"] == i1["iters"] and i0["halt_reason"] == i1["halt_reason"] and i0["rounds"] == i1["rounds"]
    assert z0 == z1 or (math.isinf(z0) and math.isinf(z1))
    assert np.array_equal(x0, x1)
    assert (m0["found_iter"], m0["found_round"], m0["found_index"]) == (m1["found_iter"], m1["found_round"], m1["found_index"])
    print("graph note:", s.graph_note())


def test_nccl_exchange_config1_incumbent(gf):
    try:
        nid = gf.nccl_unique_id()
    except gf.GforsError:
        pytest.skip("libnccl.so.2 not loadable")
    inst = G.make_config(1, 2)
    _, i0, (z0, x0, m0) = _solve(gf, inst, max_iters=2000)
    _, i1, (z1, x1, m1) = _solve(gf, inst, max_iters=2000, rank=0, world=1, nccl_id=nid)
    assert z0 == z1 and np.array_equal(x0, x1) and i0["iters"] == i1["iters"]
