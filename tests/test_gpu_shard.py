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


# ----------------------------------------------------------------------------- loopback ranks
def _loop(gf, inst, R, graph=1, opts=(), **kw):
    s = gf.Solver(0, world=R, loopback=True)
    for k, v in opts:
        s.set_option(k, v)
    s.load(inst)
    s.preprocess()
    info = s.run(use_graph=graph, trace_cap=4096, **kw)
    return s, info, s.best_incumbent()


@pytest.mark.parametrize("R", [2, 4, 8])
@pytest.mark.parametrize("graph", [1, 0])
def test_loopback_ranks_equal_one_rank_with_R_times_k_b(gf, R, graph):
    """SURVEY §4(i) / App. B rank invariance: R ranks with k_b each, exchanging records through the
    merge (record -> merge -> Philox regeneration of the winner -> CheckHalt), reproduce one rank with
    R*k_b bit for bit: iterations, halt reason, rounds, incumbent (z, x, iteration, round, global
    index) and the whole trace."""
    inst = G.SMALL["setcover"](2)
    kw = dict(max_iters=600, k_b=64)
    s1 = gf.Solver(0)
    s1.load(inst)
    s1.preprocess()
    i1 = s1.run(use_graph=graph, trace_cap=4096, max_iters=600, k_b=64 * R)
    z1, x1, m1 = s1.best_incumbent()
    s, iR, (zR, xR, mR) = _loop(gf, inst, R, graph, **kw)
    assert (i1["iters"], i1["halt_reason"], i1["rounds"]) == (iR["iters"], iR["halt_reason"], iR["rounds"])
    assert iR["candidates"] == i1["candidates"]
    assert z1 == zR or (math.isinf(z1) and math.isinf(zR))
    assert np.array_equal(x1, xR)
    assert (m1["found_iter"], m1["found_round"], m1["found_index"]) == (mR["found_iter"], mR["found_round"], mR["found_index"])
    assert np.array_equal(s1.trace(), s.trace())


@pytest.mark.parametrize("R,rank,blk", [(2, 1, 3), (4, 2, 5), (8, 7, 0)])
@pytest.mark.parametrize("graph", [1, 0])
def test_loopback_time_limit_flag_halts_every_rank_together(gf, R, rank, blk, graph):
    """CheckHalt's time limit must be agreed: one rank whose clock passes its deadline
    during block `blk` flags it in its record, the merge ORs the flags, and the loop (of every rank)
    stops after that block with halt reason 3 — never with one rank leaving the exchange early."""
    inst = G.SMALL["setcover"](3)
    _, info, _ = _loop(gf, inst, R, graph, opts=[("force_deadline_rank", rank), ("force_deadline_block", blk)],
                       max_iters=1000, k_b=64, **FIXED)
    assert info["halt_reason"] == 3
    assert info["iters"] == (blk + 1) * 10


def test_loopback_real_time_limit(gf):
    """A time limit that has already passed when the first record is written halts after block 1."""
    inst = G.SMALL["setcover"](1)
    _, info, _ = _loop(gf, inst, 4, 1, max_iters=1000, k_b=64, time_limit_s=1e-9, **FIXED)
    assert info["halt_reason"] == 3 and info["iters"] == 10


def test_nccl_path_time_limit_flag(gf):
    """The same agreement on the NCCL path (1-rank communicator: its own flag goes through the
    all-gather and the merge)."""
    try:
        nid = gf.nccl_unique_id()
    except gf.GforsError:
        pytest.skip("libnccl.so.2 not loadable")
    inst = G.SMALL["setcover"](1)
    s = gf.Solver(0, rank=0, world=1, nccl_id=nid)
    s.set_option("force_deadline_rank", 0).set_option("force_deadline_block", 2)
    s.load(inst)
    s.preprocess()
    info = s.run(max_iters=1000, k_b=64, **FIXED)
    assert info["halt_reason"] == 3 and info["iters"] == 30


def test_capture_failure_falls_back_to_eager_loop(gf):
    """If the loop graph cannot be captured (e.g. a collective that cannot live in a conditional
    body) the sharded run falls back to the eager loop with identical results."""
    inst = G.SMALL["setcover"](2)
    _, i0, (z0, x0, m0) = _loop(gf, inst, 2, 1, max_iters=400, k_b=64)
    s, i1, (z1, x1, m1) = _loop(gf, inst, 2, 1, opts=[("force_capture_fail", 1)], max_iters=400, k_b=64)
    assert "forced capture failure" in s.graph_note()
    assert (i0["iters"], i0["halt_reason"], i0["rounds"]) == (i1["iters"], i1["halt_reason"], i1["rounds"])
    assert z0 == z1 or (math.isinf(z0) and math.isinf(z1))
    assert np.array_equal(x0, x1)
    assert (m0["found_iter"], m0["found_round"], m0["found_index"]) == (m1["found_iter"], m1["found_round"], m1["found_index"])


def test_set_option_rejects_unknown_key(gf):
    s = gf.Solver(0)
    with pytest.raises(gf.GforsError, match="unknown key"):
        s.set_option("no_such_option", 1)


# ----------------------------------------------------------------------------- row-sharded dual (f4)
def _state_after(s):
    x, xb, y = s.get_state()
    return x, xb, y


@pytest.mark.parametrize("R", [2, 4, 8])
@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("graph", [1, 0])
def test_row_sharded_dual_bit_identical(gf, R, prec, graph):
    """with params.row_shard each of R ranks (loopback) computes the dual of its
    nnz-balanced range of row blocks, the ranks all-gather y (and K_u xbar at the trigger) and recompute
    w; iterates, trace and incumbent are bit-identical to the unsharded loop with the same samples
    (one rank, k_b * R candidates) — through the dense phase (gather dual) and the push modes."""
    inst = G.set_cover(6000, 30000, 2, 98, 5, "rs_setcover")
    kw = dict(max_iters=600, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0, use_graph=graph,
              trace_cap=4096)
    s1 = gf.Solver(0)
    s1.load(inst)
    s1.preprocess(precision=prec)
    i1 = s1.run(k_b=64 * R, **kw)
    sR = gf.Solver(0, world=R, loopback=True)
    sR.load(inst)
    sR.preprocess(precision=prec)
    iR = sR.run(k_b=64, row_shard=1, **kw)
    assert (i1["iters"], i1["rounds"], i1["halt_reason"]) == (iR["iters"], iR["rounds"], iR["halt_reason"])
    for a, b in zip(_state_after(s1), _state_after(sR)):
        assert np.array_equal(a, b)
    assert np.array_equal(s1.trace(), sR.trace())
    z1, x1, m1 = s1.best_incumbent()
    zR, xR, mR = sR.best_incumbent()
    assert (z1 == zR or (math.isinf(z1) and math.isinf(zR))) and np.array_equal(x1, xR)
    assert iR["launches"] > i1["launches"]  # the per-rank dual launches and the exchange ran


def test_row_sharded_dual_partition_covers_rows(gf):
    """The split is by nonzeros over whole row blocks: with R = 3 ranks on a skewed instance the run is
    still bit-identical (ranks own unequal row counts; the gather slots are padded to the largest)."""
    inst = G.set_cover(5000, 20000, 2, 98, 9, "rs_skew")
    # make the first rows much longer so row counts per rank differ a lot
    kw = dict(max_iters=200, k_int=10, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)
    s1 = gf.Solver(0)
    s1.load(inst)
    s1.preprocess(precision=64)
    s1.run(k_b=192, **kw)
    s3 = gf.Solver(0, world=3, loopback=True)
    s3.load(inst)
    s3.preprocess(precision=64)
    s3.run(k_b=64, row_shard=1, **kw)
    for a, b in zip(_state_after(s1), _state_after(s3)):
        assert np.array_equal(a, b)


def test_row_sharded_nccl_path(gf):
    """The NCCL form of the exchange (ncclAllGather of the packed y / u slots inside the loop graph),
    exercised with a 1-rank communicator: bit-identical to the unsharded run."""
    try:
        nid = gf.nccl_unique_id()
    except gf.GforsError:
        pytest.skip("libnccl.so.2 not loadable")
    inst = G.SMALL["setcover"](4)
    kw = dict(max_iters=300, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)
    s1 = gf.Solver(0)
    s1.load(inst)
    s1.preprocess()
    s1.run(**kw)
    sn = gf.Solver(0, rank=0, world=1, nccl_id=nid)
    sn.load(inst)
    sn.preprocess()
    sn.run(row_shard=1, **kw)
    for a, b in zip(_state_after(s1), _state_after(sn)):
        assert np.array_equal(a, b)


def test_row_shard_errors(gf):
    s = gf.Solver(0)
    s.load(G.SMALL["setcover"](1))
    s.preprocess()
    with pytest.raises(gf.GforsError, match="row_shard"):
        s.run(max_iters=20, row_shard=1)
