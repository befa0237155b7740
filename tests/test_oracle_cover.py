"""Pins of the oracle's cover completion (reading R27; "first generate a feasible
candidate from the fractional solution p"): on set cover every lane becomes feasible, feasible lanes
are unchanged, sampled ones are kept, and every added variable is the largest-p variable (ties: lowest
index) of a row the lane violated.  CPU only."""
import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O


def _pts(bits):
    return np.array([((bits[:, l // 64] >> np.uint64(l % 64)) & np.uint64(1)).astype(np.uint8)
                     for l in range(64 * bits.shape[1])])


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_cover_completion_properties(seed):
    inst = G.set_cover(80, 300, 2, 12, seed)
    o = O.Oracle(inst)
    rng = np.random.default_rng(seed)
    p = np.round(rng.random(300) * 0.2, 2)  # ties are common
    bits = O.sample(p, seed, 0, 0, 2)
    f0, _ = o.eval(bits)
    out = o.cover_complete(p, bits)
    f1, _ = o.eval(out)
    assert f1.all()
    K = G.dense_K(inst)
    X0, X1 = _pts(bits), _pts(out)
    for l in range(X0.shape[0]):
        if f0[l]:
            assert np.array_equal(X0[l], X1[l])
        assert np.all(X1[l] >= X0[l])
        viol = np.flatnonzero(K @ X0[l] < 1)
        bests = set()
        for j in viol:
            cols = np.flatnonzero(K[j])
            top = cols[np.argmax(p[cols])]  # argmax returns the lowest index among ties
            bests.add(int(top))
        assert set(np.flatnonzero(X1[l] > X0[l]).tolist()) <= bests


def test_cover_completion_skips_other_rows():
    """Rows that are not covering rows (rhs != 1, a coefficient != 1, or equalities) get no additions."""
    inst = G.random_general(30, 10, 4, 5, 2)
    o = O.Oracle(inst)
    bits = O.sample(np.full(30, 0.3), 4, 0, 0, 1)
    out = o.cover_complete(np.full(30, 0.3), bits)
    m1 = o.m1
    Ku = G.dense_K(inst)[o.row_perm()] * np.where(inst["sense"][o.row_perm()] == -1, -1.0, 1.0)[:, None]
    ru = inst["r"][o.row_perm()] * np.where(inst["sense"][o.row_perm()] == -1, -1.0, 1.0)
    elig = [(j < m1 and ru[j] == 1 and np.all(Ku[j][Ku[j] != 0] == 1) and np.any(Ku[j])) for j in range(inst["m"])]
    if not any(elig):
        assert np.array_equal(out, bits)
