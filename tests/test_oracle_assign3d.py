"""Pins of the oracle's customised 3D-assignment sampler (PAPER Alg. 4; SPEC L342-350;
next row f3): feasibility by construction, the SPEC worked cases, monotone local improvement,
uniform random completion, and lane-range composition.  CPU only."""
import math

import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O


def _lane_points(bits, n3):
    lanes = 64 * bits.shape[1]
    return np.array([((bits[:, l // 64] >> np.uint64(l % 64)) & np.uint64(1)).astype(np.uint8) for l in range(lanes)])


@pytest.mark.parametrize("n,gamma,L", [(2, 4.0, 4), (5, 4.0, 10), (7, 1.0, 0), (9, 2.5, 18), (6, 0.0001, 3)])
def test_every_lane_is_a_3d_assignment(n, gamma, L):
    """every returned row satisfies all three constraint groups of eq. assign3d exactly
    (checked with the oracle's EvalBest on the original rows and directly on the triples)."""
    inst = G.assignment3d(n, n)
    o = O.Oracle(inst)
    c = o.canonical_c()
    p = np.random.default_rng(n).random(n ** 3)
    bits = O.sample_assign3d(p, n, c, 11, 3, 0, 2, gamma, L)
    feas, z = o.eval(bits)
    assert feas.all()
    for x in _lane_points(bits, n ** 3):
        t = np.flatnonzero(x)
        assert t.size == n
        for axis in (t // (n * n), (t // n) % n, t % n):
            assert np.array_equal(np.sort(axis), np.arange(n))


def test_spec_examples():
    """n = 1 -> (0,0,0); p >= 0.9 on a full permutation triple set with gamma = 1 and
    no local steps -> that assignment in every lane."""
    bits = O.sample_assign3d(np.array([0.3]), 1, np.array([5.0]), 1, 0, 0, 1, 4.0, 2)
    assert bits[0, 0] == np.uint64(0xFFFFFFFFFFFFFFFF)
    n = 6
    rng = np.random.default_rng(1)
    sj, sk = rng.permutation(n), rng.permutation(n)
    p = rng.random(n ** 3) * 0.5
    target = np.arange(n) * n * n + sj * n + sk
    p[target] = 0.9 + 0.05 * rng.random(n)
    bits = O.sample_assign3d(p, n, rng.integers(1, 100, n ** 3).astype(float), 4, 0, 0, 2, 1.0, 0)
    expect = np.zeros(n ** 3, dtype=np.uint8)
    expect[target] = 1
    for x in _lane_points(bits, n ** 3):
        assert np.array_equal(x, expect)


def test_local_improvement_never_worsens():
    """Step (4) only applies strictly improving interchanges: with the same completion draws, every
    lane's cost after L steps is <= its cost with L = 0, and strictly lower somewhere."""
    n = 8
    inst = G.assignment3d(n, 3)
    o = O.Oracle(inst)
    c = o.canonical_c()
    p = np.random.default_rng(2).random(n ** 3)
    _, z0 = o.eval(O.sample_assign3d(p, n, c, 5, 1, 0, 2, 2.0, 0))
    _, zL = o.eval(O.sample_assign3d(p, n, c, 5, 1, 0, 2, 2.0, 40))
    assert np.all(zL <= z0) and np.any(zL < z0)


def test_random_completion_is_uniform():
    """Step (3): with one pre-assigned triple and n = 3, the 2! * 2! = 4 completions are equally
    likely (counts over 4096 lanes within 4 sigma of 1024)."""
    n = 3
    p = np.zeros(27)
    p[0] = 1.0  # partial assignment {(0,0,0)} (K = 1)
    bits = O.sample_assign3d(p, n, np.ones(27), 77, 9, 0, 64, 0.3, 0)
    counts = {}
    for x in _lane_points(bits, 27):
        key = tuple(np.flatnonzero(x))
        counts[key] = counts.get(key, 0) + 1
    assert len(counts) == 4
    for v in counts.values():
        assert abs(v - 1024) <= 4 * math.sqrt(4096 * 0.25 * 0.75)


def test_lane_ranges_compose():
    n = 4
    c = np.arange(64, dtype=float)
    p = np.random.default_rng(3).random(64)
    full = O.sample_assign3d(p, n, c, 9, 2, 0, 3, 4.0, 8)
    a = O.sample_assign3d(p, n, c, 9, 2, 0, 1, 4.0, 8)
    b = O.sample_assign3d(p, n, c, 9, 2, 1, 2, 4.0, 8)
    assert np.array_equal(full, np.concatenate([a, b], axis=1))
