"""Caller allocator of gfors_device_opts (include/gfors.h): with torch's caching
allocator every device buffer of the context comes from torch (visible in memory_allocated, returned
at close), and the solve is bit-identical to one on the library's private pool."""
import numpy as np
import pytest

from gen import instances as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gf():
    import paper_2510_27117_b200 as gf
    return gf


@pytest.mark.parametrize("family", ["config1", "mis"])
def test_torch_allocator_same_solve_and_accounting(gf, family):
    import torch
    inst = G.make_config(1, 1) if family == "config1" else G.SMALL["mis"](3)
    res = []
    for alloc in (None, "torch"):
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated(0)
        s = gf.Solver(0, allocator=alloc)
        s.load(inst)
        s.preprocess(precision=64)
        info = s.run(max_iters=600, k_b=128)
        z, x, meta = s.best_incumbent()
        used = torch.cuda.memory_allocated(0) - base
        s.close()
        torch.cuda.synchronize()
        after = torch.cuda.memory_allocated(0) - base
        res.append((info["iters"], info["halt_reason"], z, x, meta["found_iter"]))
        if alloc == "torch":
            assert used > 0 and after == 0, (used, after)
        else:
            assert used == 0
    assert res[0][:3] == res[1][:3] and np.array_equal(res[0][3], res[1][3]) and res[0][4] == res[1][4]


def test_allocator_pair_required(gf):
    import ctypes as C
    with pytest.raises(gf.GforsError):
        gf.Solver(0, allocator=(gf.ALLOC_FN(lambda n, c: None), gf.FREE_FN()))


def test_allocator_failure_is_oom(gf):
    s = gf.Solver(0, allocator=(gf.ALLOC_FN(lambda n, c: None), gf.FREE_FN(lambda p, c: None)))
    with pytest.raises(gf.GforsError, match="E_OOM"):
        s.load(G.make_config(1, 1))
    s.close()


def test_release_memory(gf):
    """gfors_release_memory: refused while a solver of the device lives, then returns the pool's memory."""
    s = gf.Solver(0)
    s.load(G.make_config(1, 1))
    with pytest.raises(gf.GforsError):
        gf.release_memory(0)
    s.close()
    gf.release_memory(0)
    with pytest.raises(gf.GforsError):
        gf.release_memory(99)
