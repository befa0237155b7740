"""Large pinned host inputs take the device validation path of gfors_load (load_impl.inc,
validate_K_device: the caller's K is DMA'd once and checked + classified by a kernel).  It must build
exactly the problem the host path builds (same evaluation, same run) and fail with the host path's
error messages."""
import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gf():
    import paper_2510_27117_b200 as gf
    return gf


def _pinned(inst):
    import torch
    return {k: (torch.from_numpy(np.ascontiguousarray(v)).pin_memory().numpy() if isinstance(v, np.ndarray) else v)
            for k, v in inst.items()}


def _instances():
    cover = G.set_cover(30_000, 120_000, 2, 98, 5, name="pinned_cover")        # SIGN rows, ~1.5M nonzeros
    mkp = G.multi_knapsack(40_000, 30, 0.9, 3, name="pinned_mkp")               # int8 values, ~1.1M nonzeros
    mixed = dict(cover)                                                         # LE rows: non-canonical order
    mixed["k_val"] = cover["k_val"].copy()
    mixed["sense"] = cover["sense"].copy()
    ptr = cover["k_rowptr"]
    for j in range(0, cover["m"], 3):
        mixed["k_val"][ptr[j]:ptr[j + 1]] *= -1.0
        mixed["r"] = mixed["r"].copy() if j == 0 else mixed["r"]
        mixed["r"][j] = -cover["r"][j]
        mixed["sense"][j] = -1
    frac = dict(mkp)
    frac["k_val"] = mkp["k_val"] * 0.5                                          # fp64 values
    return {"cover": cover, "mkp": mkp, "mixed": mixed, "frac": frac}


@pytest.mark.parametrize("name", ["cover", "mkp", "mixed", "frac"])
def test_pinned_load_builds_the_same_problem(gf, name):
    inst = _instances()[name]
    assert int(inst["k_rowptr"][-1]) >= 1 << 20
    p = G.p_vectors(inst["n"], 3)["unif"]
    bits = O.sample(p, 9, 1, 0, 2)
    res = []
    for host in (inst, _pinned(inst)):
        s = gf.Solver(0)
        s.load(host)
        s.preprocess(precision=64)
        f, z = s.eval(bits)
        info = s.run(max_iters=40, k_b=128, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)
        x, xb, y = s.get_state()
        res.append((f, z, info["iters"], x, xb, y, s.scaled()))
        s.close()
    a, b = res
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    for u, v in zip(a[3:6], b[3:6]):
        assert np.array_equal(u, v)
    for u, v in zip(a[6], b[6]):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("fault", ["col_range", "col_order", "nan", "zero"])
def test_pinned_load_error_messages(gf, fault):
    inst = dict(_instances()["cover"])
    inst["k_col"] = inst["k_col"].copy()
    inst["k_val"] = inst["k_val"].copy()
    ptr = inst["k_rowptr"]
    j = 12345
    q = int(ptr[j]) + 1
    if fault == "col_range":
        inst["k_col"][q] = inst["n"] + 7
    elif fault == "col_order":
        inst["k_col"][q] = inst["k_col"][q - 1]
    elif fault == "nan":
        inst["k_val"][q] = np.nan
    else:
        inst["k_val"][q] = 0.0
    msgs = []
    for host in (inst, _pinned(inst)):
        s = gf.Solver(0)
        with pytest.raises(gf.GforsError) as e:
            s.load(host)
        msgs.append(str(e.value))
        s.close()
    assert msgs[0] == msgs[1], msgs
