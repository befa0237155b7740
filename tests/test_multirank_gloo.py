"""N > 1 path on CPU (world size 2, gloo): sample-sharded EvalBest.

Rank r draws the global sample words [r*W, (r+1)*W) (Philox counter carries the global word,
DESIGN.md §7), evaluates them (CPU oracle here, the CUDA evaluator on GPUs), all-gathers its
(z, global index, valid) record through torch.distributed and applies the library's merge rule
(gfors_merge_records, host-only).  The merged result must equal one rank drawing all 2W words."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, W, rounds, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    from gen import instances as G
    from oracle import oracle as O
    import paper_2510_27117_b200 as gf

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inst = G.make_config(1, 3)
    o = O.Oracle(inst)
    p = np.full(inst["n"], 0.7)
    out = []
    for rnd in range(rounds):
        bits = O.sample(p, 99, rnd, rank * W, W)
        feas, z = o.eval(bits)
        best = -1
        for l in range(64 * W):
            if feas[l] and (best < 0 or z[l] < z[best]):
                best = l
        rec = torch.tensor([z[best] if best >= 0 else np.inf, 64 * rank * W + max(best, 0), 1.0 if best >= 0 else 0.0],
                           dtype=torch.float64)
        gathered = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, rec)
        zs = np.array([g[0].item() for g in gathered])
        idx = np.array([int(g[1].item()) for g in gathered], dtype=np.int64)
        val = np.array([int(g[2].item()) for g in gathered], dtype=np.int32)
        win = gf.merge_records(zs, idx, val)
        out.append((win, zs[win] if win >= 0 else np.inf, idx[win] if win >= 0 else -1))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, out))


def test_two_rank_sharded_evalbest_equals_single_rank():
    pytest.importorskip("torch.distributed")
    W, rounds, world = 1, 6, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, W, rounds, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    assert res[0] == res[1]  # every rank reaches the same decision

    # single rank drawing all 2W words
    from gen import instances as G
    from oracle import oracle as O
    inst = G.make_config(1, 3)
    o = O.Oracle(inst)
    p = np.full(inst["n"], 0.7)
    for rnd in range(rounds):
        bits = O.sample(p, 99, rnd, 0, world * W)
        feas, z = o.eval(bits)
        ok = np.nonzero(feas)[0]
        if ok.size == 0:
            assert res[0][rnd][0] == -1
            continue
        l = ok[np.argmin(z[ok])]  # argmin returns the lowest index among ties
        assert res[0][rnd][1] == z[l] and res[0][rnd][2] == l
