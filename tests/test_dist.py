"""The multi-GPU product partition protocol (paper_0707_2347_b200/dist.py) on
CPU: world_size 2 and 3 over gloo, with the top-level block combinations in
exact residue arithmetic and the products injected from the CPU oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, alpha, beta, q, levels=1):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    from paper_0707_2347_b200.dist import TorchModP, partitioned_multiply

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = 65521

    def mm(X, Y):
        return torch.from_numpy(O.classical_modp(X.numpy().astype(np.uint32),
                                                 Y.numpy().astype(np.uint32)).astype(np.float64))

    be = TorchModP(p, mm)
    if rank == 0:
        A = O.fill_random(n, n, 1).astype(np.float64)
        B = O.fill_random(n, n, 2).astype(np.float64)
        C0 = O.fill_random(n, n, 3).astype(np.float64)
        At, Bt, Ct = torch.from_numpy(A), torch.from_numpy(B), torch.from_numpy(C0.copy())
        local = partitioned_multiply(At, Bt, Ct, alpha, beta, be, levels=levels)
        want = O.classical_modp(A.astype(np.uint32), B.astype(np.uint32), C0.astype(np.uint32),
                                alpha, beta)
        q.put(("root", bool((Ct.numpy().astype(np.uint32) == want).all()), sorted(local)))
    else:
        local = partitioned_multiply(None, None, None, alpha, beta, be, levels=levels)
        q.put((rank, True, sorted(local)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,levels", [(2, 1), (3, 1), (2, 2), (3, 2)])
def test_partition_gloo(world, levels):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 64, 3, 7, q, levels))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    res = [q.get() for _ in range(world)]
    owned = []
    for who, ok, prods in res:
        assert ok, who
        owned += prods
    assert sorted(owned) == list(range(7 ** levels))  # every product computed exactly once


def test_makespan_bound():
    from paper_0707_2347_b200.dist import makespan_bound
    assert makespan_bound(1) == 1.0
    assert makespan_bound(2) == 7 / 4
    assert makespan_bound(4) == 3.5
    assert makespan_bound(8) == 7.0
    assert makespan_bound(4, 49) == 49 / 13


def test_choose_levels_and_indices():
    from paper_0707_2347_b200.dist import choose_levels, product_indices
    assert [choose_levels(g) for g in (1, 2, 3, 4, 7, 8)] == [1, 2, 2, 2, 1, 1]
    idx = product_indices(2)
    assert len(idx) == 49 and idx[0] == (0, 0) and idx[-1] == (6, 6)
