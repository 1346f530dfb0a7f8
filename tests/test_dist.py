"""The multi-GPU product partition protocol (paper_0707_2347_b200/dist.py) on
CPU: world sizes 2, 3, 4 and 8 over gloo, one, two and three Winograd levels
(7, 49, 343 products), the operand combinations in exact residue arithmetic and
the products injected from the CPU oracle."""
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


def _worker(rank, world, port, n, alpha, beta, q, levels, window):
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
        st = partitioned_multiply(At, Bt, Ct, alpha, beta, be, levels=levels, window=window)
        want = O.classical_modp(A.astype(np.uint32), B.astype(np.uint32), C0.astype(np.uint32),
                                alpha, beta)
        ok = bool((Ct.numpy().astype(np.uint32) == want).all())
        ok = ok and bool((At.numpy() == A).all() and (Bt.numpy() == B).all())  # read-only
        q.put(("root", ok, st.products, st.peak_extra_bytes, st.bytes_received))
    else:
        st = partitioned_multiply(None, None, None, alpha, beta, be, levels=levels, window=window)
        q.put((rank, True, st.products, st.peak_extra_bytes, st.bytes_sent))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,levels,window", [(2, 1, 2), (3, 1, 1), (2, 2, 2), (3, 2, 3),
                                                 (4, 3, 2), (8, 1, 2), (8, 3, 1)])
def test_partition_gloo(world, levels, window):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    n = 64
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, 3, 7, q, levels, window))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    res = [q.get() for _ in range(world)]
    owned = []
    f = 2 ** levels
    blk = (n // f) ** 2 * 8
    chain = sum((n >> lv) ** 2 * 8 for lv in range(1, levels + 1))  # S (or T) levels held at once
    for who, ok, prods, peak, traffic in res:
        assert ok, who
        owned += prods
        if who == "root":
            # root: its operand chains + product + at most `window` posted receives
            assert peak <= 2 * chain + blk + window * blk, (who, peak)
            assert traffic == blk * (7 ** levels - len(prods))
        else:
            # a copy of A and B, then its operands and every product still in flight
            assert peak <= 2 * n * n * 8 + 2 * chain + len(prods) * blk, (who, peak)
            assert traffic == blk * len(prods)
    assert sorted(owned) == list(range(7 ** levels))  # every product computed exactly once


def test_makespan_bound():
    from paper_0707_2347_b200.dist import makespan_bound
    assert makespan_bound(1) == 1.0
    assert makespan_bound(2) == 7 / 4
    assert makespan_bound(4) == 3.5
    assert makespan_bound(8) == 7.0
    assert makespan_bound(4, 49) == 49 / 13
    assert abs(makespan_bound(8, 343) - 343 / 43) < 1e-12


def test_choose_levels_and_indices():
    from paper_0707_2347_b200.dist import choose_levels, product_indices, targets
    assert [choose_levels(g) for g in (1, 2, 3, 4, 5, 6, 7, 8)] == [1, 2, 3, 3, 2, 3, 1, 3]
    # products must stay above the cutoff: C5 (32768, cutoff 1024) allows all three levels
    assert choose_levels(8, 32768, 1024) == 3 and choose_levels(8, 2048, 512) == 1
    idx = product_indices(2)
    assert len(idx) == 49 and idx[0] == (0, 0) and idx[-1] == (6, 6)
    assert len(product_indices(3)) == 343
    # P1 (index 0) reaches every C block; with three levels 4^3 blocks of C
    C = torch.zeros(16, 16)
    assert len(targets(C, (0, 0, 0))) == 64
    assert all(b.shape == (2, 2) for b, _ in targets(C, (0, 0, 0)))


def test_local_variant():
    from paper_0707_2347_b200.dist import local_variant
    assert local_variant("acc2", 512, 512, 512) == "ip"
    assert local_variant("iprect", 1024, 512, 1024) == "iprect"
    assert local_variant("std2", 512, 1024, 256) == "std2"
