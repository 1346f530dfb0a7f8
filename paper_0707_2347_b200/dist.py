"""Multi-GPU product partition of the top Winograd level.

One process per GPU.  The root rank holds A, B, C.  The top level uses the
Table-1 (std2) formulas:

    P1 = A11 B11        P2 = A12 B21        P3 = S4 B22          P4 = A22 T4
    P5 = S1 T1          P6 = S2 T2          P7 = S3 T3
    S1 = A21+A22  S2 = S1-A11  S3 = A11-A21  S4 = A12-S2
    T1 = B12-B11  T2 = B22-T1  T3 = B22-B12  T4 = T2-B21
    C11 = P1+P2   C12 = P1+P6+P5+P3   C21 = P1+P6+P7-P4   C22 = P1+P6+P7+P5

Product i is owned by rank i mod G.  The root forms each remote product's
operands (S_i, T_i) and sends them (point-to-point, NCCL over NVLink on GPUs);
every rank computes its products with the single-GPU memory-lean plan of the
local schedule (C-ABI run_variant); the P_i come back to the root, which folds
each one into the C quadrants as it arrives (alpha, beta applied once).  The
network carries only operand blocks and products, as north_star specifies.

The exchange logic is backend-agnostic: ``CudaBackend`` runs the block
combinations and products through libwinomem_b200 on the rank's GPU; tests
drive the same protocol on CPU tensors over gloo with an injected product.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Sequence, Tuple

import torch
import torch.distributed as dist

# quadrant coefficients over (11, 12, 21, 22)
S_COEF = [(1, 0, 0, 0), (0, 1, 0, 0), (1, 1, -1, -1), (0, 0, 0, 1), (0, 0, 1, 1),
          (-1, 0, 1, 1), (1, 0, -1, 0)]
T_COEF = [(1, 0, 0, 0), (0, 0, 1, 0), (0, 0, 0, 1), (1, -1, -1, 1), (-1, 1, 0, 0),
          (1, -1, 0, 1), (0, -1, 0, 1)]
# C quadrant (11, 12, 21, 22) += coef * P_i
C_COEF = [(1, 1, 1, 1), (1, 0, 0, 0), (0, 1, 0, 0), (0, 0, -1, 0), (0, 1, 0, 1), (0, 1, 1, 1),
          (0, 0, 1, 1)]


def owner(i: int, world: int) -> int:
    return i % world


def quads(M: torch.Tensor) -> List[torch.Tensor]:
    r, c = M.shape[0] // 2, M.shape[1] // 2
    return [M[:r, :c], M[:r, c:], M[r:, :c], M[r:, c:]]


@dataclass
class TorchModP:
    """Reference backend on torch tensors (any device): exact residue arithmetic
    in float64.  Used by the CPU protocol tests; the product is injected."""
    p: int
    mm: Callable[[torch.Tensor, torch.Tensor], torch.Tensor]

    def lincomb(self, coefs: Sequence[int], blocks: Sequence[torch.Tensor]) -> torch.Tensor:
        out = torch.zeros_like(blocks[0])
        for c, b in zip(coefs, blocks):
            if c:
                out = out + c * b
        return torch.remainder(out, self.p)

    def product(self, X: torch.Tensor, Y: torch.Tensor) -> torch.Tensor:
        return self.mm(X, Y)

    def fold(self, Cq: torch.Tensor, coef: int, P: torch.Tensor):
        Cq.copy_(torch.remainder(Cq + coef * P, self.p))

    def finish(self, Cq: torch.Tensor, acc: torch.Tensor, alpha: int, beta: int):
        Cq.copy_(torch.remainder(alpha * acc + beta * Cq, self.p))


class CudaBackend:
    """libwinomem_b200 on this rank's GPU: block combinations with the block
    addition kernels, products with the single-GPU memory-lean plan."""

    def __init__(self, p: int, variant: str, cutoff: int, device: int, real: bool = False):
        from . import winomem as W
        self.W = W
        self.p, self.variant, self.cutoff, self.device, self.real = p, variant, cutoff, device, real
        # REAL64 primitives read the uint32 scalar as a signed int32
        self.m = (1 << 32) if real else p

    def _mat(self, t: torch.Tensor):
        return self.W.Matrix.wrap(t, self.W.Modulus(self.p), real=self.real)

    def lincomb(self, coefs, blocks):
        W = self.W
        out = torch.empty_like(blocks[0])
        terms = [(c % self.m, b) for c, b in zip(coefs, blocks) if c]
        O = self._mat(out)
        first = True
        for c, b in terms:
            Bm = self._mat(b)
            if first:
                W.block_scale_copy(O.view(), Bm.view(), c)
                first = False
            else:
                W.block_addsub(O.view(), O.view(), Bm.view(), 1, c)
        return out

    def product(self, X, Y):
        out = torch.empty((X.shape[0], Y.shape[1]), dtype=X.dtype, device=X.device)
        self.W.run_variant(self.variant, self._mat(X), self._mat(Y), self._mat(out),
                           alpha=1, beta=0, cutoff=self.cutoff)
        return out

    def zero(self, Cq):
        Cq.zero_()

    def fold(self, Cq, coef, P):
        M = self._mat(Cq)
        self.W.block_addsub(M.view(), M.view(), self._mat(P).view(), 1, coef % self.m)

    def finish(self, Cq, acc, alpha, beta):
        M = self._mat(Cq)
        self.W.block_addsub(M.view(), self._mat(acc).view(), M.view(), alpha % self.m,
                            beta % self.m)


def partitioned_multiply(A, B, C, alpha: int, beta: int, backend, group=None, root: int = 0):
    """C <- alpha*A*B + beta*C with the 7 top-level products spread over the
    ranks of `group`.  A, B, C are only read on the root; other ranks pass
    None (their shapes are broadcast).  Returns the products computed locally."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    meta = torch.zeros(4, dtype=torch.int64)
    dev = A.device if rank == root else None
    if rank == root:
        meta[:] = torch.tensor([A.shape[0], A.shape[1], B.shape[1], 0])
    if dist.get_backend(group) == "nccl":
        meta = meta.cuda()
    dist.broadcast(meta, src=root, group=group)
    m, k, n = (int(x) for x in meta[:3].tolist())
    if rank != root:
        dev = meta.device if meta.is_cuda else torch.device("cpu")
    h_m, h_k, h_n = m // 2, k // 2, n // 2
    mine = [i for i in range(7) if owner(i, world) == rank]

    if rank == root:
        Aq, Bq = quads(A), quads(B)
        acc = [torch.zeros((h_m, h_n), dtype=A.dtype, device=dev) for _ in range(4)]
        # operands of remote products go out first so remote ranks start early
        reqs, keep = [], []
        for i in range(7):
            o = owner(i, world)
            if o == root:
                continue
            X = backend.lincomb(S_COEF[i], Aq)
            Y = backend.lincomb(T_COEF[i], Bq)
            keep += [X, Y]
            reqs.append(dist.isend(X, dst=o, group=group))
            reqs.append(dist.isend(Y, dst=o, group=group))
        # post every product receive now: a remote rank may finish its first
        # product before the root has handed out all operands
        pending = []
        for i in range(7):
            o = owner(i, world)
            if o == root:
                continue
            P = torch.empty((h_m, h_n), dtype=A.dtype, device=dev)
            pending.append((i, P, dist.irecv(P, src=o, group=group)))
        local = {}
        for i in mine:
            X = backend.lincomb(S_COEF[i], Aq)
            Y = backend.lincomb(T_COEF[i], Bq)
            P = backend.product(X, Y)
            local[i] = P
            for q in range(4):
                if C_COEF[i][q]:
                    backend.fold(acc[q], C_COEF[i][q], P)
        for i, P, req in pending:
            req.wait()
            for q in range(4):
                if C_COEF[i][q]:
                    backend.fold(acc[q], C_COEF[i][q], P)
        for r in reqs:
            r.wait()
        Cq = quads(C)
        for q in range(4):
            backend.finish(Cq[q], acc[q], alpha, beta)
        return local
    local = {}
    for i in mine:
        X = torch.empty((h_m, h_k), dtype=torch.float64, device=dev)
        Y = torch.empty((h_k, h_n), dtype=torch.float64, device=dev)
        dist.recv(X, src=root, group=group)
        dist.recv(Y, src=root, group=group)
        P = backend.product(X, Y)
        local[i] = P
        dist.send(P, dst=root, group=group)
    return local


def local_variant(variant: str, m: int, k: int, n: int) -> str:
    """Schedule for the plain products P_i = S_i T_i on each rank."""
    if variant == "ipmm":
        return "ipmm"
    if variant in ("ip", "ovl", "ovl2", "ovr", "iprect", "ipovmm", "aclr"):
        return "ip" if m == k == n else "iprect"
    return "std2"


def makespan_bound(world: int, products: int = 7) -> float:
    """Ideal speed-up of the partition in product units."""
    per = -(-products // world)
    return products / per
