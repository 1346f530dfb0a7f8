"""Multi-GPU product partition of the top one or two Winograd levels.

One process per GPU.  The root rank holds A, B, C.  The top level uses the
Table-1 (std2) formulas:

    P1 = A11 B11        P2 = A12 B21        P3 = S4 B22          P4 = A22 T4
    P5 = S1 T1          P6 = S2 T2          P7 = S3 T3
    S1 = A21+A22  S2 = S1-A11  S3 = A11-A21  S4 = A12-S2
    T1 = B12-B11  T2 = B22-T1  T3 = B22-B12  T4 = T2-B21
    C11 = P1+P2   C12 = P1+P6+P5+P3   C21 = P1+P6+P7-P4   C22 = P1+P6+P7+P5

With two levels the same formulas are applied again to each S_i / T_i, giving
49 products P_(i,j) of quarter size; P_(i,j) folds into sub-quadrant q2 of C
quadrant q1 with coefficient C_COEF[i][q1] * C_COEF[j][q2].  Product t is owned
by rank t mod G.  The root forms each remote product's
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


def product_indices(levels: int) -> List[Tuple[int, ...]]:
    """The 7^levels products of `levels` Winograd levels, as index tuples
    (outer level first), in the order they are assigned to ranks."""
    out: List[Tuple[int, ...]] = [()]
    for _ in range(levels):
        out = [t + (i,) for t in out for i in range(7)]
    return out


def _operand(M, idx, coef, backend):
    """S_idx(A) / T_idx(B) through the levels: quadrant combination of the
    previous level's operand."""
    X = M
    for i in idx:
        X = backend.lincomb(coef[i], quads(X))
    return X


def _target(acc_quads, idx):
    """(accumulator block, coefficient) a product P_idx folds into: P_(i1,i2)
    adds C_COEF[i1][q1] * C_COEF[i2][q2] * P to sub-quadrant q2 of quadrant q1."""
    out = []
    for q1 in range(4):
        c1 = C_COEF[idx[0]][q1]
        if not c1:
            continue
        if len(idx) == 1:
            out.append((acc_quads[q1], c1))
            continue
        for q2 in range(4):
            c2 = C_COEF[idx[1]][q2]
            if c2:
                out.append((quads(acc_quads[q1])[q2], c1 * c2))
    return out


def partitioned_multiply(A, B, C, alpha: int, beta: int, backend, group=None, root: int = 0,
                         levels: int = 1):
    """C <- alpha*A*B + beta*C with the 7^levels products of the top `levels`
    Winograd levels (7 or 49) spread over the ranks of `group` (product t on
    rank t mod G).  A, B, C are only read on the root; other ranks pass None
    (their shapes are broadcast).  Returns the products computed locally, keyed
    by their index in product_indices(levels)."""
    if levels not in (1, 2):
        raise ValueError("levels must be 1 (7 products) or 2 (49 products)")
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
    f = 2 ** levels
    b_m, b_k, b_n = m // f, k // f, n // f
    prods = product_indices(levels)
    mine = [t for t in range(len(prods)) if owner(t, world) == rank]

    if rank == root:
        acc = [torch.zeros((m // 2, n // 2), dtype=A.dtype, device=dev) for _ in range(4)]
        # operands of remote products go out first so remote ranks start early
        reqs, keep = [], []
        for t, idx in enumerate(prods):
            o = owner(t, world)
            if o == root:
                continue
            X = _operand(A, idx, S_COEF, backend)
            Y = _operand(B, idx, T_COEF, backend)
            keep += [X, Y]
            reqs.append(dist.isend(X, dst=o, group=group))
            reqs.append(dist.isend(Y, dst=o, group=group))
        # post every product receive now: a remote rank may finish its first
        # product before the root has handed out all operands
        pending = []
        for t, idx in enumerate(prods):
            o = owner(t, world)
            if o == root:
                continue
            P = torch.empty((b_m, b_n), dtype=A.dtype, device=dev)
            pending.append((idx, P, dist.irecv(P, src=o, group=group)))
        local = {}
        for t in mine:
            idx = prods[t]
            P = backend.product(_operand(A, idx, S_COEF, backend), _operand(B, idx, T_COEF, backend))
            local[t] = P
            for blk, coef in _target(acc, idx):
                backend.fold(blk, coef, P)
        for idx, P, req in pending:
            req.wait()
            for blk, coef in _target(acc, idx):
                backend.fold(blk, coef, P)
        for r in reqs:
            r.wait()
        Cq = quads(C)
        for q in range(4):
            backend.finish(Cq[q], acc[q], alpha, beta)
        return local
    local = {}
    for t in mine:
        X = torch.empty((b_m, b_k), dtype=torch.float64, device=dev)
        Y = torch.empty((b_k, b_n), dtype=torch.float64, device=dev)
        dist.recv(X, src=root, group=group)
        dist.recv(Y, src=root, group=group)
        P = backend.product(X, Y)
        local[t] = P
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


def choose_levels(world: int) -> int:
    """7 products when they already fill the ranks as well as 49 would (G = 1,
    7, 8: same makespan, fewer and larger products); 49 otherwise (G = 2: 1.96x
    instead of 1.75x, G = 4: 3.77x instead of 3.5x)."""
    return 1 if makespan_bound(world, 7) >= makespan_bound(world, 49) else 2
