"""Multi-GPU product partition of the top Winograd levels.

One process per GPU.  The root rank holds A, B, C.  The top level uses the
Table-1 (std2) formulas:

    P1 = A11 B11        P2 = A12 B21        P3 = S4 B22          P4 = A22 T4
    P5 = S1 T1          P6 = S2 T2          P7 = S3 T3
    S1 = A21+A22  S2 = S1-A11  S3 = A11-A21  S4 = A12-S2
    T1 = B12-B11  T2 = B22-T1  T3 = B22-B12  T4 = T2-B21
    C11 = P1+P2   C12 = P1+P6+P5+P3   C21 = P1+P6+P7-P4   C22 = P1+P6+P7+P5

With L levels the formulas are applied again to each operand, giving 7^L
products P_(i1..iL) of size n/2^L; P_(i1..iL) folds into the nested
sub-quadrant (q1..qL) of C with coefficient prod_l C_COEF[i_l][q_l].
Product t (in `product_indices` order) is owned by rank t mod G.

Protocol (NCCL over NVLink on GPUs; gloo in the CPU tests):
  1. the root broadcasts A and B (one collective each);
  2. every rank forms its own operands S_t, T_t from its copy with the one-pass
     combination kernel (wm_lincomb: up to four quadrants per level), so no rank
     waits for the root to build operands;
  3. every rank multiplies them with the single-GPU memory-lean plan (the
     in-place schedule `ip` on square operands: the operands are scratch
     copies, so the local product needs no temporaries at all);
  4. remote products go back to the root with non-blocking sends in product
     order; the root scales C by beta once and folds alpha * coef * P_t straight
     into the C blocks as each product arrives -- no full-size accumulator.
     The root keeps at most `window` receives posted, in product order, which is
     also each sender's order, so every pair of ranks sees its messages in the
     same order on its channel (no cross-ordering deadlock).
The network carries only the operand sources and the products, as north_star
specifies.  Every rank reports the peak extra bytes it held (operand copies,
operands, products, receive buffers, plus the local plan's temporaries).

The exchange logic is backend-agnostic: ``CudaBackend`` runs the combinations,
folds and products through libwinomem_b200 on the rank's GPU; tests drive the
same protocol on CPU tensors over gloo with an injected product.
"""
from __future__ import annotations

from dataclasses import dataclass, field
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

MAX_LEVELS = 3


def owner(i: int, world: int) -> int:
    return i % world


def quads(M: torch.Tensor) -> List[torch.Tensor]:
    r, c = M.shape[0] // 2, M.shape[1] // 2
    return [M[:r, :c], M[:r, c:], M[r:, :c], M[r:, c:]]


def _bytes(t: torch.Tensor) -> int:
    return t.numel() * t.element_size()


@dataclass
class TorchModP:
    """Reference backend on torch tensors (any device): exact residue arithmetic
    in float64.  Used by the CPU protocol tests; the product is injected."""
    p: int
    mm: Callable[[torch.Tensor, torch.Tensor], torch.Tensor]

    def lincomb(self, terms: Sequence[Tuple[int, torch.Tensor]]) -> torch.Tensor:
        out = torch.zeros_like(terms[0][1])
        for c, b in terms:
            out = out + c * b
        return torch.remainder(out, self.p)

    def product(self, X: torch.Tensor, Y: torch.Tensor) -> Tuple[torch.Tensor, int]:
        return self.mm(X, Y), 0

    def scale(self, Cq: torch.Tensor, beta: int):
        Cq.copy_(torch.remainder(beta * Cq, self.p))

    def fold(self, Cq: torch.Tensor, coef: int, P: torch.Tensor):
        Cq.copy_(torch.remainder(Cq + coef * P, self.p))


class CudaBackend:
    """libwinomem_b200 on this rank's GPU: operand combinations and folds with
    the one-pass combination kernel, products with the single-GPU memory-lean
    plan of `variant`."""

    def __init__(self, p: int, variant: str, cutoff: int, device: int, real: bool = False):
        from . import winomem as W
        self.W = W
        self.p, self.variant, self.cutoff, self.device, self.real = p, variant, cutoff, device, real
        # REAL64 primitives read the uint32 scalar as a signed int32
        self.m = (1 << 32) if real else p
        self.launches = 0  # kernels this backend issued (bench.py's gpu_launches)

    def _mat(self, t: torch.Tensor):
        return self.W.Matrix.wrap(t, self.W.Modulus(self.p), real=self.real)

    def lincomb(self, terms):
        out = torch.empty_like(terms[0][1])
        self.W.lincomb(self._mat(out).view(), [(c % self.m, self._mat(b).view()) for c, b in terms])
        self.launches += 1
        return out

    def product(self, X, Y):
        out = torch.empty((X.shape[0], Y.shape[1]), dtype=X.dtype, device=X.device)
        rep = self.W.run_variant(self.variant, self._mat(X), self._mat(Y), self._mat(out),
                                 alpha=1, beta=0, cutoff=self.cutoff)
        self.launches += rep.n_launches
        return out, rep.peak_extra_bytes

    def scale(self, Cq, beta):
        M = self._mat(Cq)
        self.W.block_scale_copy(M.view(), M.view(), beta % self.m)
        self.launches += 1

    def fold(self, Cq, coef, P):
        M = self._mat(Cq)
        self.W.block_addsub(M.view(), M.view(), self._mat(P).view(), 1, coef % self.m)
        self.launches += 1


def product_indices(levels: int) -> List[Tuple[int, ...]]:
    """The 7^levels products of `levels` Winograd levels, as index tuples
    (outer level first), in the order they are assigned to ranks."""
    out: List[Tuple[int, ...]] = [()]
    for _ in range(levels):
        out = [t + (i,) for t in out for i in range(7)]
    return out


def operand(M, idx, table, backend, stats=None):
    """S_idx(A) / T_idx(B): one combination of at most four quadrants per level
    (each level's block is freed once the next one is formed; the result stays
    held in `stats`)."""
    X = M
    for i in idx:
        Y = backend.lincomb([(c, q) for c, q in zip(table[i], quads(X)) if c])
        if stats is not None:
            stats.hold(_bytes(Y))
            if X is not M:
                stats.release(_bytes(X))
        X = Y
    return X


def targets(C, idx):
    """(block of C, coefficient) pairs product P_idx folds into."""
    out = [(C, 1)]
    for i in idx:
        out = [(quads(blk)[q], coef * C_COEF[i][q]) for blk, coef in out for q in range(4)
               if C_COEF[i][q]]
    return out


@dataclass
class PartitionStats:
    """What one rank did: the products it computed, the peak extra device bytes
    it held at once (beyond the root's caller-owned A, B, C), and its traffic."""
    products: List[int] = field(default_factory=list)
    peak_extra_bytes: int = 0
    bytes_sent: int = 0
    bytes_received: int = 0
    _live: int = 0

    def hold(self, nbytes: int, transient: int = 0):
        self._live += nbytes
        self.peak_extra_bytes = max(self.peak_extra_bytes, self._live + transient)

    def release(self, nbytes: int):
        self._live -= nbytes


def partitioned_multiply(A, B, C, alpha: int, beta: int, backend, group=None, root: int = 0,
                         levels: int = 1, window: int = 2) -> PartitionStats:
    """C <- alpha*A*B + beta*C with the 7^levels products of the top `levels`
    Winograd levels spread over the ranks of `group` (product t on rank t mod
    G).  A, B, C are only read on the root; other ranks pass None (shapes are
    broadcast)."""
    if levels < 1 or levels > MAX_LEVELS:
        raise ValueError(f"levels must be 1..{MAX_LEVELS}")
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    gr = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    stats = PartitionStats()
    meta = torch.zeros(3, dtype=torch.int64)
    if rank == root:
        meta[:] = torch.tensor([A.shape[0], A.shape[1], B.shape[1]])
    nccl = dist.get_backend(group) == "nccl"
    if nccl:
        meta = meta.cuda()
    dist.broadcast(meta, src=gr(root), group=group)
    m, k, n = (int(x) for x in meta.tolist())
    f = 2 ** levels
    if m % f or k % f or n % f:
        raise ValueError(f"{m}x{k}x{n} does not split into {f}x{f} blocks")
    dev = A.device if rank == root else (meta.device if nccl else torch.device("cpu"))

    # 1. operand sources to every rank
    if rank != root:
        A = torch.empty((m, k), dtype=torch.float64, device=dev)
        B = torch.empty((k, n), dtype=torch.float64, device=dev)
        stats.hold(_bytes(A) + _bytes(B))
        stats.bytes_received += _bytes(A) + _bytes(B)
    dist.broadcast(A, src=gr(root), group=group)
    dist.broadcast(B, src=gr(root), group=group)

    prods = product_indices(levels)
    mine = [t for t in range(len(prods)) if owner(t, world) == rank]
    stats.products = mine
    remote = [t for t in range(len(prods)) if owner(t, world) != rank] if rank == root else []
    pshape = (m // f, n // f)
    pbytes = (m // f) * (n // f) * 8

    # 2. the root: C <- beta*C once, then receives posted in product order
    posted: List[Tuple[int, torch.Tensor, object]] = []
    nxt = 0
    if rank == root:
        for blk in quads(C):
            backend.scale(blk, beta)

        def post():
            nonlocal nxt
            t = remote[nxt]
            buf = torch.empty(pshape, dtype=torch.float64, device=dev)
            stats.hold(pbytes)
            posted.append((t, buf, dist.irecv(buf, src=gr(owner(t, world)), group=group)))
            nxt += 1

        while nxt < len(remote) and len(posted) < window:
            post()

    def fold(t, P):
        for blk, coef in targets(C, prods[t]):
            backend.fold(blk, alpha * coef, P)

    # 3. local products
    sends = []
    for t in mine:
        X = operand(A, prods[t], S_COEF, backend, stats)
        Y = operand(B, prods[t], T_COEF, backend, stats)
        P, plan_peak = backend.product(X, Y)
        stats.hold(_bytes(P), transient=plan_peak)
        stats.release(_bytes(X) + _bytes(Y))
        del X, Y
        if rank == root:
            fold(t, P)
            stats.release(_bytes(P))
        else:
            sends.append((P, dist.isend(P, dst=gr(root), group=group)))
            stats.bytes_sent += _bytes(P)

    # 4. the root folds the remote products as they arrive
    while posted:
        t, buf, req = posted.pop(0)
        req.wait()
        stats.bytes_received += pbytes
        fold(t, buf)
        stats.release(pbytes)
        del buf
        if nxt < len(remote):
            post()
    for P, req in sends:
        req.wait()
    if rank != root:
        del A, B
    return stats


def local_variant(variant: str, m: int, k: int, n: int) -> str:
    """Schedule for the plain products P_t = S_t T_t on each rank.  S_t and T_t
    are freshly formed scratch copies, so the in-place schedule may overwrite
    them: `ip` on squares (zero temporaries, whatever the caller's variant),
    `iprect` for the rectangle it supports, std2 otherwise."""
    if m == k == n:
        return "ip"
    if k <= min(m, n) and m % k == 0 and n % k == 0:
        return "iprect"
    return "std2"


def makespan_bound(world: int, products: int = 7) -> float:
    """Ideal speed-up of the partition in product units."""
    per = -(-products // world)
    return products / per


def choose_levels(world: int, n: int = 1 << 30, cutoff: int = 1) -> int:
    """The fewest levels (7, 49 or 343 products) whose makespan bound is within
    2% of the best one, while each product stays above the cutoff: G = 2 -> 49
    (1.96x), G = 4 -> 343 (3.99x), G = 7 -> 7, G = 8 -> 343 (7.98x vs 7.0x)."""
    usable = [L for L in range(1, MAX_LEVELS + 1) if (n >> L) >= max(2 * cutoff, 2)] or [1]
    best = max(makespan_bound(world, 7 ** L) for L in usable)
    return next(L for L in usable if makespan_bound(world, 7 ** L) >= 0.98 * best)
