"""Python mirror of the reference ``winomem`` API over the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/winomem/): ``Modulus``, ``Matrix``, ``MatView``,
``MultiplyOptions``, ``CostReport``, ``run_variant``, ``multiply``, ``ipmm``,
``ipovmm``, ``classical_mul``, ``block_addsub``, ``block_scale_copy``,
``quad_split``, ``expected_costs`` and the exception taxonomy.  A ``Matrix``
lives in HBM (a float64 CUDA tensor, torch used only as the allocator); every
operation runs through ``libwinomem_b200.so`` on the GPU.  There is no CPU
fallback: without the library or a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, Optional

import numpy as np

from . import _lib
from ._lib import wm_dmat, wm_report

kDefaultModulus = 65521


# ---- exception taxonomy (ring.hpp:23-43, workspace.hpp:20-22, schedule.hpp:30-43)
class WinomemError(RuntimeError):
    code = -1


class dimension_error(WinomemError):
    code = 1


class odd_dimension_error(dimension_error):
    code = 2


class partial_overlap_error(WinomemError):
    code = 3


class alias_error(WinomemError):
    code = 4


class shape_error(WinomemError):
    code = 5


class contract_error(WinomemError):
    code = 6


class io_error(WinomemError):
    code = 7


class workspace_error(WinomemError):
    code = 8


class unknown_schedule_error(WinomemError):
    code = 9


class parse_error(WinomemError):
    code = 10


class contract_violation_error(WinomemError):
    code = 11


class unknown_slot_error(WinomemError):
    code = 15


class cuda_error(WinomemError):
    code = 12


class nccl_error(WinomemError):
    code = 13


class invalid_argument(WinomemError):
    code = 14


_BY_CODE = {c.code: c for c in (dimension_error, odd_dimension_error, partial_overlap_error,
                                alias_error, shape_error, contract_error, io_error,
                                workspace_error, unknown_schedule_error, parse_error,
                                contract_violation_error, cuda_error, nccl_error,
                                invalid_argument, unknown_slot_error)}


def _check(rc):
    if rc != 0:
        raise _BY_CODE.get(rc, WinomemError)(_lib.last_error())


# ---- ring ------------------------------------------------------------------
class Modulus:
    """Odd prime modulus (ring.hpp:47-86).  The device path needs p < 2^16."""

    def __init__(self, p: int = kDefaultModulus):
        if p <= 2 or p >= (1 << 31) or not self.is_prime(p):
            raise dimension_error(f"modulus must be an odd prime in (2, 2^31): {p}")
        self._p = int(p)

    def p(self):
        return self._p

    def minus_one(self):
        return self._p - 1

    def __eq__(self, o):
        return isinstance(o, Modulus) and o._p == self._p

    @staticmethod
    def is_prime(n):
        if n < 2:
            return False
        if n % 2 == 0:
            return n == 2
        d = 3
        while d * d <= n:
            if n % d == 0:
                return False
            d += 2
        return True


@dataclass
class MultiplyOptions:
    """executor.hpp:22-26"""
    alpha: int = 1
    beta: int = 0
    cutoff: int = 1


@dataclass
class CostReport:
    """meter.hpp:53-75 plus the device plan figures."""
    variant: str = ""
    m: int = 0
    k: int = 0
    n: int = 0
    cutoff: int = 1
    mults: int = 0
    adds: int = 0
    peak_extra_words: int = 0
    total_alloc_words: int = 0
    word_moves: int = 0
    classical_calls: int = 0
    schedule_calls: Dict[str, int] = field(default_factory=dict)
    peak_extra_bytes: int = 0
    n_ops: int = 0
    n_launches: int = 0
    fused_frames: int = 0
    add_bytes: int = 0
    leaf_flops: int = 0
    add_bytes_issued: int = 0
    frame_gemm_bytes: int = 0
    frame_bytes: int = 0
    frame_prep_bytes: int = 0
    frame_comb_bytes: int = 0
    frame_leaf_flops: int = 0

    def ops(self):
        return self.mults + self.adds

    @staticmethod
    def csv_header():
        return "variant,m,k,n,cutoff,mults,adds,peak_extra,total_alloc"

    def csv_row(self):
        return (f"{self.variant},{self.m},{self.k},{self.n},{self.cutoff},{self.mults},"
                f"{self.adds},{self.peak_extra_words},{self.total_alloc_words}")


def last_alloc_log():
    """CostMeter::alloc_log (meter.hpp:15-19) of the last plan on this thread:
    [(words, depth, slot), ...] in acquisition order."""
    L = _lib.lib()
    need = L.wm_plan_alloc_log(None, 0)
    buf = C.create_string_buffer(need + 1)
    L.wm_plan_alloc_log(buf, need + 1)
    out = []
    for ev in buf.value.decode().split(";"):
        if ev:
            w, d, slot = ev.split(":", 2)
            out.append((int(w), int(d), slot))
    return out


def _report(variant, m, k, n, cutoff, r: wm_report) -> CostReport:
    buf = C.create_string_buffer(4096)
    _lib.lib().wm_plan_schedule_calls(buf, 4096)
    calls = {}
    for item in buf.value.decode().split(","):
        if item:
            a, b = item.split(":")
            calls[a] = int(b)
    return CostReport(variant, m, k, n, cutoff, r.mults, r.adds, r.peak_extra_words,
                      r.total_alloc_words, r.word_moves, r.classical_calls, calls,
                      r.peak_extra_bytes, r.n_ops, r.n_launches, r.fused_frames, r.add_bytes,
                      r.leaf_flops, r.add_bytes_issued, r.frame_gemm_bytes, r.frame_bytes,
                      r.frame_prep_bytes, r.frame_comb_bytes, r.frame_leaf_flops)


# ---- device context ------------------------------------------------------
class Context:
    """One C-ABI context (stream + plan cache) per (device, field, p)."""

    _cache: Dict[tuple, "Context"] = {}

    def __init__(self, device=0, p=kDefaultModulus, real=False, **options):
        import torch

        self.torch = torch
        self.device = device
        self.p = p
        self.real = real
        self.stream = torch.cuda.Stream(device=device)
        h = C.c_void_p()
        _check(_lib.lib().wm_ctx_create(device, p, 1 if real else 0,
                                        C.c_void_p(self.stream.cuda_stream), C.byref(h)))
        self.h = h
        for k_, v in options.items():
            self.set_option(k_, v)

    @classmethod
    def get(cls, device=0, p=kDefaultModulus, real=False):
        key = (device, p, real)
        if key not in cls._cache:
            cls._cache[key] = Context(device, p, real)
        return cls._cache[key]

    def set_option(self, key, value):
        _check(_lib.lib().wm_ctx_set_option(self.h, key.encode(), int(value)))

    def get_option(self, key):
        v = C.c_int64()
        _check(_lib.lib().wm_ctx_get_option(self.h, key.encode(), C.byref(v)))
        return v.value

    # stream interop with torch's current stream
    def enter(self):
        self.stream.wait_stream(self.torch.cuda.current_stream(self.device))

    def leave(self):
        self.torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def sync(self):
        _check(_lib.lib().wm_ctx_sync(self.h))

    def close(self):
        if self.h:
            _lib.lib().wm_ctx_destroy(self.h)
            self.h = None


# ---- matrices ---------------------------------------------------------------
class MatView:
    """Non-owning window {matrix, row0, col0, rows, cols} (ring.hpp:122-177)."""

    def __init__(self, mat: "Matrix", r0, c0, rows, cols):
        self.mat, self.r0, self.c0, self.rows, self.cols = mat, r0, c0, rows, cols

    @property
    def stride(self):
        return self.mat.cols()

    def window(self, r0, c0, r, c):
        if r0 + r > self.rows or c0 + c > self.cols:
            raise dimension_error("window exceeds view bounds")
        return MatView(self.mat, self.r0 + r0, self.c0 + c0, r, c)

    def dmat(self) -> wm_dmat:
        ld = self.mat.ld()
        base = self.mat.t.data_ptr() + 8 * (self.r0 * ld + self.c0)
        return wm_dmat(base, self.rows, self.cols, ld)

    def words(self):
        return self.rows * self.cols


def quad_split(v: MatView):
    """ring.hpp:222-228"""
    if v.rows % 2 or v.cols % 2:
        raise odd_dimension_error("quad_split requires even dimensions")
    r, c = v.rows // 2, v.cols // 2
    return [v.window(0, 0, r, c), v.window(0, c, r, c), v.window(r, 0, r, c),
            v.window(r, c, r, c)]


class Matrix:
    """Dense row-major matrix in HBM (float64 storage) over Z/pZ or the reals."""

    def __init__(self, rows, cols, mod: Optional[Modulus] = None, device=0, real=False):
        import torch

        if rows == 0 or cols == 0:
            raise dimension_error("matrix dimensions must be positive")
        self.mod_ = mod or Modulus(kDefaultModulus)
        self.real = real
        self.device = device
        self.t = torch.zeros((rows, cols), dtype=torch.float64, device=f"cuda:{device}")

    @classmethod
    def wrap(cls, t, mod: Optional[Modulus] = None, real=False):
        """A Matrix over an existing float64 CUDA tensor (row-major, unit column
        stride; any row stride) -- no copy."""
        if t.dtype != t.new_zeros(0, dtype=t.dtype).dtype or str(t.dtype) != "torch.float64":
            raise invalid_argument("wrap expects a float64 tensor")
        if t.dim() != 2 or t.stride(1) != 1:
            raise invalid_argument("wrap expects a 2-D tensor with unit column stride")
        m = cls.__new__(cls)
        m.mod_ = mod or Modulus(kDefaultModulus)
        m.real = real
        m.device = t.device.index or 0
        m.t = t
        return m

    def ld(self):
        return self.t.stride(0)

    def ctx(self):
        return Context.get(self.device, self.mod_.p(), self.real)

    def rows(self):
        return self.t.shape[0]

    def cols(self):
        return self.t.shape[1]

    def mod(self):
        return self.mod_

    def size(self):
        return self.t.numel()

    def view(self) -> MatView:
        return MatView(self, 0, 0, self.rows(), self.cols())

    def fill_random(self, seed):
        """Matrix::fill_random (ring.hpp:202-205), generated on the device."""
        ctx = self.ctx()
        ctx.enter()
        _check(_lib.lib().wm_fill_random(ctx.h, self.view().dmat(), seed))
        ctx.leave()

    def fill_zero(self):
        self.t.zero_()

    def to_u32(self) -> np.ndarray:
        ctx = self.ctx()
        out = np.empty((self.rows(), self.cols()), dtype=np.uint32)
        ctx.enter()
        _check(_lib.lib().wm_download_u32(ctx.h, out.ctypes.data, self.cols(), self.view().dmat()))
        return out

    def from_u32(self, arr: np.ndarray):
        arr = np.ascontiguousarray(arr, dtype=np.uint32)
        assert arr.shape == (self.rows(), self.cols())
        ctx = self.ctx()
        ctx.enter()
        _check(_lib.lib().wm_upload_u32(ctx.h, self.view().dmat(), arr.ctypes.data, self.cols()))
        ctx.sync()
        return self

    def hash(self):
        """Matrix::hash: FNV-1a over canonical u32 residues (ring.hpp:208)."""
        a = self.to_u32()
        return int(_lib.lib().wm_fnv1a64_u32(a.ctypes.data, a.size))

    def copy(self):
        m = Matrix.__new__(Matrix)
        m.mod_, m.real, m.device = self.mod_, self.real, self.device
        m.t = self.t.clone()
        return m

    def __eq__(self, o):
        return (self.rows(), self.cols()) == (o.rows(), o.cols()) and bool(
            (self.t == o.t).all().item())


def _ctx_of(*mats):
    c = mats[0].ctx()
    c.enter()
    return c


# ---- primitives (ring.hpp) -----------------------------------------------
def block_addsub(dst: MatView, a: MatView, b: MatView, sa, sb, mod: Modulus = None):
    ctx = _ctx_of(dst.mat)
    _check(_lib.lib().wm_block_addsub(ctx.h, dst.dmat(), a.dmat(), b.dmat(), sa, sb))
    ctx.leave()


def block_scale_copy(dst: MatView, src: MatView, s, mod: Modulus = None):
    ctx = _ctx_of(dst.mat)
    _check(_lib.lib().wm_block_scale_copy(ctx.h, dst.dmat(), src.dmat(), s))
    ctx.leave()


def lincomb(dst: MatView, terms, mod: Modulus = None):
    """dst <- sum coef * src over 1..4 (coef, MatView) terms in one pass
    (wm_lincomb); dst may alias a source exactly."""
    ctx = _ctx_of(dst.mat)
    n = len(terms)
    srcs = (_lib.wm_dmat * n)(*[v.dmat() for _, v in terms])
    coefs = (C.c_uint32 * n)(*[int(c) & 0xFFFFFFFF for c, _ in terms])
    _check(_lib.lib().wm_lincomb(ctx.h, dst.dmat(), n, srcs, coefs))
    ctx.leave()


def classical_mul(Cv: MatView, Av: MatView, Bv: MatView, alpha, beta, mod: Modulus = None):
    ctx = _ctx_of(Cv.mat)
    _check(_lib.lib().wm_classical_mul(ctx.h, Cv.dmat(), Av.dmat(), Bv.dmat(), alpha, beta))
    ctx.leave()


# ---- drivers ----------------------------------------------------------------
def run_variant(variant: str, A: Matrix, B: Matrix, C_: Matrix,
                opt: MultiplyOptions = None, **kw) -> CostReport:
    """run_variant (drivers.hpp:213-222) on device-resident matrices."""
    opt = opt or MultiplyOptions(**kw)
    if not (A.mod() == B.mod() and A.mod() == C_.mod()):
        raise dimension_error("operands use different moduli")
    ctx = _ctx_of(A, B, C_)
    r = wm_report()
    if A.real:
        _check(_lib.lib().wm_run_variant_real(ctx.h, variant.encode(), A.view().dmat(),
                                              B.view().dmat(), C_.view().dmat(),
                                              float(opt.alpha), float(opt.beta), opt.cutoff,
                                              C.byref(r)))
    else:
        p = A.mod().p()
        _check(_lib.lib().wm_run_variant(ctx.h, variant.encode(), A.view().dmat(),
                                         B.view().dmat(), C_.view().dmat(), opt.alpha % p,
                                         opt.beta % p, opt.cutoff, C.byref(r)))
    ctx.leave()
    return _report(variant, A.rows(), A.cols(), B.cols(), opt.cutoff, r)


# ---- matrix files (ring.hpp:386-449) -----------------------------------------
def matrix_file_info(path: str, binary=False):
    """(rows, cols, p) from a matrix file header (io_error if malformed)."""
    r, c, p = C.c_uint64(), C.c_uint64(), C.c_uint32()
    _check(_lib.lib().wm_matrix_file_info(path.encode(), 1 if binary else 0, C.byref(r),
                                          C.byref(c), C.byref(p)))
    return r.value, c.value, p.value


def read_matrix_host(path: str, binary=False):
    """read_text / read_binary into a host u32 array -> (array, p)."""
    r, c, p = matrix_file_info(path, binary)
    out = np.empty((r, c), dtype=np.uint32)
    _check(_lib.lib().wm_matrix_read_host(path.encode(), 1 if binary else 0, out.ctypes.data,
                                          out.size))
    return out, p


def write_matrix_host(path: str, a: np.ndarray, p=kDefaultModulus, binary=False):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    _check(_lib.lib().wm_matrix_write_host(path.encode(), 1 if binary else 0, a.shape[0],
                                           a.shape[1], p, a.ctypes.data))


def read_text(path: str, device=0, binary=False) -> "Matrix":
    """read_text (ring.hpp:401-412): a device Matrix straight from the file."""
    r, c, p = matrix_file_info(path, binary)
    M = Matrix(r, c, Modulus(p), device=device)
    ctx = M.ctx()
    ctx.enter()
    _check(_lib.lib().wm_matrix_read_device(ctx.h, path.encode(), 1 if binary else 0,
                                            M.view().dmat()))
    return M


def read_binary(path: str, device=0) -> "Matrix":
    """read_binary (ring.hpp:436-446)."""
    return read_text(path, device, binary=True)


def write_text(M: "Matrix", path: str, binary=False):
    """write_text (ring.hpp:390-399) from a device Matrix."""
    ctx = M.ctx()
    ctx.enter()
    _check(_lib.lib().wm_matrix_write_device(ctx.h, path.encode(), 1 if binary else 0,
                                             M.view().dmat()))


def write_binary(M: "Matrix", path: str):
    """write_binary (ring.hpp:428-434)."""
    write_text(M, path, binary=True)


def parse_schedule(text: str):
    """parse_schedule (schedule.hpp:679-684): validate DSL text; returns
    (canonical rendering, equals-the-builtin-of-that-name).  Raises parse_error /
    contract_violation_error like the reference."""
    L = _lib.lib()
    need, match = C.c_int(), C.c_int()
    _check(L.wm_parse_schedule(text.encode(), None, 0, C.byref(need), C.byref(match)))
    buf = C.create_string_buffer(need.value + 1)
    _check(L.wm_parse_schedule(text.encode(), buf, need.value + 1, C.byref(need), C.byref(match)))
    return buf.value.decode(), bool(match.value)


def plan_report_parsed(text: str, m, k, n, cutoff=1, alpha=1, beta=0,
                       p=kDefaultModulus) -> CostReport:
    """Host-only: the CostReport run_parsed_schedule would produce."""
    r = wm_report()
    _check(_lib.lib().wm_plan_report_parsed(text.encode(), p, m, k, n, alpha % p, beta % p,
                                            cutoff, C.byref(r)))
    return _report("parsed", m, k, n, cutoff, r)


def render_schedule(name: str) -> str:
    """render_schedule (schedule.hpp:617-684) of a builtin schedule."""
    L = _lib.lib()
    need = C.c_int()
    _check(L.wm_render_schedule(name.encode(), None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value + 1)
    _check(L.wm_render_schedule(name.encode(), buf, need.value + 1, C.byref(need)))
    return buf.value.decode()


def run_parsed_schedule(text: str, A: Matrix, B: Matrix, C_: Matrix,
                        opt: MultiplyOptions = None, **kw) -> CostReport:
    """run_parsed_schedule (executor.hpp:304-342): the DSL schedule runs at the
    top frame on the device; its recursion tags dispatch to the builtins."""
    opt = opt or MultiplyOptions(**kw)
    if A.real:
        raise invalid_argument("parsed schedules run over Z/pZ")
    ctx = _ctx_of(A, B, C_)
    p = A.mod().p()
    r = wm_report()
    _check(_lib.lib().wm_run_parsed_schedule(ctx.h, text.encode(), A.view().dmat(),
                                             B.view().dmat(), C_.view().dmat(), opt.alpha % p,
                                             opt.beta % p, opt.cutoff, C.byref(r)))
    ctx.leave()
    return _report("parsed", A.rows(), A.cols(), B.cols(), opt.cutoff, r)


def multiply(variant, A, B, C_, opt: MultiplyOptions = None, **kw) -> CostReport:
    """multiply (executor.hpp:240-299)."""
    return run_variant(variant, A, B, C_, opt, **kw)


def ipmm(A, B, C_, cutoff=1) -> CostReport:
    """ipmm (drivers.hpp:137-158)."""
    return run_variant("ipmm", A, B, C_, MultiplyOptions(1, 0, cutoff))


def ipovmm(A, B, C_, cutoff=1) -> CostReport:
    """ipovmm (drivers.hpp:52-99)."""
    return run_variant("ipovmm", A, B, C_, MultiplyOptions(1, 0, cutoff))


def run_variant_host(variant, A: np.ndarray, B: np.ndarray, C_: np.ndarray, alpha=1, beta=0,
                     cutoff=1, p=kDefaultModulus, device=0) -> CostReport:
    """End-to-end over host u32 residues (the reference's Matrix& semantics):
    C_ (and A / B when the contract allows overwriting) are updated in place."""
    for a in (A, B, C_):
        if a.dtype != np.uint32 or not a.flags["C_CONTIGUOUS"]:
            raise invalid_argument("host matrices must be C-contiguous uint32")
    m, k = A.shape
    n = B.shape[1]
    ctx = Context.get(device, p, False)
    ctx.enter()
    r = wm_report()
    _check(_lib.lib().wm_run_variant_host_u32(ctx.h, variant.encode(), m, k, n, A.ctypes.data,
                                              B.ctypes.data, C_.ctypes.data, alpha % p,
                                              beta % p, cutoff, C.byref(r)))
    return _report(variant, m, k, n, cutoff, r)


def plan_report(variant, m, k, n, cutoff=1, alpha=1, beta=0, p=kDefaultModulus, real=False,
                fuse_frames=False) -> CostReport:
    """Host-only: the exact CostReport and plan size, without executing."""
    r = wm_report()
    _check(_lib.lib().wm_plan_report(variant.encode(), 1 if real else 0, p, m, k, n, alpha,
                                     beta, cutoff, 1 if fuse_frames else 0, C.byref(r)))
    return _report(variant, m, k, n, cutoff, r)


def expected_costs(variant, m, k, n, cutoff) -> CostReport:
    """models::expected_costs (models.hpp:202-229)."""
    r = wm_report()
    _check(_lib.lib().wm_expected_costs(variant.encode(), m, k, n, cutoff, C.byref(r)))
    return CostReport(variant, m, k, n, cutoff, r.mults, r.adds, r.peak_extra_words,
                      r.total_alloc_words, r.word_moves)


def compare(measured: CostReport, expected: CostReport):
    """meter.hpp:91-105: field-by-field differences."""
    diffs = []
    for f in ("mults", "adds", "peak_extra_words", "total_alloc_words"):
        a, b = getattr(measured, f), getattr(expected, f)
        if a != b:
            diffs.append(f"{f}: measured={a} expected={b}")
    return diffs


BUILTIN_NAMES = ["std2", "acc3", "ip", "ovl", "ovl2", "ovr", "aclr", "accr", "acc2", "acr"]
_ACC = {"acc3", "aclr", "accr", "acc2", "acr"}


def variant_accumulates(v):
    if v in ("ipmm", "ipovmm", "iprect", "classic"):
        return False
    if v.startswith("blocked_acc_t"):
        return True
    if v not in BUILTIN_NAMES:
        raise unknown_schedule_error("unknown schedule: " + v)
    return v in _ACC


# ---- multi-GPU product partition through the C-ABI (wm_dist_*) ----------------
class DistContext:
    """wm_dist_create / wm_dist_run_variant: the native multi-GPU product
    partition (csrc/wm_dist.cpp) over an NCCL communicator of `world` ranks,
    one per process (or thread) and GPU.  Rank 0 makes the 128-byte NCCL id
    with ``DistContext.unique_id()`` and ships it to the others."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        rc = _lib.lib().wm_dist_unique_id(buf)
        if rc:
            raise _BY_CODE.get(rc, WinomemError)(_lib.lib().wm_dist_last_error().decode())
        return buf.raw

    def __init__(self, rank, world, uid: bytes, device=0, p=kDefaultModulus, real=False):
        self.ctx = Context.get(device, p, real)
        self.h = C.c_void_p()
        rc = _lib.lib().wm_dist_create(self.ctx.h, rank, world, uid, C.byref(self.h))
        if rc:
            raise _BY_CODE.get(rc, WinomemError)(_lib.lib().wm_dist_last_error().decode())
        self.rank, self.world = rank, world

    def run_variant(self, variant, A=None, B=None, C_=None, alpha=1, beta=0, cutoff=1, levels=0,
                    window=2) -> dict:
        empty = wm_dmat(None, 0, 0, 0)
        dm = lambda M: M.view().dmat() if M is not None else empty  # noqa: E731
        r = _lib.wm_dist_report()
        self.ctx.enter()
        rc = _lib.lib().wm_dist_run_variant(self.h, variant.encode(), dm(A), dm(B), dm(C_), alpha,
                                            beta, cutoff, levels, window, C.byref(r))
        self.ctx.leave()
        if rc:
            raise _BY_CODE.get(rc, WinomemError)(_lib.lib().wm_dist_last_error().decode())
        return dict(levels=r.levels, products=r.products, peak_extra_bytes=r.peak_extra_bytes,
                    bytes_sent=r.bytes_sent, bytes_received=r.bytes_received)

    def close(self):
        if self.h:
            _lib.lib().wm_dist_destroy(self.h)
            self.h = None
