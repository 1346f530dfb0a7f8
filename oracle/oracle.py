"""TEST INFRASTRUCTURE ONLY -- the CPU oracle (checker), never the product.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It loads

* ``oracle/build/liboracle.so``  -- the plain-C restatement (wm_oracle.c) of the
  reference ring layer (ring.hpp:93-114, 241-278, 315-384);
* ``oracle/_ref/libwinomem_ref.so`` -- the UNMODIFIED reference headers behind a
  C shim (ref_shim.cpp), used to pin the restatement and as the CPU baseline.

Both are built by ``make -C oracle`` (``__graft_entry__.build()`` runs it).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

u64 = C.c_uint64
u32 = C.c_uint32
P_u32 = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
P_f64 = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
P_u64 = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")

DEFAULT_P = 65521


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "build", "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.wmo_splitmix_fill.argtypes = [P_u32, u64, u64, u32]
        L.wmo_splitmix_raw.argtypes = [P_u64, u64, u64]
        L.wmo_real_fill.argtypes = [P_f64, u64, u64]
        L.wmo_fnv1a64.argtypes = [P_u32, u64]
        L.wmo_fnv1a64.restype = u64
        L.wmo_block_addsub.argtypes = [u64, u64, u32, P_u32, u64, P_u32, u64, P_u32, u64, u32, u32]
        L.wmo_classical_modp.argtypes = [u64, u64, u64, P_u32, u64, P_u32, u64, P_u32, u64,
                                         u32, u32, u32, C.c_int]
        L.wmo_classical_f64.argtypes = [u64, u64, u64, P_f64, u64, P_f64, u64, P_f64, u64,
                                        C.c_double, C.c_double, C.c_int]
        L.wmo_winograd_f64.argtypes = [u64, P_f64, u64, P_f64, u64, P_f64, u64, u64]
        _LIB = L
    return _LIB


def ref_available():
    return os.path.exists(os.path.join(HERE, "_ref", "libwinomem_ref.so"))


def ref():
    """The reference implementation itself (compiled from its own headers)."""
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "libwinomem_ref.so")
        if not os.path.exists(path):
            build()
        R = C.CDLL(path)
        R.ref_run_variant.argtypes = [C.c_char_p, u64, u64, u64, u32, P_u32, P_u32, P_u32,
                                      u32, u32, C.c_int, P_u64, C.c_char_p, C.c_int,
                                      C.c_char_p, C.c_int]
        R.ref_expected_costs.argtypes = [C.c_char_p, u64, u64, u64, C.c_int, P_u64,
                                         C.c_char_p, C.c_int]
        R.ref_classical_mul.argtypes = [u64, u64, u64, u32, P_u32, P_u32, P_u32, u32, u32]
        R.ref_block_addsub.argtypes = [u64, u64, u32, P_u32, P_u32, P_u32, u32, u32]
        R.ref_fill_random.argtypes = [P_u32, u64, u64, u32]
        R.ref_hash.argtypes = [P_u32, u64]
        R.ref_hash.restype = u64
        R.ref_render_builtin.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        R.ref_run_parsed.argtypes = [C.c_char_p, u64, u64, u64, u32, P_u32, P_u32, P_u32, u32,
                                     u32, C.c_int, P_u64, C.c_char_p, C.c_int]
        R.ref_write_matrix.argtypes = [C.c_char_p, C.c_int, u64, u64, u32, C.c_void_p]
        R.ref_read_matrix.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.c_void_p,
                                      u64]
        _REF = R
    return _REF


# --------------------------------------------------------------- helpers

def fill_random(rows, cols, seed, p=DEFAULT_P):
    out = np.empty(rows * cols, dtype=np.uint32)
    lib().wmo_splitmix_fill(out, out.size, seed, p)
    return out.reshape(rows, cols)


def real_fill(rows, cols, seed):
    out = np.empty(rows * cols, dtype=np.float64)
    lib().wmo_real_fill(out, out.size, seed)
    return out.reshape(rows, cols)


def fnv1a64(a):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return int(lib().wmo_fnv1a64(a.reshape(-1), a.size))


def classical_modp(A, B, C0=None, alpha=1, beta=0, p=DEFAULT_P, threads=None):
    A = np.ascontiguousarray(A, dtype=np.uint32)
    B = np.ascontiguousarray(B, dtype=np.uint32)
    m, k = A.shape
    k2, n = B.shape
    assert k == k2
    Cm = np.zeros((m, n), dtype=np.uint32) if C0 is None else np.array(C0, dtype=np.uint32, order="C")
    threads = threads or min(os.cpu_count() or 1, 64)
    lib().wmo_classical_modp(m, k, n, A.reshape(-1), k, B.reshape(-1), n, Cm.reshape(-1), n,
                             alpha % p, beta % p, p, threads)
    return Cm


def classical_f64(A, B, C0=None, alpha=1.0, beta=0.0, threads=None):
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    m, k = A.shape
    _, n = B.shape
    Cm = np.zeros((m, n)) if C0 is None else np.array(C0, dtype=np.float64, order="C")
    threads = threads or min(os.cpu_count() or 1, 64)
    lib().wmo_classical_f64(m, k, n, A.reshape(-1), k, B.reshape(-1), n, Cm.reshape(-1), n,
                            float(alpha), float(beta), threads)
    return Cm


def winograd_f64(A, B, cutoff):
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    n = A.shape[0]
    Cm = np.zeros((n, n))
    lib().wmo_winograd_f64(n, A.reshape(-1), n, B.reshape(-1), n, Cm.reshape(-1), n, cutoff)
    return Cm


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def ref_run_variant(variant, A, B, C0, alpha=1, beta=0, cutoff=1, p=DEFAULT_P):
    """Run the reference's own run_variant on copies; returns (A, B, C, report, sched)."""
    A = np.array(A, dtype=np.uint32, order="C")
    B = np.array(B, dtype=np.uint32, order="C")
    Cm = np.array(C0, dtype=np.uint32, order="C")
    m, k = A.shape
    n = B.shape[1]
    rep = np.zeros(6, dtype=np.uint64)
    sched = C.create_string_buffer(4096)
    err = C.create_string_buffer(512)
    rc = ref().ref_run_variant(variant.encode(), m, k, n, p, A.reshape(-1), B.reshape(-1),
                               Cm.reshape(-1), alpha, beta, cutoff, rep, sched, 4096, err, 512)
    if rc:
        raise RefError(rc, err.value.decode())
    report = dict(zip(["mults", "adds", "peak_extra_words", "total_alloc_words", "word_moves",
                       "classical_calls"], [int(x) for x in rep]))
    calls = {}
    for item in sched.value.decode().split(","):
        if item:
            name, cnt = item.split(":")
            calls[name] = int(cnt)
    return A, B, Cm, report, calls


def ref_primitive_on_windows(op, buf, wins, s0, s1=0, p=DEFAULT_P):
    """One reference primitive (0 block_addsub, 1 block_scale_copy, 2 classical_mul)
    on windows {r0, c0, rows, cols} of ONE buffer; returns (code, buffer after)."""
    L = ref()
    f = L.ref_primitive_on_windows
    f.argtypes = [C.c_int, u64, u64, u32, P_u32, P_u64, u32, u32, C.c_char_p, C.c_int]
    f.restype = C.c_int
    out = np.array(buf, dtype=np.uint32, order="C")
    w = np.zeros(12, dtype=np.uint64)
    for i, win in enumerate(wins):
        w[4 * i:4 * i + 4] = win
    err = C.create_string_buffer(512)
    rc = f(op, out.shape[0], out.shape[1], p, out.reshape(-1), w, s0, s1, err, 512)
    return rc, out


def ref_alloc_log(variant, m, k, n, alpha=1, beta=0, cutoff=1):
    """The reference CostMeter's alloc_log of run_variant, as "words:depth:slot;..."."""
    L = ref()
    f = L.ref_alloc_log
    f.argtypes = [C.c_char_p, u64, u64, u64, u32, u32, C.c_int, C.c_char_p, C.c_int]
    f.restype = C.c_int
    buf = C.create_string_buffer(1 << 22)
    rc = f(variant.encode(), m, k, n, alpha, beta, cutoff, buf, 1 << 22)
    if rc < 0:
        raise RefError(-rc, "reference raised")
    return buf.value.decode()


def ref_expected_costs(variant, m, k, n, cutoff):
    rep = np.zeros(6, dtype=np.uint64)
    err = C.create_string_buffer(512)
    rc = ref().ref_expected_costs(variant.encode(), m, k, n, cutoff, rep, err, 512)
    if rc:
        raise RefError(rc, err.value.decode())
    return dict(zip(["mults", "adds", "peak_extra_words", "total_alloc_words", "word_moves"],
                    [int(x) for x in rep[:5]]))


def ref_render_builtin(name):
    buf = C.create_string_buffer(1 << 16)
    n = ref().ref_render_builtin(name.encode(), buf, 1 << 16)
    if n < 0:
        raise RefError(-n, name)
    return buf.value.decode()


def ref_write_matrix(path, a, p=DEFAULT_P, binary=False):
    """The reference's write_text / write_binary (ring.hpp:390-434)."""
    a = np.ascontiguousarray(a, dtype=np.uint32)
    rc = ref().ref_write_matrix(path.encode(), 1 if binary else 0, a.shape[0], a.shape[1], p,
                                a.ctypes.data)
    if rc < 0:
        raise RefError(-rc, path)


def ref_read_matrix(path, binary=False):
    """The reference's read_text / read_binary (ring.hpp:401-446) -> (array, p);
    raises RefError(code) on a reference exception."""
    r, c, p = C.c_uint64(), C.c_uint64(), C.c_uint32()
    rc = ref().ref_read_matrix(path.encode(), 1 if binary else 0, C.byref(r), C.byref(c),
                               C.byref(p), None, 0)
    if rc < 0:
        raise RefError(-rc, path)
    out = np.zeros((r.value, c.value), dtype=np.uint32)
    ref().ref_read_matrix(path.encode(), 1 if binary else 0, C.byref(r), C.byref(c), C.byref(p),
                          out.ctypes.data, out.size)
    return out, p.value


def ref_run_parsed(text, A, B, C0, alpha=1, beta=0, cutoff=1, p=DEFAULT_P):
    """The reference's parse_schedule + run_parsed_schedule -> (C, A, B, report)."""
    A = np.ascontiguousarray(A, dtype=np.uint32).copy()
    B = np.ascontiguousarray(B, dtype=np.uint32).copy()
    Cm = np.ascontiguousarray(C0, dtype=np.uint32).copy()
    rep = np.zeros(8, dtype=np.uint64)
    err = C.create_string_buffer(512)
    rc = ref().ref_run_parsed(text.encode(), A.shape[0], A.shape[1], B.shape[1], p, A.reshape(-1),
                              B.reshape(-1), Cm.reshape(-1), alpha, beta, cutoff, rep, err, 512)
    if rc:
        raise RefError(rc, err.value.decode())
    return Cm, A, B, dict(zip(["mults", "adds", "peak_extra_words", "total_alloc_words",
                               "word_moves"], [int(x) for x in rep[:5]]))
