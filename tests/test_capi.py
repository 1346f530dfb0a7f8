"""The C-ABI library loads and exports every entry point include/*.h declares.
CPU only: no compute calls, only host-side planning entries."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("winomem_b200.h",):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(wm_[a-z0-9_]+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    from paper_0707_2347_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    decl = _declared()
    assert len(decl) >= 20
    missing = [n for n in sorted(decl) if not hasattr(L, n)]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= decl


def test_version_and_error_without_gpu():
    from paper_0707_2347_b200 import _lib
    L = _lib.lib()
    assert b"sm_100a" in L.wm_version()
    h = ctypes.c_void_p()
    rc = L.wm_ctx_create(0, 65521, 0, None, ctypes.byref(h))
    import torch
    if not torch.cuda.is_available():
        assert rc == 12 and b"no CUDA device" in L.wm_last_error()
    else:
        assert rc == 0
        L.wm_ctx_destroy(h)


def test_modulus_checks():
    from paper_0707_2347_b200 import Modulus, dimension_error
    import pytest
    Modulus(65521)
    Modulus(3)
    for bad in (1, 2, 4, 65520):
        with pytest.raises(dimension_error):
            Modulus(bad)


def test_cpp_dropin_header_compiles():
    """include/winomem_b200.hpp (the C++ drop-in over the C-ABI) compiles and
    links against the library on the host."""
    import subprocess
    import tempfile
    hpp = os.path.join(ROOT, "include", "winomem_b200.hpp")
    if not os.path.exists(hpp):
        return
    src = os.path.join(ROOT, "tests", "cpp", "dropin_smoke.cpp")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "dropin")
        r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src,
                            "-o", exe, os.path.join(ROOT, "paper_0707_2347_b200",
                                                    "libwinomem_b200.so"),
                            "-Wl,-rpath," + os.path.join(ROOT, "paper_0707_2347_b200")],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        r = subprocess.run([exe, "--plan-only"], capture_output=True, text=True, timeout=60)
        assert r.returncode == 0, r.stdout + r.stderr


def test_product_library_has_no_probes():
    """The measurement probes (wm_diag_*) live in libwinomem_b200_diag.so only."""
    from paper_0707_2347_b200 import _lib
    L = ctypes.CDLL(_lib.PRODUCT_LIB)
    for name in ("wm_diag_trace", "wm_diag_plan_dag", "wm_diag_direct_check", "wm_diag_chain",
                 "wm_diag_time_leaf", "wm_diag_frame_gemm"):
        assert not hasattr(L, name), name
    D = ctypes.CDLL(_lib.DIAG_LIB)
    assert hasattr(D, "wm_diag_direct_check") and hasattr(D, "wm_run_variant")
