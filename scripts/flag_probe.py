"""Dependent-launch floor: griddepcontrol.wait (PDL) vs a counter handoff."""
import os; os.environ.setdefault("WM_DIAG", "1")  # the wm_diag_* probes live in the diag library  # noqa: E702,E401
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0707_2347_b200._lib import lib  # noqa: E402

L = lib()
for f in (L.wm_diag_chain, L.wm_diag_chain_flag):
    f.argtypes = [C.c_int] * 6 + [C.POINTER(C.c_double)]
for (threads, nin, nout, nbuf, what) in [(256, 0, 0, 1, "empty 1 CTA"), (32768, 1, 1, 1, "1 MB r+w"),
                                        (131072, 2, 2, 2, "8 MB r+w (L2)"),
                                        (262144, 4, 4, 8, "32 MB r+w (HBM)")]:
    a, b = C.c_double(), C.c_double()
    ra = L.wm_diag_chain(threads, 256, nin, nout, 400, nbuf, C.byref(a))
    rb = L.wm_diag_chain_flag(threads, 256, nin, nout, 400, nbuf, C.byref(b))
    print(f"{what:20s} pdl {a.value:6.2f} us  flag {b.value:6.2f} us  rc {ra} {rb}", flush=True)
