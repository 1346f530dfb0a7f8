"""Floor of a dependent (PDL) chain of prep/comb-sized streaming kernels."""
import os; os.environ.setdefault("WM_DIAG", "1")  # the wm_diag_* probes live in the diag library  # noqa: E702,E401
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0707_2347_b200 import _lib  # noqa: E402

L = _lib.lib()
f = L.wm_diag_chain
f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
us = C.c_double()
# prep of a c=256 frame: 32768 threads x (8..12 reads of 16 B, ~7 writes of 4 B ~ 2 x 16 B)
for (threads, block, nin, nout, nbuf, tag) in [
        (32768, 128, 12, 2, 4, "prep-like L2"), (32768, 128, 12, 2, 64, "prep-like HBM"),
        (32768, 256, 12, 2, 4, "prep-like L2 b256"), (65536, 128, 6, 1, 4, "prep-like 2x threads"),
        (32768, 128, 4, 4, 4, "comb-like L2"), (32768, 128, 1, 1, 4, "1r1w L2"),
        (32768, 128, 0, 0, 4, "empty"), (4096, 128, 1, 1, 4, "tiny")]:
    rc = f(threads, block, nin, nout, 200, nbuf, C.byref(us))
    mb = threads * 16 * (nin + nout) / 1e6
    print(f"{tag:24s} rc={rc} {us.value:6.2f} us/kernel  ({mb:.1f} MB -> {mb / us.value:.0f} GB/s)")
