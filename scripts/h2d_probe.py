"""Pinned host -> device copy rate: contiguous vs quadrant 2-D copies."""
import os; os.environ.setdefault("WM_DIAG", "1")  # the wm_diag_* probes live in the diag library  # noqa: E702,E401
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0707_2347_b200._lib import lib  # noqa: E402

L = lib()
L.wm_diag_h2d.argtypes = [C.c_void_p, C.c_ulonglong, C.c_ulonglong, C.c_int, C.c_int,
                          C.POINTER(C.c_double)]
h = torch.zeros((4096, 4096), dtype=torch.int32).pin_memory()
for mode, name in [(0, "contiguous"), (1, "4 quadrants 2-D"), (2, "2 row halves")]:
    g = C.c_double()
    rc = L.wm_diag_h2d(h.data_ptr(), 4096, 4096, mode, 10, C.byref(g))
    print(f"{name:18s} {g.value:7.1f} GB/s rc {rc}", flush=True)
