"""Run one leaf product size a few times (for ncu captures)."""
import os; os.environ.setdefault("WM_DIAG", "1")  # the wm_diag_* probes live in the diag library  # noqa: E702,E401
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0707_2347_b200 as W  # noqa: E402
from paper_0707_2347_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
kern = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # 1 auto, 100*bn+split forced
L = _lib.lib()
L.wm_diag_time_leaf.argtypes = [C.c_void_p, _lib.wm_dmat, _lib.wm_dmat, _lib.wm_dmat, C.c_int,
                                C.c_int, C.POINTER(C.c_double)]
ctx = W.Context.get()
A, B, Cm = W.Matrix(n, n), W.Matrix(n, n), W.Matrix(n, n)
A.fill_random(1)
B.fill_random(2)
torch.cuda.synchronize()
v = C.c_double()
rc = L.wm_diag_time_leaf(ctx.h, A.view().dmat(), B.view().dmat(), Cm.view().dmat(), 20, kern,
                         C.byref(v))
print("rc", rc, "us", v.value)
