"""Sweep int8 leaf configurations (BN, K-split) per leaf size; graph-replayed."""
import os; os.environ.setdefault("WM_DIAG", "1")  # the wm_diag_* probes live in the diag library  # noqa: E702,E401
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0707_2347_b200 as W  # noqa: E402
from paper_0707_2347_b200 import _lib  # noqa: E402

L = _lib.lib()
L.wm_diag_time_leaf.argtypes = [C.c_void_p, _lib.wm_dmat, _lib.wm_dmat, _lib.wm_dmat, C.c_int,
                                C.c_int, C.POINTER(C.c_double)]
ctx = W.Context.get()
out = {}
for n in (128, 256, 512, 1024):
    A, B, Cm = W.Matrix(n, n), W.Matrix(n, n), W.Matrix(n, n)
    A.fill_random(1)
    B.fill_random(2)
    torch.cuda.synchronize()
    for cfg in (1, 2, 3201, 3202, 3204, 6401, 6402, 6404, 13201, 13202, 13204, 16401, 16402, 16404):
        v = C.c_double()
        rc = L.wm_diag_time_leaf(ctx.h, A.view().dmat(), B.view().dmat(), Cm.view().dmat(), 50,
                                 cfg, C.byref(v))
        out[f"{n}_{cfg}"] = round(v.value, 2) if rc == 0 else None
print(json.dumps(out, indent=1))
