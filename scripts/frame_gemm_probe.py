"""Seven-product frame GEMM in isolation: tiling sweep + per-CTA phase trace."""
import os; os.environ.setdefault("WM_DIAG", "1")  # the wm_diag_* probes live in the diag library  # noqa: E702,E401
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_0707_2347_b200 as W  # noqa: E402
from paper_0707_2347_b200 import _lib  # noqa: E402

L = _lib.lib()
L.wm_diag_frame_gemm.argtypes = [C.c_void_p, C.c_uint32, C.c_int, C.c_int,
                                 C.POINTER(C.c_double), C.c_void_p, C.POINTER(C.c_int)]
ctx = W.Context.get()
out = {}
for c in (256,):
    for cfg in (0, 3201):
        us = C.c_double()
        n = C.c_int()
        rc = L.wm_diag_frame_gemm(ctx.h, c, cfg, 50, C.byref(us), None, C.byref(n))
        out[f"c{c}_cfg{cfg}"] = (round(us.value, 2), n.value) if rc == 0 else _lib.last_error()
    # trace the no-split BN32 configuration (8 chunks per CTA at c=256)
    us = C.c_double()
    n = C.c_int()
    L.wm_diag_frame_gemm(ctx.h, c, 3201, 5, C.byref(us), None, C.byref(n))
    tr = np.zeros(n.value * 16, dtype=np.uint64)
    L.wm_diag_frame_gemm(ctx.h, c, 3201, 5, C.byref(us), tr.ctypes.data, C.byref(n))
    tr = tr.reshape(n.value, 16).astype(np.int64)
    t0 = tr[:, 0].min()
    phases = {}
    names = ["start", "init", "gdc_wait", "first_chunk", "loop_end", "mma_done", "part_written",
             "cluster_sync1", "reduced", "pre_dealloc", "end", "full2", "lempty2",
             "full5", "lempty5", "mma4_issue"]
    for i, nm in enumerate(names):
        col = tr[:, i]
        col = col[col > 0]
        if len(col):
            phases[nm] = (round(float(np.median(col - t0)) / 1e3, 2), round(float(np.max(col - t0)) / 1e3, 2))
    out[f"c{c}_trace_us(median,max)"] = phases
print(json.dumps(out, indent=1))
