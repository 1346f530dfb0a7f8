"""Direct-limb frame GEMM: correctness (host check) and timing per shape."""
import os; os.environ.setdefault("WM_DIAG", "1")  # the wm_diag_* probes live in the diag library  # noqa: E702,E401
import ctypes as C
import json

import numpy as np
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_0707_2347_b200 import winomem as W  # noqa: E402
from paper_0707_2347_b200._lib import lib  # noqa: E402

L = lib()
L.wm_diag_direct_check.argtypes = [C.c_void_p, C.c_uint32, C.c_int, C.c_int, C.c_uint64,
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.c_void_p]
L.wm_diag_direct_check.restype = C.c_int
ctx = W.Context(p=65521)
res = {}
for c in (128, 256, 512):
    for bn in (32, 64, 128):
        for bconv in (0, 1):
            bad = C.c_uint64()
            us = C.c_double()
            tr = np.zeros((c // 128) * 7 * (c // (bn % 1000)) * 16, dtype=np.uint64)
            rc = L.wm_diag_direct_check(ctx.h, c, bn, bconv, 7 + c, C.byref(bad), C.byref(us),
                                        tr.ctypes.data)
            key = f"c{c}_bn{bn}_bconv{bconv}"
            res[key] = {"rc": rc, "mismatches": bad.value, "us": round(us.value, 2)}
            if rc:
                res[key]["err"] = L.wm_last_error().decode() if hasattr(L, "wm_last_error") else ""
            t = tr.reshape(-1, 16).astype(np.int64)
            t0 = t[:, 0].min()
            names = ["start", "init", "gdc", "full0", "full_last", "done", "stored", "end"]
            res[key]["trace_med"] = {nm: round(float(np.median(t[:, i] - t0)) / 1000, 2)
                                     for i, nm in enumerate(names)}
            res[key]["trace_max"] = round(float((t[:, 7] - t0).max()) / 1000, 2)
            print(key, res[key], flush=True)
print(json.dumps(res))
