"""The leaf rule of leaf_kernel = 2 (tcgen05 int8 limbs where the tiles fit, FP64
DMMA otherwise), measured: graph-replayed time of one mod-p leaf product per
size on both kernels.  Run under `ncu --set full -k regex:k_leaf_dmma|k_gemm_tma`
for the tensor-pipe utilisation of the same launches.

    python scripts/leaf_choice.py [reps]
"""
import os; os.environ.setdefault("WM_DIAG", "1")  # noqa: E702,E401
import ctypes as C
import json
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0707_2347_b200 as W  # noqa: E402
from paper_0707_2347_b200 import _lib  # noqa: E402

L = _lib.lib()
L.wm_diag_time_leaf.argtypes = [C.c_void_p, _lib.wm_dmat, _lib.wm_dmat, _lib.wm_dmat, C.c_int,
                                C.c_int, C.POINTER(C.c_double)]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
ctx = W.Context.get()
out = {}
for n in (128, 256, 512, 1024, 2048):
    A, B, Cm = W.Matrix(n, n), W.Matrix(n, n), W.Matrix(n, n)
    A.fill_random(1)
    B.fill_random(2)
    torch.cuda.synchronize()
    row = {}
    for name, kern in (("dmma_us", 0), ("int8_us", 2)):
        v = C.c_double()
        rc = L.wm_diag_time_leaf(ctx.h, A.view().dmat(), B.view().dmat(), Cm.view().dmat(), reps,
                                 kern, C.byref(v))
        row[name] = round(v.value, 2) if rc == 0 else None
    if row["dmma_us"] and row["int8_us"]:
        row["int8_speedup"] = round(row["dmma_us"] / row["int8_us"], 2)
        row["dmma_tflops"] = round(2 * n ** 3 / row["dmma_us"] / 1e6, 2)
        row["int8_eff_tflops"] = round(2 * n ** 3 / row["int8_us"] / 1e6, 2)
    out[str(n)] = row
    print(n, row, flush=True)
print(json.dumps(out))
