"""Calibration microbenchmarks on the B200 (design inputs, not the bench):
launch latency, per-SM / chip streaming bandwidth, leaf GEMM rates (DMMA vs
tcgen05 int8 limbs) at the leaf sizes of the BASELINE configs."""
import os; os.environ.setdefault("WM_DIAG", "1")  # the wm_diag_* probes live in the diag library  # noqa: E702,E401
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_0707_2347_b200 as W  # noqa: E402
from paper_0707_2347_b200 import _lib  # noqa: E402

L = _lib.lib()
L.wm_diag_launch_latency.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
L.wm_diag_stream.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
out = {}

for pdl in (0, 1):
    for blocks in (1, 148):
        v = C.c_double()
        L.wm_diag_launch_latency(1000, pdl, blocks, C.byref(v))
        out[f"launch_us_pdl{pdl}_blocks{blocks}"] = v.value

for blocks in (1, 8, 32, 148, 296, 592):
    for write in (0, 1):
        for size in (64 << 20, 2 << 30):
            v = C.c_double()
            L.wm_diag_stream(size, blocks, write, 5, C.byref(v))
            out[f"stream_{'copy' if write else 'read'}_{size >> 20}MB_blocks{blocks}"] = v.value

ctx = W.Context.get()
L.wm_diag_time_leaf.argtypes = [C.c_void_p, _lib.wm_dmat, _lib.wm_dmat, _lib.wm_dmat, C.c_int,
                                C.c_int, C.POINTER(C.c_double)]
for leaf in (0, 1):
    for n in (128, 256, 512, 1024, 2048, 4096):
        # distinct buffers per rep would defeat L2; report the L2-warm figure
        A, B, Cm = W.Matrix(n, n), W.Matrix(n, n), W.Matrix(n, n)
        A.fill_random(1)
        B.fill_random(2)
        torch.cuda.synchronize()
        reps = max(3, min(500, int(4e10 / (2 * n ** 3))))
        v = C.c_double()
        rc = L.wm_diag_time_leaf(ctx.h, A.view().dmat(), B.view().dmat(), Cm.view().dmat(),
                                 reps, leaf, C.byref(v))
        t = v.value * 1e-6
        out[f"leaf{'_i8' if leaf else '_dmma'}_{n}_us"] = v.value if rc == 0 else None
        out[f"leaf{'_i8' if leaf else '_dmma'}_{n}_tflops"] = 2 * n ** 3 / t / 1e12 if rc == 0 else None
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/microbench.json", "w"), indent=1)
