"""Small multiplications through every device path, for compute-sanitizer
(memcheck / racecheck / synccheck): fused frames (direct limb GEMM, folds),
unfused int8 and DMMA leaves, additions, the streamed host boundary."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0707_2347_b200 as W  # noqa: E402
from oracle import oracle as O  # noqa: E402

ctx = W.Context.get()
ctx.set_option("graphs", 0)  # plain launches: the sanitizer sees every kernel
ctx.set_option("dag", 3)     # the three concurrent issue lanes of the product path
bad = 0
for (v, n, c, acc) in [("std2", 1024, 128, False),  # config 1: 49 fused frames
                       ("std2", 512, 128, False), ("acc2", 512, 128, True), ("ip", 512, 128, False),
                       ("aclr", 512, 128, True), ("ipmm", 512, 128, False), ("acc3", 512, 128, True)]:
    for leaf in (2, 0):
        ctx.set_option("leaf_kernel", leaf)
        A, B, C = W.Matrix(n, n), W.Matrix(n, n), W.Matrix(n, n)
        A.fill_random(1)
        B.fill_random(2)
        if acc:
            C.fill_random(3)
        a0, b0, c0 = A.to_u32(), B.to_u32(), C.to_u32()
        W.run_variant(v, A, B, C, alpha=3, beta=5 if acc else 0, cutoff=c)
        ok = (C.to_u32() == O.classical_modp(a0, b0, c0 if acc else None, 3, 5 if acc else 0)).all()
        bad += not ok
        print(v, leaf, "ok" if ok else "MISMATCH", flush=True)
print("mismatches", bad)
