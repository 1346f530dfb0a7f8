"""Measure the tensor-pipe denominators MEASURED_PEAKS.json lacks:
cuBLAS float64 GEMM (DMMA) and cuBLASLt int8 GEMM (torch._int_mm), burst, best
of 10 with CUDA events.  Writes profiles/r1/tensor_peaks.json."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def best(fn, flops, reps=10):
    fn()
    torch.cuda.synchronize()
    out = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out = max(out, flops / (e0.elapsed_time(e1) / 1e3))
    return out


n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
f64 = best(lambda: a @ b, 2.0 * n ** 3)
ai = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
bi = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
i8 = best(lambda: torch._int_mm(ai, bi), 2.0 * n ** 3)
res = {"fp64_tflops": f64 / 1e12, "int8_tops": i8 / 1e12,
       "how": "torch.matmul float64 8192^3 (cuBLAS DGEMM) and torch._int_mm int8 8192^3 "
              "(cuBLASLt), 2*N^3 ops, best of 10, CUDA events",
       "gpu": torch.cuda.get_device_name()}
os.makedirs(os.path.join(ROOT, "profiles", "r1"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "profiles", "r1", "tensor_peaks.json"), "w"), indent=1)
print(json.dumps(res))
