"""Measure the tensor-pipe denominators MEASURED_PEAKS.json lacks:
cuBLAS float64 GEMM (DMMA) and cuBLASLt int8 GEMM (torch._int_mm), burst (best
of 10) and sustained (back to back for ~3 s), CUDA events, with the SM clock
and throttle reasons sampled through NVML while each measurement runs
(B200_PROFILING.md clocks line).  Writes profiles/r2/tensor_peaks.json."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import Clocks  # noqa: E402


def measure(fn, flops, reps=10, sustain_s=3.0):
    fn()
    torch.cuda.synchronize()
    with Clocks(torch.cuda.current_device()) as clk:
        best = 0.0
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = max(best, flops / (e0.elapsed_time(e1) / 1e3))
        # sustained: enough back-to-back launches for ~sustain_s
        iters = max(10, int(sustain_s * best / flops))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        sus = iters * flops / (e0.elapsed_time(e1) / 1e3)
    return best, sus, clk.summary()


def main():
    out = {"gpu": torch.cuda.get_device_name(),
           "how": "torch.matmul float64 (cuBLAS DGEMM) and torch._int_mm int8 (cuBLASLt) on "
                  "N^3, 2*N^3 ops; burst = best of 10, sustained = back to back ~3 s; "
                  "CUDA events; clocks sampled by NVML during each measurement"}
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    bst, sus, clk = measure(lambda: a @ b, 2.0 * n ** 3)
    out["fp64_tflops"], out["fp64_tflops_sustained"], out["fp64_clocks"] = bst / 1e12, sus / 1e12, clk
    del a, b
    for n in (8192, 16384):
        ai = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
        bi = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
        bst, sus, clk = measure(lambda: torch._int_mm(ai, bi), 2.0 * n ** 3)
        out[f"int8_tops_{n}"], out[f"int8_tops_sustained_{n}"] = bst / 1e12, sus / 1e12
        out[f"int8_clocks_{n}"] = clk
        del ai, bi
    out["int8_tops"] = max(out["int8_tops_8192"], out["int8_tops_16384"])
    out["int8_tops_sustained"] = max(out["int8_tops_sustained_8192"], out["int8_tops_sustained_16384"])
    os.makedirs(os.path.join(ROOT, "profiles", "r2"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", "r2", "tensor_peaks.json"), "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
