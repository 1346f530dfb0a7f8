"""One multiplication of a BASELINE config through the product path (for ncu
launch lists): the inputs are generated on the device, one warm-up
multiplication is captured into its graph, then ONE measured multiplication.

    python scripts/one_step.py C2
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_0707_2347_b200 as W  # noqa: E402


def main():
    import torch
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cfg = bench.CONFIGS[name]
    real = cfg["field"] == "real"
    m, k, n = cfg["m"], cfg["k"], cfg["n"]
    A, B, C = (W.Matrix(m, k, real=real), W.Matrix(k, n, real=real), W.Matrix(m, n, real=real))
    A.fill_random(cfg["seed"])
    B.fill_random(cfg["seed"] + 1)
    if cfg["beta"]:
        C.fill_random(cfg["seed"] + 2)
    for _ in range(2):
        rep = W.run_variant(cfg["variant"], A, B, C, alpha=cfg["alpha"], beta=cfg["beta"],
                            cutoff=cfg["cutoff"])
    torch.cuda.synchronize()
    print(name, "launches per multiplication", rep.n_launches)


if __name__ == "__main__":
    main()
