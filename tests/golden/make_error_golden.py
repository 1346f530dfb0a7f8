"""Generate tests/golden/error_cases.json from the REFERENCE implementation.

TEST INFRASTRUCTURE.  Illegal calls and their exception class (as the WM_E_*
status code of include/winomem_b200.h), as the unmodified reference
(oracle/_ref) raises them:
  * run_variant on shapes a schedule rejects, beta on a plain product, unknown
    variants, drivers outside their shape domain (drivers.hpp, executor.hpp);
  * the primitives on windows of ONE buffer -- partial overlap, exact aliasing
    (legal for block_addsub, illegal for classical_mul), dimension mismatch
    (ring.hpp:241-384); the legal ones record the buffer hash afterwards.
The GPU suite replays every case through the C-ABI (tests/test_gpu_parity.py).

    python tests/golden/make_error_golden.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from oracle import oracle as O  # noqa: E402

ACC = {"acc3", "aclr", "accr", "acc2", "acr"}

VARIANT_CASES = [
    # (variant, m, k, n, cutoff, alpha, beta)
    ("ip", 8, 4, 8, 1, 1, 0), ("ovl", 16, 8, 16, 1, 1, 0), ("ovr", 8, 16, 8, 2, 1, 0),
    ("aclr", 8, 16, 8, 1, 1, 1), ("accr", 16, 8, 8, 1, 1, 1), ("acc2", 4, 8, 4, 1, 1, 1),
    ("ovl2", 8, 8, 16, 1, 1, 0),
    ("std2", 8, 8, 8, 1, 1, 5), ("ip", 8, 8, 8, 1, 1, 3), ("ovl", 16, 16, 16, 2, 3, 1),
    ("nope", 8, 8, 8, 1, 1, 0), ("Std2", 8, 8, 8, 1, 1, 0), ("blocked_acc_tx", 8, 8, 8, 1, 1, 1),
    ("ipovmm", 8, 8, 8, 1, 1, 0), ("ipovmm", 4, 8, 8, 1, 1, 0),
    ("std2", 8, 8, 8, 0, 1, 0), ("acc3", 8, 8, 8, -1, 1, 1),
    # legal neighbours, for contrast (no error expected)
    ("std2", 8, 4, 8, 1, 1, 0), ("acc3", 8, 16, 4, 1, 1, 1), ("ipovmm", 16, 8, 4, 1, 1, 0),
]

# (op, rows, cols, [dst, a, b windows], s0, s1)
PRIMITIVE_CASES = [
    (0, 4, 4, [(1, 1, 2, 2), (0, 0, 2, 2), (2, 2, 2, 2)], 1, 1),   # dst partially overlaps a
    (0, 4, 4, [(0, 0, 2, 2), (2, 2, 2, 2), (1, 1, 2, 2)], 1, 1),   # dst partially overlaps b
    (0, 4, 4, [(0, 0, 2, 2), (0, 0, 2, 2), (2, 2, 2, 2)], 1, 1),   # dst == a: legal
    (0, 4, 4, [(2, 2, 2, 2), (0, 0, 2, 2), (2, 2, 2, 2)], 3, 7),   # dst == b: legal
    (0, 4, 4, [(0, 0, 2, 2), (0, 0, 2, 1), (2, 2, 2, 2)], 1, 1),   # dimension mismatch
    (0, 8, 8, [(0, 0, 4, 4), (4, 4, 4, 4), (0, 4, 4, 4)], 65520, 65520),
    (1, 4, 4, [(1, 0, 2, 2), (0, 0, 2, 2)], 5, 0),                 # scale_copy partial overlap
    (1, 4, 4, [(0, 0, 2, 2), (0, 0, 2, 2)], 5, 0),                 # in place: legal
    (1, 4, 4, [(0, 0, 2, 2), (2, 2, 2, 2)], 65520, 0),
    (1, 4, 4, [(0, 0, 2, 2), (2, 2, 1, 2)], 1, 0),                 # dimension mismatch
    (2, 4, 4, [(0, 0, 2, 2), (0, 0, 2, 2), (2, 2, 2, 2)], 1, 0),   # C == A: alias
    (2, 4, 4, [(1, 1, 2, 2), (0, 0, 2, 2), (2, 2, 2, 2)], 1, 0),   # C overlaps A
    (2, 4, 4, [(2, 2, 2, 2), (0, 0, 2, 2), (2, 2, 2, 2)], 1, 0),   # C == B: alias
    (2, 6, 6, [(0, 0, 2, 2), (2, 2, 2, 3), (2, 0, 2, 2)], 1, 0),   # inner dimensions
    (2, 8, 8, [(0, 0, 4, 4), (4, 4, 4, 4), (0, 4, 4, 4)], 3, 9),   # legal, disjoint
]


def main():
    variant_cases = []
    for (v, m, k, n, cutoff, alpha, beta) in VARIANT_CASES:
        acc = v in ACC or v.startswith("blocked")
        A, B = O.fill_random(m, k, 21), O.fill_random(k, n, 22)
        C0 = O.fill_random(m, n, 23) if acc else O.fill_random(m, n, 0) * 0
        rec = dict(variant=v, m=m, k=k, n=n, cutoff=cutoff, alpha=alpha, beta=beta, seed=21)
        try:
            _, _, C2, _, _ = O.ref_run_variant(v, A, B, C0, alpha, beta, cutoff)
            rec["error"] = 0
            rec["c_hash"] = "%016x" % O.fnv1a64(C2)
        except O.RefError as e:
            rec["error"] = e.code
        variant_cases.append(rec)
    prim_cases = []
    for (op, rows, cols, wins, s0, s1) in PRIMITIVE_CASES:
        buf = O.fill_random(rows, cols, 31 + op)
        rc, after = O.ref_primitive_on_windows(op, buf, wins, s0, s1)
        rec = dict(op=op, rows=rows, cols=cols, windows=wins, s0=s0, s1=s1, seed=31 + op, error=rc)
        if rc == 0:
            rec["buf_hash"] = "%016x" % O.fnv1a64(after)
        prim_cases.append(rec)
    out = os.path.join(os.path.dirname(__file__), "error_cases.json")
    json.dump(dict(generator="reference via oracle/_ref/libwinomem_ref.so", modulus=65521,
                   variant_cases=variant_cases, primitive_cases=prim_cases),
              open(out, "w"), indent=1)
    errs = sum(1 for c in variant_cases + prim_cases if c["error"])
    print(len(variant_cases) + len(prim_cases), "cases,", errs, "errors ->", out)


if __name__ == "__main__":
    main()
