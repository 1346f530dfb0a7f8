"""Generate tests/golden/small_cases.json from the REFERENCE implementation.

TEST INFRASTRUCTURE.  Runs the unmodified reference (oracle/_ref, compiled
from /root/reference/proj/include) on seeded small problems and records, per
case, the input seeds, scalars and cutoff, the result hash (FNV-1a over u32
residues), the hashes of A and B afterwards (contract checks) and the full
CostReport.  The GPU parity tests replay every case through the C-ABI and
compare bit-for-bit; the CPU tests pin the oracle and the planner to them.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from oracle import oracle as O  # noqa: E402

ACC = {"acc3", "aclr", "accr", "acc2", "acr"}
SQUARE = [2, 4, 8, 16, 32, 64]


def shapes(v):
    if v == "ipmm":
        return [(n, k, n) for n in (2, 4, 8, 16, 32) for k in (2, 4, 8, 16, 32, 64) if k >= n]
    if v == "ipovmm":
        return [(8, 8, 2), (8, 4, 2), (4, 8, 2), (16, 8, 4), (32, 16, 8), (64, 64, 32)]
    if v in ("std2", "acc3", "acr"):
        out = [(n, n, n) for n in SQUARE]
        out += [(m, k, n) for m in (2, 4, 8) for k in (2, 4, 8) for n in (2, 4, 8)
                if not (m == k == n)]
        out += [(64, 16, 32), (16, 64, 32), (32, 64, 64)]
        return out
    if v.startswith("blocked"):
        return [(n, n, n) for n in (4, 8, 16, 32)]
    return [(n, n, n) for n in SQUARE]


def main():
    variants = ["std2", "acc3", "ip", "ovl", "ovl2", "ovr", "aclr", "accr", "acc2", "acr",
                "ipmm", "ipovmm", "classic", "blocked_acc_t2", "blocked_acc_t2_acc2"]
    cases = []
    for v in variants:
        acc = v in ACC or v.startswith("blocked")
        for (m, k, n) in shapes(v):
            for cutoff in (1, 2, 4):
                for seed in (11, 12):
                    for (alpha, beta) in ([(1, 1 if acc else 0)] + ([(3, 7)] if acc else [(5, 0)])):
                        if v in ("ipmm", "ipovmm") and (alpha, beta) != (1, 0):
                            continue
                        A = O.fill_random(m, k, seed)
                        B = O.fill_random(k, n, seed + 1)
                        C0 = O.fill_random(m, n, seed + 2) if acc else O.fill_random(m, n, 0) * 0
                        try:
                            A2, B2, C2, rep, calls = O.ref_run_variant(v, A, B, C0, alpha, beta,
                                                                      cutoff)
                        except O.RefError as e:
                            cases.append(dict(variant=v, m=m, k=k, n=n, cutoff=cutoff, seed=seed,
                                              alpha=alpha, beta=beta, error=e.code))
                            continue
                        cases.append(dict(variant=v, m=m, k=k, n=n, cutoff=cutoff, seed=seed,
                                          alpha=alpha, beta=beta,
                                          c_hash="%016x" % O.fnv1a64(C2),
                                          a_after="%016x" % O.fnv1a64(A2),
                                          b_after="%016x" % O.fnv1a64(B2),
                                          a_before="%016x" % O.fnv1a64(A),
                                          b_before="%016x" % O.fnv1a64(B),
                                          report=rep, schedule_calls=calls))
    # odd / mixed dimensions (dynamic peeling, executor.hpp:210-236)
    for (m, k, n) in [(3, 3, 3), (5, 7, 9), (6, 6, 6), (12, 10, 14), (7, 16, 5), (9, 2, 9)]:
        for v in ("std2", "acc3"):
            acc = v == "acc3"
            seed = m * 31 + k * 7 + n + (1 if acc else 0)
            A = O.fill_random(m, k, seed)
            B = O.fill_random(k, n, seed + 1)
            C0 = O.fill_random(m, n, seed + 2) if acc else O.fill_random(m, n, 0) * 0
            A2, B2, C2, rep, calls = O.ref_run_variant(v, A, B, C0, 1, 1 if acc else 0, 1)
            cases.append(dict(variant=v, m=m, k=k, n=n, cutoff=1, seed=seed, alpha=1,
                              beta=1 if acc else 0, c_hash="%016x" % O.fnv1a64(C2),
                              a_after="%016x" % O.fnv1a64(A2), b_after="%016x" % O.fnv1a64(B2),
                              a_before="%016x" % O.fnv1a64(A), b_before="%016x" % O.fnv1a64(B),
                              report=rep, schedule_calls=calls))
    out = os.path.join(os.path.dirname(__file__), "small_cases.json")
    json.dump(dict(generator="reference run_variant via oracle/_ref/libwinomem_ref.so",
                   modulus=65521, cases=cases), open(out, "w"), separators=(",", ":"))
    print(len(cases), "cases ->", out)


if __name__ == "__main__":
    main()
