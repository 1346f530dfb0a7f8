"""Recompute the full-size golden result hashes of BASELINE configs 1-4.

TEST INFRASTRUCTURE.  Run in the build container (needs oracle/_ref, i.e. the
reference headers, for configs 1-2).  Writes tests/golden/config_hashes.json.
  C1: reference run_variant("std2", 1024^3, cutoff 128, seed 1)
  C2: reference run_variant("acc2", 4096^3, cutoff 256, seed 2, alpha=beta=1)
  C3: oracle classical product 8192x4096x8192, seed 3 (no reference schedule
      for an in-place rectangle; any exact algorithm gives the same residues)
  C4: oracle classical product 16384^3, seed 4
Each is checked against SURVEY.md Appendix A.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from oracle import oracle as O  # noqa: E402

APPENDIX_A = {"C1": "daa9cb46175f2616", "C2": "a1055f79e7327495",
              "C3": "0acdeefa67888e7c", "C4": "f3592b33d92d1db6"}
CONFIGS = {
    "C1": dict(variant="std2", m=1024, k=1024, n=1024, cutoff=128, seed=1, alpha=1, beta=0),
    "C2": dict(variant="acc2", m=4096, k=4096, n=4096, cutoff=256, seed=2, alpha=1, beta=1),
    "C3": dict(variant="iprect", m=8192, k=4096, n=8192, cutoff=256, seed=3, alpha=1, beta=0),
    "C4": dict(variant="ipmm", m=16384, k=16384, n=16384, cutoff=512, seed=4, alpha=1, beta=0),
}


def compute(name):
    c = CONFIGS[name]
    A = O.fill_random(c["m"], c["k"], c["seed"])
    B = O.fill_random(c["k"], c["n"], c["seed"] + 1)
    C0 = O.fill_random(c["m"], c["n"], c["seed"] + 2) if c["beta"] else None
    t = time.time()
    if name in ("C1", "C2"):
        Cm = C0 if C0 is not None else O.fill_random(c["m"], c["n"], 0) * 0
        _, _, out, rep, _ = O.ref_run_variant(c["variant"], A, B, Cm, c["alpha"], c["beta"],
                                              c["cutoff"])
        how = "reference run_variant"
    else:
        out = O.classical_modp(A, B, C0, c["alpha"], c["beta"])
        how = "oracle classical_modp (threads=%d)" % (os.cpu_count() or 1)
    h = "%016x" % O.fnv1a64(out)
    return dict(c, hash=h, how=how, seconds=round(time.time() - t, 1))


if __name__ == "__main__":
    names = sys.argv[1:] or list(CONFIGS)
    path = os.path.join(os.path.dirname(__file__), "config_hashes.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for nm in names:
        r = compute(nm)
        r["appendix_a"] = APPENDIX_A[nm]
        r["agrees_with_appendix_a"] = r["hash"] == APPENDIX_A[nm]
        print(nm, r, flush=True)
        data[nm] = r
        json.dump(data, open(path, "w"), indent=1)
