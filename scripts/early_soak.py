import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0707_2347_b200 as W
GOLD = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "config_hashes.json")))
bad = 0
for name in ("C1", "C2", "C3", "C4"):
    c = GOLD[name]
    for dag in (2, 3, 4, 6):
        A, B, C = W.Matrix(c["m"], c["k"]), W.Matrix(c["k"], c["n"]), W.Matrix(c["m"], c["n"])
        ctx = A.ctx()
        ctx.set_option("dag", dag)
        oks = []
        for rep in range(6):
            A.fill_random(c["seed"]); B.fill_random(c["seed"] + 1)
            if c["beta"]:
                C.fill_random(c["seed"] + 2)
            W.run_variant(c["variant"], A, B, C, alpha=c["alpha"], beta=c["beta"], cutoff=c["cutoff"])
            oks.append("%016x" % C.hash() == c["appendix_a"])
        bad += oks.count(False)
        print(name, "dag", dag, oks, flush=True)
        del A, B, C
print("mismatches", bad)
