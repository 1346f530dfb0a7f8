import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0707_2347_b200 as W
import bench
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "config_hashes.json")))
for name in ("C1", "C2", "C3"):
    c = GOLD[name]
    for mode in (0, 1, 2, 3):
        for dag in (3, 1):
            A, B, C = W.Matrix(c["m"], c["k"]), W.Matrix(c["k"], c["n"]), W.Matrix(c["m"], c["n"])
            A.fill_random(c["seed"]); B.fill_random(c["seed"] + 1)
            if c["beta"]:
                C.fill_random(c["seed"] + 2)
            ctx = A.ctx()
            ctx.set_option("early_loads", mode)
            ctx.set_option("dag", dag)
            oks = []
            for rep in range(3):
                if rep:
                    if c["variant"] in ("iprect", "ip"):
                        A.fill_random(c["seed"]); B.fill_random(c["seed"] + 1)
                    C.fill_random(c["seed"] + 2) if c["beta"] else None
                W.run_variant(c["variant"], A, B, C, alpha=c["alpha"], beta=c["beta"], cutoff=c["cutoff"])
                oks.append("%016x" % C.hash() == c["appendix_a"])
            print(name, "early", mode, "dag", dag, oks, flush=True)
