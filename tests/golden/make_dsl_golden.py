"""Generate tests/golden/dsl_renderings.json: the reference's own canonical DSL
rendering (render_schedule(builtin(name)), schedule.hpp:617-684) of every
builtin schedule, produced by the unmodified reference headers compiled into
oracle/_ref.  Run in the container that has /root/reference:

    python tests/golden/make_dsl_golden.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

NAMES = ["std2", "acc3", "ip", "ovl", "ovl2", "ovr", "aclr", "accr", "acc2", "acr"]

if __name__ == "__main__":
    out = {"source": "reference render_schedule(builtin(name)) via oracle/_ref",
           "renderings": {n: O.ref_render_builtin(n) for n in NAMES}}
    json.dump(out, open(os.path.join(HERE, "dsl_renderings.json"), "w"), indent=1)
    print("wrote", len(out["renderings"]), "renderings")
