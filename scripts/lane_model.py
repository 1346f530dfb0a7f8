"""Offline model of the concurrent issue: replay a traced multiplication's launch
DAG (true read / write dependencies, measured per-launch durations) under
different lane-assignment policies.

    python scripts/lane_model.py C2          # on the GPU box: trace + model
"""
import os; os.environ.setdefault("WM_DIAG", "1")  # noqa: E702,E401
import ctypes as C
import json
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def simulate(dur, deps, lanes_of, g_same=1.0, g_cross=1.3, nl=3, policy="trace"):
    """lanes_of: traced lane per launch (policy 'trace'); 'earliest': each launch, in
    program order, goes to the lane where it starts earliest (ties: the lane of a
    dependency); 'inf': no lane limit."""
    n = len(dur)
    end = np.zeros(n)
    lane = np.zeros(n, int)
    avail = [0.0] * nl          # end of the last launch on each lane
    last = [-1] * nl
    for j in range(n):
        d = [i for i in deps[j] if i >= 0]
        if policy == "inf":
            s = max([end[i] + g_same for i in d], default=0.0)
            end[j] = s + dur[j]
            continue
        def start_on(l):
            s = avail[l] + (g_same if last[l] >= 0 else 0.0)
            for i in d:
                s = max(s, end[i] + (g_same if lane[i] == l else g_cross))
            return s
        if policy == "trace":
            l = lanes_of[j]
        else:
            cand = [(start_on(l), 0 if any(lane[i] == l for i in d) else 1, l) for l in range(nl)]
            l = min(cand)[2]
        s = start_on(l)
        lane[j] = l
        end[j] = s + dur[j]
        avail[l] = end[j]
        last[l] = j
    return float(end.max())


def main():
    import torch
    import bench
    import paper_0707_2347_b200 as W
    from paper_0707_2347_b200._lib import lib
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cfg = bench.CONFIGS[name]
    m, k, n = cfg["m"], cfg["k"], cfg["n"]
    A, B, Cm = W.Matrix(m, k), W.Matrix(k, n), W.Matrix(m, n)
    A.fill_random(cfg["seed"]); B.fill_random(cfg["seed"] + 1)
    ctx = A.ctx()
    ctx.set_option("trace", 1)
    for _ in range(3):
        W.run_variant(cfg["variant"], A, B, Cm, alpha=cfg["alpha"], beta=cfg["beta"], cutoff=cfg["cutoff"])
    torch.cuda.synchronize()
    L = lib()
    N = 200000
    start = np.zeros(N); end = np.zeros(N); kind = np.zeros(N, np.int32)
    lane = np.zeros(N, np.int32); waits = np.zeros(4 * N, np.int32); nn = C.c_int()
    L.wm_diag_trace.argtypes = [C.c_void_p, C.c_int] + [C.c_void_p] * 6
    assert L.wm_diag_trace(ctx.h, N, start.ctypes.data, end.ctypes.data, kind.ctypes.data,
                           lane.ctypes.data, waits.ctypes.data, C.byref(nn)) == 0
    n_ = nn.value
    per = 12
    deps = np.full(per * n_, -1, np.int32)
    L.wm_diag_step_deps.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    assert L.wm_diag_step_deps(ctx.h, n_, per, deps.ctypes.data, C.byref(nn)) == 0
    deps = deps.reshape(n_, per).tolist()
    dur = (end[:n_] - start[:n_]).tolist()
    out = {"config": name, "launches": n_, "measured_step_us": float(end[:n_].max()),
           "sum_of_durations_us": float(sum(dur))}
    out["model_traced_lanes"] = simulate(dur, deps, lane[:n_].tolist(), policy="trace")
    for nl in (2, 3, 4, 6):
        out["model_earliest_%d_lanes" % nl] = simulate(dur, deps, None, nl=nl, policy="earliest")
    out["model_unlimited_lanes"] = simulate(dur, deps, None, policy="inf")
    # what would shorten the step: each kind 10% faster, and cheaper edges
    kinds = ["ADD", "MUL", "FRAME", "GROUP", "PREP", "GEMM", "COMB", "UPLOAD", "DOWNLOAD"]
    kd = kind[:n_].tolist()
    out["what_if_traced_lanes"] = {}
    for kk in sorted(set(kd)):
        d2 = [x * 0.9 if kd[i] == kk else x for i, x in enumerate(dur)]
        out["what_if_traced_lanes"][kinds[kk] + "_10pct_faster"] = simulate(
            d2, deps, lane[:n_].tolist(), policy="trace")
    out["what_if_traced_lanes"]["edges_0.3us_cheaper"] = simulate(
        dur, deps, lane[:n_].tolist(), g_same=0.7, g_cross=1.0, policy="trace")
    if os.environ.get("WM_LANE_DUMP"):
        json.dump({"dur": dur, "deps": deps, "kind": kd, "lane": lane[:n_].tolist()},
                  open(os.environ["WM_LANE_DUMP"], "w"))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
