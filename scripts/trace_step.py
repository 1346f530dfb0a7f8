"""Launch timeline of one multiplication (timing event after every launch,
concurrent issue) and its critical path, attributed per launch kind.

    python scripts/trace_step.py [C2]
"""
import os; os.environ.setdefault("WM_DIAG", "1")  # the wm_diag_* probes live in the diag library  # noqa: E702,E401
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_0707_2347_b200 as W  # noqa: E402
from paper_0707_2347_b200._lib import lib  # noqa: E402

KINDS = ["ADD", "MUL", "FRAME", "GROUP", "PREP", "GEMM", "COMB", "UPLOAD", "DOWNLOAD"]


def main():
    import torch
    name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "C2"
    cfg = bench.CONFIGS[name]
    m, k, n = cfg["m"], cfg["k"], cfg["n"]
    A, B, Cm = W.Matrix(m, k), W.Matrix(k, n), W.Matrix(m, n)
    A.fill_random(cfg["seed"]); B.fill_random(cfg["seed"] + 1)
    ctx = A.ctx()
    for kv in filter(None, os.environ.get("WM_OPTS", "").split(",")):
        a, b = kv.split("=")
        ctx.set_option(a, int(b))
    ctx.set_option("trace", 1)
    run = lambda: W.run_variant(cfg["variant"], A, B, Cm, alpha=cfg["alpha"], beta=cfg["beta"],
                                cutoff=cfg["cutoff"])
    if "--e2e" in sys.argv:  # the host boundary streamed through the graph (pinned u32)
        from oracle import oracle as O
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
        hA, hB = pin(O.fill_random(m, k, cfg["seed"])), pin(O.fill_random(k, n, cfg["seed"] + 1))
        hC = pin(O.fill_random(m, n, cfg["seed"] + 2))
        import time

        def run():
            t0 = time.perf_counter()
            W.run_variant_host(cfg["variant"], hA, hB, hC, cfg["alpha"], cfg["beta"], cfg["cutoff"])
            print("e2e wall ms", round((time.perf_counter() - t0) * 1e3, 3), file=sys.stderr)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    L = lib()
    L.wm_diag_trace.argtypes = [C.c_void_p, C.c_int] + [C.c_void_p] * 6
    N = 200000
    start = np.zeros(N); end = np.zeros(N); kind = np.zeros(N, np.int32)
    lane = np.zeros(N, np.int32); waits = np.zeros(4 * N, np.int32); nn = C.c_int()
    rc = L.wm_diag_trace(ctx.h, N, start.ctypes.data, end.ctypes.data, kind.ctypes.data,
                         lane.ctypes.data, waits.ctypes.data, C.byref(nn))
    assert rc == 0, L.wm_last_error()
    n_ = nn.value
    start, end, kind, lane = start[:n_], end[:n_], kind[:n_], lane[:n_]
    dump = os.environ.get("WM_TRACE_DUMP")
    if dump:  # the raw timeline, for offline analysis
        json.dump({"start": start.tolist(), "end": end.tolist(), "kind": kind.tolist(),
                   "lane": lane.tolist()}, open(dump, "w"))
    waits = waits[:4 * n_].reshape(n_, 4)
    prev_on_lane = np.full(n_, -1)
    last = {}
    for j in range(n_):
        prev_on_lane[j] = last.get(lane[j], -1)
        last[lane[j]] = j
    # critical path: from the last-ending launch, follow the predecessor that ended
    # last; a launch's time on the path = its end - that predecessor's end, split
    # into the gap before its first CTA started and its own span
    j = int(np.argmax(end))
    crit, gaps, edges = {}, {}, {}
    lane_edges = {"same": [0, 0.0], "cross": [0, 0.0]}  # critical edges: count, gap us
    path = 0
    while j >= 0:
        preds = [p for p in [prev_on_lane[j]] + [w for w in waits[j] if w >= 0] if p >= 0]
        p = max(preds, key=lambda q: end[q]) if preds else -1
        pe = end[p] if p >= 0 else 0.0
        k_ = KINDS[kind[j]]
        e_ = (KINDS[kind[p]] if p >= 0 else "-") + ">" + k_
        edges[e_] = edges.get(e_, 0) + 1
        crit[k_] = crit.get(k_, 0.0) + end[j] - max(start[j], pe)
        gaps[k_] = gaps.get(k_, 0.0) + max(0.0, start[j] - pe)
        if p >= 0:
            le = lane_edges["same" if lane[p] == lane[j] else "cross"]
            le[0] += 1
            le[1] += max(0.0, start[j] - pe)
        path += 1
        j = p
    span = {}
    for j in range(n_):
        k_ = KINDS[kind[j]]
        span.setdefault(k_, []).append(end[j] - start[j])
    stats = {k_: {"n": len(v), "mean_us": round(float(np.mean(v)), 2),
                  "p50_us": round(float(np.median(v)), 2)} for k_, v in span.items()}
    busy = crit
    timed = start >= 0
    first_compute = float(start[timed].min()) if timed.any() else -1.0
    print(json.dumps({"config": name, "launches": int(n_), "step_us": float(end.max()),
                      "first_kernel_start_us": first_compute,
                      "untimed_launches": int((~timed).sum()),
                      "critical_launches": path,
                      "critical_span_us_by_kind": {k_: round(v, 1) for k_, v in crit.items()},
                      "critical_gap_us_by_kind": {k_: round(v, 1) for k_, v in gaps.items()},
                      "span_stats": stats,
                      "critical_edges_by_lane": {k_: {"n": v[0], "gap_us": round(v[1], 1)}
                                                 for k_, v in lane_edges.items()},
                      "critical_edges": dict(sorted(edges.items(), key=lambda kv: -kv[1])[:12]),
                      "lanes": {int(l): int((lane == l).sum()) for l in np.unique(lane)}}))


if __name__ == "__main__":
    main()
