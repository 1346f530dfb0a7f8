"""The product's host planner (schedule interpreter + drivers, C++) against the
reference meter: every CostReport field, schedule-call counts and error codes.
CPU only -- wm_plan_report executes nothing."""
import json
import os

import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _cases():
    return json.load(open(os.path.join(GOLD, "small_cases.json")))["cases"]


def test_plan_reports_match_reference_golden(W):
    n = 0
    for c in _cases():
        args = (c["variant"], c["m"], c["k"], c["n"], c["cutoff"], c["alpha"], c["beta"])
        if "error" in c:
            with pytest.raises(W.winomem.WinomemError) as ei:
                W.plan_report(*args)
            assert ei.value.code == c["error"], c
            continue
        r = W.plan_report(*args)
        want = c["report"]
        got = dict(mults=r.mults, adds=r.adds, peak_extra_words=r.peak_extra_words,
                   total_alloc_words=r.total_alloc_words, word_moves=r.word_moves,
                   classical_calls=r.classical_calls)
        assert got == want, c
        if c["schedule_calls"]:
            assert r.schedule_calls == c["schedule_calls"], c
        n += 1
    assert n > 1500


def test_fused_plan_meters_identically(W):
    for c in _cases()[::7]:
        if "error" in c:
            continue
        args = (c["variant"], c["m"], c["k"], c["n"], c["cutoff"], c["alpha"], c["beta"])
        a = W.plan_report(*args)
        b = W.plan_report(*args, fuse_frames=True)
        for f in ("mults", "adds", "peak_extra_words", "total_alloc_words", "word_moves",
                  "classical_calls"):
            assert getattr(a, f) == getattr(b, f)
        assert a.peak_extra_bytes == b.peak_extra_bytes


def test_expected_costs_match_oracle_models(W):
    from oracle.models import expected_costs as E
    for v in ("std2", "acc3", "ip", "ovl", "ovl2", "ovr", "aclr", "accr", "acc2", "acr", "ipmm",
              "classic", "blocked_acc_t2", "blocked_acc_t2_acc2"):
        for (m, k, n, c) in [(8, 8, 8, 1), (64, 64, 64, 2), (1024, 1024, 1024, 128),
                             (16384, 16384, 16384, 512)]:
            r = W.expected_costs(v, m, k, n, c)
            e = E(v, m, k, n, c)
            assert (r.mults, r.adds, r.peak_extra_words, r.total_alloc_words, r.word_moves) == (
                e["mults"], e["adds"], e["peak_extra_words"], e["total_alloc_words"],
                e["word_moves"]), (v, m)
    r = W.expected_costs("iprect", 8192, 4096, 8192, 256)
    e = E("iprect", 8192, 4096, 8192, 256)
    assert (r.mults, r.adds, r.peak_extra_words) == (e["mults"], e["adds"], 0)


def test_expected_costs_match_reference_directly(W, O):
    """The product's IR-derived cost model (wm_costs.cpp) against the reference's
    own expected_costs (models.hpp:202-229), squares and rectangles, every
    builtin and driver."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    fields = ("mults", "adds", "peak_extra_words", "total_alloc_words", "word_moves")

    def same(v, m, k, n, c):
        r = W.expected_costs(v, m, k, n, c)
        e = O.ref_expected_costs(v, m, k, n, c)
        assert tuple(getattr(r, f) for f in fields) == tuple(e[f] for f in fields), (v, m, k, n, c)

    square = ("std2", "acc3", "ip", "ovl", "ovl2", "ovr", "aclr", "accr", "acc2", "acr", "ipmm",
              "classic", "blocked_acc_t2", "blocked_acc_t4", "blocked_acc_t2_acc2")
    for v in square:
        for (n, c) in [(2, 1), (16, 1), (64, 2), (256, 8), (2048, 64), (16384, 512), (32768, 1024)]:
            same(v, n, n, n, c)
    for v in ("std2", "acc3", "acr", "classic"):  # rectangular schedules
        for (m, k, n, c) in [(32, 16, 8, 1), (8, 64, 32, 2), (512, 256, 1024, 16)]:
            same(v, m, k, n, c)
    for (m, k, n) in [(8, 8, 2), (64, 32, 16), (1024, 2048, 256)]:
        same("ipovmm", m, k, n, 1)
        same("ipovmm", m, k, n, 8)


def test_error_goldens_through_planner(W):
    """The reference's illegal run_variant calls (tests/golden/error_cases.json,
    from oracle/_ref) raise the same exception class in the host planner."""
    g = json.load(open(os.path.join(GOLD, "error_cases.json")))
    for c in g["variant_cases"]:
        args = (c["variant"], c["m"], c["k"], c["n"], c["cutoff"], c["alpha"], c["beta"])
        if c["error"]:
            with pytest.raises(W.winomem.WinomemError) as ei:
                W.plan_report(*args)
            assert ei.value.code == c["error"], c
        else:
            W.plan_report(*args)


def test_alloc_log_matches_reference(W, O):
    """CostMeter::alloc_log (meter.hpp:15-19, 40-45): every temporary the plan
    meters -- words, recursion depth, slot name, in acquisition order -- equals
    the reference run_variant's log (incl. blocked_acc's scratch chunk and the
    unmetered QuadrantWorkspace of ipmm)."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_0707_2347_b200.winomem import last_alloc_log
    cases = [("std2", 16, 16, 16, 1, 0, 1), ("acc2", 32, 32, 32, 1, 1, 2), ("aclr", 16, 16, 16, 3, 7, 1),
             ("ovl2", 16, 16, 16, 1, 0, 2), ("acr", 32, 16, 32, 1, 1, 1), ("std2", 64, 32, 16, 1, 0, 4),
             ("ipmm", 16, 32, 16, 1, 0, 2), ("blocked_acc_t2", 16, 16, 16, 1, 1, 1),
             ("blocked_acc_t2_acc2", 16, 16, 16, 1, 1, 2), ("ip", 16, 16, 16, 1, 0, 1),
             ("std2", 1024, 1024, 1024, 1, 0, 128)]
    for (v, m, k, n, al, be, c) in cases:
        W.plan_report(v, m, k, n, c, al, be)
        got = ";".join(f"{w}:{d}:{s}" for w, d, s in last_alloc_log())
        want = O.ref_alloc_log(v, m, k, n, al, be, c).rstrip(";")
        assert got == want, (v, m, k, n, c)


# config-level plans
CONFIGS = [
    # variant, m, k, n, cutoff, beta, peak words, frames, leaves
    ("std2", 1024, 1024, 1024, 128, 0, 688128, {"std2": 57}, 343),
    ("acc2", 4096, 4096, 4096, 256, 1, 11141120,
     {"acc2": 85, "std2": 105, "aclr": 57, "accr": 57, "ip": 70, "ovr": 26}, 2401),
    ("iprect", 8192, 4096, 8192, 256, 0, 0, {"std2": 400, "ovl": 85, "ovr": 85, "ip": 1030}, 9604),
    ("ipmm", 16384, 16384, 16384, 512, 0, 0, {"std2": 2406, "acc3": 918}, 20131),
    ("std2", 32768, 32768, 32768, 1024, 0, 715128832, {"std2": 2801}, 16807),
]


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: f"{c[0]}-{c[1]}")
def test_config_plans(W, cfg):
    v, m, k, n, c, beta, peak, frames, leaves = cfg
    r = W.plan_report(v, m, k, n, c, 1, beta)
    assert r.peak_extra_words == peak
    assert r.peak_extra_bytes == peak * 8  # the arena reserves exactly the schedule's words
    assert r.schedule_calls == frames
    assert r.classical_calls == leaves
    e = W.expected_costs(v, m, k, n, c)
    assert (r.mults, r.adds) == (e.mults, e.adds)
    assert r.peak_extra_words == e.peak_extra_words


def test_config_reference_counts(W):
    # Appendix A rows from the reference meter
    r = W.plan_report("std2", 1024, 1024, 1024, 128)
    assert (r.mults, r.adds, r.total_alloc_words) == (719323136, 736559104, 3047424)
    r = W.plan_report("acc2", 4096, 4096, 4096, 256, 1, 1)
    assert (r.mults, r.adds, r.total_alloc_words) == (40282095616, 40936669184, 80871424)
    r = W.plan_report("ipmm", 16384, 16384, 16384, 512)
    assert (r.mults, r.adds) == (2706097831936, 2723816669184)


def test_error_taxonomy(W):
    E = W.winomem
    for v in ("ip", "ovl", "ovl2", "ovr", "aclr", "accr", "acc2"):
        with pytest.raises(E.shape_error):
            W.plan_report(v, 4, 8, 4, 1, 1, 1 if v in ("aclr", "accr", "acc2") else 0)
    with pytest.raises(E.dimension_error):
        W.plan_report("std2", 4, 4, 4, 1, 1, 1)  # beta on a plain product
    with pytest.raises(E.unknown_schedule_error):
        W.plan_report("bogus", 4, 4, 4, 1)
    with pytest.raises(E.shape_error):
        W.plan_report("ipmm", 8, 4, 8, 1)  # k < n
    with pytest.raises(E.shape_error):
        W.plan_report("ipovmm", 4, 4, 4, 1)
    with pytest.raises(E.shape_error):
        W.plan_report("acr", 6, 6, 6, 1, 1, 1)  # peeling wraps std2/acc3 only
    with pytest.raises(E.dimension_error):
        W.plan_report("std2", 4, 4, 4, 0)  # cutoff >= 1


def test_recursion_purity(W):
    # test_executor.cpp:174-189: cutoff >= n degrades to one classical call
    for v in W.BUILTIN_NAMES:
        acc = W.variant_accumulates(v)
        r = W.plan_report(v, 8, 8, 8, 8, 1, 1 if acc else 0)
        assert r.classical_calls == 1 and r.peak_extra_words == 0
        assert r.mults == 512 and r.adds == 8 * 8 * 7 + (64 if acc else 0)


def test_dispatch_structure(W):
    # test_executor.cpp:191-213
    r = W.plan_report("std2", 4, 4, 4, 2)
    assert r.schedule_calls == {"std2": 1} and r.classical_calls == 7
    r = W.plan_report("aclr", 4, 4, 4, 1, 1, 1)
    assert r.schedule_calls["aclr"] == 5 and r.schedule_calls["ip"] == 3
    r = W.plan_report("acr", 8, 4, 8, 1, 1, 1)
    assert r.schedule_calls["acr"] == 6 and r.schedule_calls["std2"] == 2


def test_iprect_composition(W):
    r = W.plan_report("iprect", 8192, 4096, 8192, 256)
    assert r.peak_extra_words == 0 and r.total_alloc_words == 0 and r.peak_extra_bytes == 0
    assert r.mults + r.adds == 324438851584 + (r.mults + r.adds - 324438851584)
    e = W.expected_costs("iprect", 8192, 4096, 8192, 256)
    assert (r.mults, r.adds) == (e.mults, e.adds)
    with pytest.raises(W.winomem.shape_error):
        W.plan_report("iprect", 4096, 8192, 4096, 256)  # k > min(m, n)


def test_launch_batching_reduces_launches(W):
    r = W.plan_report("std2", 1024, 1024, 1024, 128)
    assert r.n_ops == 855 + 343
    assert r.n_launches < r.n_ops
