"""Schedule DSL (schedule.hpp:261-684): the product's parser and renderer
against the reference's own renderings of every builtin and the reference's
DSL unit cases (proj/tests/unit/test_schedule.cpp:9-62, 146-158).  CPU only."""
import json
import os

import numpy as np

import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "dsl_renderings.json")
NAMES = ["std2", "acc3", "ip", "ovl", "ovl2", "ovr", "aclr", "accr", "acc2", "acr"]


def _renderings():
    return json.load(open(GOLD))["renderings"]


@pytest.mark.parametrize("name", NAMES)
def test_reference_rendering_parses_to_builtin(W, name):
    """The reference's canonical text of each builtin parses to exactly the
    product's builtin (same instructions, scalars, recursion tags, temporaries)."""
    canon, match = W.parse_schedule(_renderings()[name])
    assert match, name
    # and the product's rendering of it parses back to the same schedule
    again, match2 = W.parse_schedule(canon)
    assert match2 and again == canon


@pytest.mark.parametrize("name", NAMES)
def test_render_round_trip(W, name):
    text = W.render_schedule(name)
    canon, match = W.parse_schedule(text)
    assert match and canon == text


def test_reference_rendering_live(W, O):
    """Same check straight from the reference library when it is built here."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    for name in NAMES:
        assert W.parse_schedule(O.ref_render_builtin(name))[1], name


def test_reference_dsl_unit_cases(W):
    E = W.winomem
    # test_schedule.cpp:9-20 -- one addition, defaults
    canon, _ = W.parse_schedule("1: S1 = A21 + A22 @ X\n")
    assert "schedule anonymous" in canon and "shape square" in canon
    assert "1: V1 = A21 + A22 @ X" in canon
    # :22-29 contract checks at parse time
    W.parse_schedule("1: C11 = IP(A11*B11) @ C11\n")
    with pytest.raises(E.contract_violation_error):
        W.parse_schedule("1: A11 = B11 + B12 @ A11\n")
    W.parse_schedule("contract overwrite-A\n1: A11 = B11 + B12 @ A11\n")
    # :31-43 labels resolve to the slot of their defining instruction
    canon, _ = W.parse_schedule("1: S3 = A11 - A21 @ X\n2: T3 = B22 - B12 @ Y\n3: P7 = S3*T3 @ C21\n")
    assert "3: V3 = V1*V2 @ C21" in canon  # untagged plain product: Std2
    # :45-54 untagged accumulating products dispatch to acc3
    canon, _ = W.parse_schedule("accumulating true\n1: U1 = alpha*A12*B21 + beta*C11 @ C11\n")
    assert "1: V1 = alpha*A12*B21 + beta*C11 @ C11" in canon
    canon, _ = W.parse_schedule("accumulating true\n1: U1 = Acc2(alpha*A12*B21 + beta*C11) @ C11\n")
    assert "Acc2(alpha*A12*B21 + beta*C11)" in canon
    # :56-62 parse errors
    with pytest.raises(E.parse_error):
        W.parse_schedule("1: S1 = A21 $ A22 @ X\n")
    with pytest.raises(E.unknown_slot_error):
        W.parse_schedule("1: S1 = A21 + NOPE @ X\n")
    with pytest.raises(E.unknown_slot_error):
        W.parse_schedule("1: S1 = A21 + A22 @ WAT\n")
    with pytest.raises(E.parse_error):
        W.parse_schedule("2: S1 = A21 + A22 @ X\n")
    with pytest.raises(E.parse_error):
        W.parse_schedule("1: P = A11*B11 + A12*B21 @ X\n")
    # scalar outside a tagged call (pure product) and the rejected literal
    canon, _ = W.parse_schedule("accumulating true\n1: U = -alpha*AccR(A22*B11) @ C21\n")
    assert "AccR(-alpha*A22*B11)" in canon
    with pytest.raises(E.parse_error):
        W.parse_schedule("1: S = 3*A11 + A12 @ X\n")


def test_unknown_builtin_render(W):
    with pytest.raises(W.winomem.unknown_schedule_error):
        W.render_schedule("nope")


# A hand-written schedule (not a builtin): std2's table with the roles of the
# two temporaries swapped (operands of the plain products in Y / X).
SWAPPED = """schedule swapped
contract read-only
accumulating false
shape rectangular
temp Y m/2 max(k/2,n/2)
temp X k/2 n/2
1: S3 = A11 - A21 @ Y
2: T3 = B22 - B12 @ X
3: P7 = S3*T3 @ C21
4: S1 = A21 + A22 @ Y
5: T1 = B12 - B11 @ X
6: P5 = S1*T1 @ C22
7: S2 = S1 - A11 @ Y
8: T2 = B22 - T1 @ X
9: P6 = S2*T2 @ C12
10: S4 = A12 - S2 @ Y
11: P3 = S4*B22 @ C11
12: P1 = A11*B11 @ Y
13: U2 = P1 + P6 @ C12
14: U3 = U2 + P7 @ C21
15: U4 = U2 + P5 @ C12
16: U7 = U3 + P5 @ C22
17: U5 = U4 + P3 @ C12
18: T4 = T2 - B21 @ X
19: P4 = A22*T4 @ C11
20: U6 = U3 - P4 @ C21
21: P2 = A12*B21 @ C11
22: U1 = P1 + P2 @ C11
"""


@pytest.mark.parametrize("case", ["std2", "acc2", "aclr", "ip", "acr", "swapped"])
def test_parsed_meter_matches_reference(W, O, case):
    """The planner's meter for a parsed schedule equals the reference's own
    run_parsed_schedule (executor.hpp:304-342), which also yields the right
    product (checked against the reference classical product)."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    text = SWAPPED if case == "swapped" else _renderings()[case]
    acc = case in ("acc2", "aclr", "acr")
    m, k, n = (32, 16, 32) if case in ("acr", "swapped") else (32, 32, 32)
    A, B = O.fill_random(m, k, 3), O.fill_random(k, n, 4)
    C0 = O.fill_random(m, n, 5) if acc else np.zeros((m, n), np.uint32)
    al, be = (3, 7) if acc else (5, 0)
    for cutoff in (1, 4):
        Cr, _, _, rep = O.ref_run_parsed(text, A, B, C0, al, be, cutoff)
        assert (Cr == O.classical_modp(A, B, C0 if acc else None, al, be)).all()
        mine = W.winomem.plan_report_parsed(text, m, k, n, cutoff, al, be)
        assert (mine.mults, mine.adds, mine.peak_extra_words, mine.total_alloc_words) == (
            rep["mults"], rep["adds"], rep["peak_extra_words"], rep["total_alloc_words"]), (case, cutoff)
