"""Schedule DSL (schedule.hpp:261-684): the product's parser and renderer
against the reference's own renderings of every builtin and the reference's
DSL unit cases (proj/tests/unit/test_schedule.cpp:9-62, 146-158).  CPU only."""
import json
import os

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
