"""Pin the CPU oracle (oracle/) against the reference's known-answer tests and
golden fixtures.  CPU only."""
import json
import os

import numpy as np
import pytest

from conftest import has_ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix_stream_pinned(O):
    # proj/tests/unit/test_io.cpp:37-46
    raw = np.zeros(3, dtype=np.uint64)
    O.lib().wmo_splitmix_raw(raw, 3, 1)
    assert [int(x) for x in raw] == [0x910a2dec89025cc1, 0xbeeb8da1658eec67, 0xf893a2eefb32555e]
    a = O.fill_random(2, 2, 1)
    assert int(a[0, 0]) == 0x910a2dec89025cc1 % 65521


def test_fill_deterministic_per_seed(O):
    # test_ring.cpp:262-270
    a, b = O.fill_random(6, 6, 123), O.fill_random(6, 6, 123)
    assert (a == b).all()
    c = O.fill_random(6, 6, 124)
    assert not (a == c).all()
    assert O.fnv1a64(a) != O.fnv1a64(c)


def _addsub(O, a, b, sa, sb, p):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    d = np.zeros_like(a)
    r, c = a.shape
    O.lib().wmo_block_addsub(r, c, p, d.reshape(-1), c, a.reshape(-1), c, b.reshape(-1), c, sa, sb)
    return d


def test_block_addsub_kats(O):
    # test_ring.cpp:47-72
    x = np.array([[1]], dtype=np.uint32)
    assert _addsub(O, x, x, 1, 65520, 65521)[0, 0] == 0
    d = _addsub(O, [[1, 2], [3, 4]], [[5, 6], [7, 8]], 1, 1, 101)
    assert d.tolist() == [[6, 8], [10, 12]]
    assert _addsub(O, [[1]], [[2]], 3, 95, 97)[0, 0] == 96


def test_block_addsub_inverse(O):
    # test_ring.cpp:88-100
    for t in range(10):
        a, b = O.fill_random(3, 5, 100 + t), O.fill_random(3, 5, 200 + t)
        s = _addsub(O, a, b, 1, 1, 65521)
        back = _addsub(O, s, b, 1, 65520, 65521)
        assert (back == a).all()


def _indep_ref(A, B, p):
    # independent k-outer reference with per-step reduction (test_ring.cpp:11-24)
    A = A.astype(object)
    B = B.astype(object)
    m, k = A.shape
    n = B.shape[1]
    C = np.zeros((m, n), dtype=object)
    for l in range(k):
        C = (C + np.outer(A[:, l], B[l, :])) % p
    return C.astype(np.uint32)


def test_classical_kats(O):
    # test_ring.cpp:102-128
    C = O.classical_modp(np.array([[1, 2], [3, 4]]), np.array([[5, 6], [7, 8]]), p=1009)
    assert C.tolist() == [[19, 22], [43, 50]]
    I = np.eye(2, dtype=np.uint32)
    B = O.fill_random(2, 2, 42)
    assert (O.classical_modp(I, B) == B).all()
    assert O.classical_modp(np.array([[1]]), np.array([[1]]))[0, 0] == 1


def test_classical_vs_independent(O):
    # test_ring.cpp:130-142 (sizes <= 16) and the large-modulus path 144-151
    seed = 7
    for m in range(1, 17, 5):
        for k in range(1, 17, 5):
            for n in range(1, 17, 5):
                A, B = O.fill_random(m, k, seed), O.fill_random(k, n, seed + 1)
                seed += 2
                assert (O.classical_modp(A, B) == _indep_ref(A, B, 65521)).all()
    A, B = O.fill_random(5, 7, 1, 2147483647), O.fill_random(7, 3, 2, 2147483647)
    assert (O.classical_modp(A, B, p=2147483647) == _indep_ref(A, B, 2147483647)).all()


def test_classical_alpha_beta(O):
    # test_ring.cpp:153-170
    A, B, C0 = O.fill_random(4, 4, 11), O.fill_random(4, 4, 12), O.fill_random(4, 4, 13)
    got = O.classical_modp(A, B, C0, 5, 9)
    P = _indep_ref(A, B, 65521).astype(np.int64)
    want = (5 * P + 9 * C0.astype(np.int64)) % 65521
    assert (got == want).all()


@pytest.mark.skipif(not has_ref(), reason="reference build (oracle/_ref) absent")
def test_oracle_matches_reference_classical(O):
    rng = np.random.default_rng(5)
    for _ in range(12):
        m, k, n = (int(x) for x in rng.integers(1, 70, 3))
        A, B, C0 = O.fill_random(m, k, 1), O.fill_random(k, n, 2), O.fill_random(m, n, 3)
        al, be = int(rng.integers(0, 65521)), int(rng.integers(0, 65521))
        want = C0.copy()
        O.ref().ref_classical_mul(m, k, n, 65521, A.reshape(-1), B.reshape(-1), want.reshape(-1),
                                  al, be)
        assert (O.classical_modp(A, B, C0, al, be) == want).all()
        assert O.fnv1a64(want) == int(O.ref().ref_hash(want.reshape(-1), want.size))


@pytest.mark.skipif(not has_ref(), reason="reference build (oracle/_ref) absent")
def test_oracle_matches_reference_addsub(O):
    for t in range(5):
        a, b = O.fill_random(7, 9, t), O.fill_random(7, 9, t + 50)
        for sa, sb in [(1, 1), (1, 65520), (3, 7), (65520, 65520)]:
            want = np.zeros_like(a)
            O.ref().ref_block_addsub(7, 9, 65521, a.reshape(-1), b.reshape(-1), want.reshape(-1),
                                     sa, sb)
            assert (_addsub(O, a, b, sa, sb, 65521) == want).all()


def test_models_spot_values():
    # test_models.cpp:22-43
    from oracle.models import expected_costs as E
    ops = lambda r: r["mults"] + r["adds"]  # noqa: E731
    assert ops(E("std2", 2, 2, 2, 1)) == 22
    assert ops(E("acc3", 2, 2, 2, 1)) == 26
    assert E("acc3", 2, 2, 2, 1)["adds"] == 19
    assert ops(E("aclr", 2, 2, 2, 1)) == 28 and ops(E("accr", 2, 2, 2, 1)) == 28
    assert ops(E("acc2", 2, 2, 2, 1)) == 30
    assert ops(E("ipmm", 2, 2, 2, 1)) == 12 and ops(E("ipmm", 4, 4, 4, 1)) == 172
    assert ops(E("blocked_acc_t2", 4, 4, 4, 1)) == 208
    assert E("std2", 4, 4, 4, 1)["peak_extra_words"] == 10
    assert E("acc3", 4, 4, 4, 1)["peak_extra_words"] == 15
    assert E("ip", 64, 64, 64, 1)["peak_extra_words"] == 0
    assert E("acc2", 32, 32, 32, 1)["peak_extra_words"] == 682


def test_models_closed_forms():
    # test_models.cpp:45-84
    from oracle.models import expected_costs as E
    for j in range(1, 9):
        n = 1 << j
        p7, p4 = 7 ** j, 4 ** j
        ops = lambda v: E(v, n, n, n, 1)["mults"] + E(v, n, n, n, 1)["adds"]  # noqa: E731
        for v in ("std2", "ip", "ovl", "ovr", "ovl2"):
            assert ops(v) == 6 * p7 - 5 * p4
        assert ops("acc3") == 6 * p7 - 4 * p4
        assert ops("aclr") == 6 * p7 - 4 * p4 + p4 * j // 2
        assert E("std2", n, n, n, 1)["peak_extra_words"] == 2 * (p4 - 1) // 3
        assert E("acc3", n, n, n, 1)["peak_extra_words"] == p4 - 1
        assert E("ovl", n, n, n, 1)["peak_extra_words"] == (p4 - 1) // 3
        for v in ("aclr", "accr", "acc2"):
            assert E(v, n, n, n, 1)["peak_extra_words"] == 2 * (p4 - 1) // 3
        assert E("std2", n, n, n, 1)["total_alloc_words"] == 2 * (p7 - p4) // 3


@pytest.mark.skipif(not has_ref(), reason="reference build (oracle/_ref) absent")
def test_models_match_reference(O):
    from oracle.models import expected_costs as E
    for v in ("std2", "acc3", "ip", "ovl", "ovl2", "ovr", "aclr", "accr", "acc2", "acr", "ipmm",
              "classic", "blocked_acc_t2", "blocked_acc_t2_acc2"):
        for (m, k, n, c) in [(16, 16, 16, 1), (64, 64, 64, 4), (1024, 1024, 1024, 128),
                             (4096, 4096, 4096, 256)]:
            assert E(v, m, k, n, c) == O.ref_expected_costs(v, m, k, n, c), (v, m, c)
    for (m, k, n) in [(8, 8, 2), (64, 32, 16)]:
        assert E("ipovmm", m, k, n, 1) == O.ref_expected_costs("ipovmm", m, k, n, 1)


def test_golden_small_cases_consistent_with_oracle(O):
    """The oracle classical product reproduces every reference result hash of
    the golden fixture (any exact algorithm yields the same residues)."""
    g = json.load(open(os.path.join(GOLD, "small_cases.json")))
    checked = 0
    for c in g["cases"]:
        if "error" in c or c["cutoff"] != 1 or c["seed"] != 11:
            continue
        acc = c["variant"] in ("acc3", "aclr", "accr", "acc2", "acr") or c["variant"].startswith(
            "blocked")
        A = O.fill_random(c["m"], c["k"], c["seed"])
        B = O.fill_random(c["k"], c["n"], c["seed"] + 1)
        C0 = O.fill_random(c["m"], c["n"], c["seed"] + 2) if acc else None
        out = O.classical_modp(A, B, C0, c["alpha"], c["beta"], threads=1)
        assert "%016x" % O.fnv1a64(out) == c["c_hash"], c
        checked += 1
    assert checked > 100


def test_config_hashes_pinned():
    g = json.load(open(os.path.join(GOLD, "config_hashes.json")))
    for name in ("C1", "C2"):
        assert g[name]["hash"] == g[name]["appendix_a"], name
