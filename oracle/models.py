"""TEST INFRASTRUCTURE ONLY -- restatement of the reference cost models.

Exact mults/adds/peak/total recurrences per schedule, evaluated down to the
cutoff with classical costs below it, restated from
/root/reference/proj/include/winomem/models.hpp:
  classical_costs  models.hpp:25-31
  Evaluator.eval   models.hpp:95-171 (std2 99-106, acc3 107-115, ip 116-119,
                   ovl/ovr 120-126, ovl2 127-135, aclr 136-142, accr 143-150,
                   acc2 151-161, acr 162-169)
  ipmm             models.hpp:47-58
  ipovmm           models.hpp:60-71
  blocked_acc      models.hpp:73-89
plus the builder's in-place rectangle driver ``iprect`` (config 3; no
reference counterpart -- composed per PAPER.md:588-598).
Pinned against the reference's own ``expected_costs`` in tests/test_oracle.py.
"""
from functools import lru_cache

ACC = {"acc3", "aclr", "accr", "acc2", "acr"}


def classical(m, k, n, acc):
    return dict(mults=m * k * n, adds=m * n * (k - 1) + (m * n if acc else 0), peak=0,
                total=0, moves=0)


def _z():
    return dict(mults=0, adds=0, peak=0, total=0, moves=0)


def make_evaluator(cutoff):
    @lru_cache(maxsize=None)
    def sched(name, m, k, n):
        acc = name in ACC
        if min(m, k, n) <= cutoff:
            return classical(m, k, n, acc)
        m2, k2, n2 = m // 2, k // 2, n // 2
        sq = n2 * n2
        r = _z()
        if name == "std2":
            s = sched("std2", m2, k2, n2)
            r["mults"] = 7 * s["mults"]
            r["adds"] = 7 * s["adds"] + 4 * m2 * k2 + 4 * k2 * n2 + 7 * m2 * n2
            r["moves"] = 7 * s["moves"]
            w = m2 * max(k2, n2) + k2 * n2
            r["peak"] = w + s["peak"]
            r["total"] = w + 7 * s["total"]
        elif name == "acc3":
            sa, sp = sched("acc3", m2, k2, n2), sched("std2", m2, k2, n2)
            r["mults"] = 5 * sa["mults"] + 2 * sp["mults"]
            r["adds"] = 5 * sa["adds"] + 2 * sp["adds"] + 4 * m2 * k2 + 4 * k2 * n2 + 6 * m2 * n2
            r["moves"] = 5 * sa["moves"] + 2 * sp["moves"]
            w = m2 * k2 + k2 * n2 + m2 * n2
            r["peak"] = w + max(sa["peak"], sp["peak"])
            r["total"] = w + 5 * sa["total"] + 2 * sp["total"]
        elif name == "ip":
            s = sched("ip", m2, k2, n2)
            r["mults"] = 7 * s["mults"]
            r["adds"] = 7 * s["adds"] + 15 * sq
        elif name in ("ovl", "ovr"):
            s, ipc = sched(name, m2, k2, n2), sched("ip", m2, k2, n2)
            r["mults"] = 4 * s["mults"] + 3 * ipc["mults"]
            r["adds"] = 4 * s["adds"] + 3 * ipc["adds"] + 15 * sq
            r["peak"] = sq + max(s["peak"], ipc["peak"])
            r["total"] = sq + 4 * s["total"]
        elif name == "ovl2":
            so, sr, ipc = sched("ovl", m2, k2, n2), sched("ovr", m2, k2, n2), sched("ip", m2, k2, n2)
            r["mults"] = 4 * so["mults"] + sr["mults"] + 2 * ipc["mults"]
            r["adds"] = 4 * so["adds"] + sr["adds"] + 2 * ipc["adds"] + 15 * sq
            r["moves"] = 2 * sq + 4 * so["moves"] + sr["moves"]
            r["peak"] = sq + max(so["peak"], sr["peak"], ipc["peak"])
            r["total"] = sq + 4 * so["total"] + sr["total"]
        elif name == "aclr":
            s, ipc = sched("aclr", m2, k2, n2), sched("ip", m2, k2, n2)
            r["mults"] = 4 * s["mults"] + 3 * ipc["mults"]
            r["adds"] = 4 * s["adds"] + 3 * ipc["adds"] + 17 * sq
            r["peak"] = 2 * sq + max(s["peak"], ipc["peak"])
            r["total"] = 2 * sq + 4 * s["total"]
        elif name == "accr":
            s, ovr, ipc = sched("accr", m2, k2, n2), sched("ovr", m2, k2, n2), sched("ip", m2, k2, n2)
            r["mults"] = 4 * s["mults"] + 2 * ovr["mults"] + ipc["mults"]
            r["adds"] = 4 * s["adds"] + 2 * ovr["adds"] + ipc["adds"] + 17 * sq
            r["peak"] = 2 * sq + max(s["peak"], ovr["peak"], ipc["peak"])
            r["total"] = 2 * sq + 4 * s["total"] + 2 * ovr["total"]
        elif name == "acc2":
            s, w = sched("acc2", m2, k2, n2), sched("std2", m2, k2, n2)
            lr, rr = sched("aclr", m2, k2, n2), sched("accr", m2, k2, n2)
            r["mults"] = 4 * s["mults"] + w["mults"] + lr["mults"] + rr["mults"]
            r["adds"] = 4 * s["adds"] + w["adds"] + lr["adds"] + rr["adds"] + 17 * sq
            r["peak"] = 2 * sq + max(s["peak"], w["peak"], lr["peak"], rr["peak"])
            r["total"] = 2 * sq + 4 * s["total"] + w["total"] + lr["total"] + rr["total"]
        elif name == "acr":
            s, w = sched("acr", m2, k2, n2), sched("std2", m2, k2, n2)
            r["mults"] = 5 * s["mults"] + 2 * w["mults"]
            r["adds"] = 5 * s["adds"] + 2 * w["adds"] + 4 * m2 * k2 + 4 * k2 * n2 + 8 * m2 * n2
            words = max(m2, k2) * n2 + m2 * k2
            r["peak"] = words + max(s["peak"], w["peak"])
            r["total"] = words + 5 * s["total"] + 2 * w["total"]
        else:
            raise KeyError("expected_costs: unknown variant " + name)
        return r

    @lru_cache(maxsize=None)
    def ipmm(n, k):
        if n <= cutoff:
            return classical(n, k, n, False)
        s, q = n // 2, 2 * k // n
        w, wa, rec = sched("std2", s, s, s), sched("acc3", s, s, s), ipmm(s, k)
        r = _z()
        r["mults"] = 3 * w["mults"] + 3 * (q - 1) * wa["mults"] + rec["mults"]
        r["adds"] = 3 * w["adds"] + 3 * (q - 1) * wa["adds"] + rec["adds"]
        return r

    return sched, ipmm


def parse_blocked(v):
    if not v.startswith("blocked_acc_t"):
        return None
    rest = v[len("blocked_acc_t"):]
    i = 0
    while i < len(rest) and rest[i].isdigit():
        i += 1
    if i == 0:
        return None
    t = int(rest[:i])
    tail = rest[i:]
    if tail == "":
        return t, "acc3"
    if tail == "_acc2":
        return t, "acc2"
    return None


def expected_costs(variant, m, k, n, cutoff):
    sched, ipmm = make_evaluator(cutoff)
    if variant == "classic":
        c = classical(m, k, n, False)
    elif variant == "ipmm":
        c = ipmm(n, k)
    elif variant == "ipovmm":
        m0, k0 = m // n, k // n
        w, o, a = sched("std2", n, n, n), sched("ovl", n, n, n), sched("acc3", n, n, n)
        c = _z()
        c["mults"] = w["mults"] + (m0 - 1) * o["mults"] + (k0 - 1) * m0 * a["mults"]
        c["adds"] = w["adds"] + (m0 - 1) * o["adds"] + (k0 - 1) * m0 * a["adds"]
        c["moves"] = (m0 - 1) * o["moves"]
    elif variant == "iprect":
        # builder composition for k <= min(m, n) (config 3): squares of side k,
        # std2 / ovl / ovr / ip with scratch carved from unwritten C blocks.
        s = k
        mb, nb = m // s, n // s
        w, o, r_, ipc = (sched(v, s, s, s) for v in ("std2", "ovl", "ovr", "ip"))
        c = _z()
        # blocks (i<mb-1, j<nb-1) std2; last block column (A_i's last use) ovl;
        # last block row (B_j's last use) ovr; the final block ip.
        parts = [w] * ((mb - 1) * (nb - 1)) + [o] * (mb - 1) + [r_] * (nb - 1) + [ipc]
        for p in parts:
            c["mults"] += p["mults"]
            c["adds"] += p["adds"]
            c["moves"] += p["moves"]
    elif parse_blocked(variant):
        t, base = parse_blocked(variant)
        s = n // t
        chunk = 2 * (s * s - 1) // 3 if base == "acc2" else s * s
        b = sched(base, s, s, s)
        calls = t * t * t
        c = dict(mults=calls * b["mults"], adds=calls * b["adds"], moves=calls * b["moves"],
                 peak=chunk, total=chunk)
    else:
        c = sched(variant, m, k, n)
    return dict(mults=c["mults"], adds=c["adds"], peak_extra_words=c["peak"],
                total_alloc_words=c["total"], word_moves=c["moves"])
