"""Generate the schedule-specific fused post/pre-addition kernels.

Every builtin schedule (csrc/wm_schedule.cpp) contains runs of consecutive
block additions with no product between them -- the S_i / T_i pre-additions
and the U_i post-addition chains of the paper's tables.  Executed one by one,
a run of r additions moves 3r blocks through HBM.  Fused, each distinct slot
is read once (if it is read before it is written) and written once (its final
value): e.g. std2 rows 13-18 (U2, U3, U4, U7, U5, T4) go from 18 block passes
to 11.

This script parses the schedule programs out of wm_schedule.cpp (the single
source of truth), finds every maximal run, and writes csrc/wm_fused_gen.cuh: one
kernel per run whose body is the run's dataflow over named registers (the slot
-> view binding and the +/-/alpha/beta scalars stay runtime parameters), plus
the table the lowering pass uses to match planned operations against runs.
Run automatically by build.py.
"""
from __future__ import annotations

import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "wm_schedule.cpp")
OUT = os.path.join(HERE, "csrc", "wm_fused_gen.cuh")

SLOTS = ["A11", "A12", "A21", "A22", "B11", "B12", "B21", "B22", "C11", "C12", "C21", "C22",
         "X", "Y", "Z"]
SLOT_ENUM = {s: e for s, e in zip(SLOTS, ["A11", "A12", "A21", "A22", "B11", "B12", "B21",
                                          "B22", "C11", "C12", "C21", "C22", "SX", "SY", "SZ"])}


def programs():
    text = open(SRC).read()
    consts = dict(re.findall(r'const char\* (k\w+) = R"\((.*?)\)";', text, flags=re.S))
    return {
        "std2": consts["kStd2"], "acc3": consts["kAcc3"], "ip": consts["kIp"],
        "ovl": consts["kOvlHead"] + consts["kOvlTail"],
        "ovl2": consts["kOvlHead"] + consts["kOvl2Tail"],
        "ovr": consts["kOvr"], "aclr": consts["kAclr"], "accr": consts["kAccr"],
        "acc2": consts["kAcc2"], "acr": consts["kAcr"],
    }


def parse(prog):
    """-> list of (row, kind, dst, operands) with kind in add/copy/product
    (a product's operands are its two factor slots)."""
    out = []
    row = 0
    for raw in prog.splitlines():
        line = raw.split("#")[0].strip()
        if not line:
            continue
        row += 1
        toks = line.split()
        dst = toks[0]
        rhs = toks[2:]
        if rhs and rhs[0].endswith(":"):
            rhs = rhs[1:]
        if "*" in rhs:
            k = rhs.index("*")
            out.append((row, "product", dst, [rhs[k - 1].lstrip("("), rhs[k + 1].rstrip(")")]))
            continue
        ops = [t for t in rhs if t in SLOTS]
        out.append((row, "add" if len(ops) == 2 else "copy", dst, ops))
    return out


def runs(ins):
    res, cur = [], []
    for r in ins:
        if r[1] == "product":
            if len(cur) >= 2:
                res.append(cur)
            cur = []
        else:
            cur.append(r)
    if len(cur) >= 2:
        res.append(cur)
    return res


def fold_remainders(ins):
    """Runs left behind when a leaf frame folds the additions producing its
    operands into its prep (wm_runtime.cu plan_folds): for every run followed by
    a product, the last writer of each factor slot may move into the product if
    no later instruction of the run reads or writes its destination or writes
    its sources.  Returns the contiguous remainders of >= 2 instructions."""
    out = []
    cur = []
    for r in ins:
        if r[1] != "product":
            cur.append(r)
            continue
        run, cur = cur, []
        if not run:
            continue
        folded = []
        for slot in r[3]:
            last = max((i for i, x in enumerate(run) if x[2] == slot), default=None)
            if last is None or last in folded:
                continue
            f = run[last]
            ok = all(f[2] not in x[3] and x[2] != f[2] and x[2] not in f[3]
                     for x in run[last + 1:])
            if ok:
                folded.append(last)
        if len(folded) == 2:  # the two folded instructions are computed together
            a, b = (run[i] for i in folded)
            if a[2] in b[3] or b[2] in a[3]:
                folded = folded[:1]
        rest = [x for i, x in enumerate(run) if i not in folded]
        if folded and len(rest) >= 2 and rest[-1][0] - rest[0][0] == len(rest) - 1:
            out.append(rest)
    return out


def main():
    groups = []
    for name, prog in programs().items():
        ins = parse(prog)
        seen = set()
        for run in runs(ins) + fold_remainders(ins):
            key = (run[0][0], len(run))
            if key in seen:
                continue
            seen.add(key)
            slots, loads, stores = [], [], []
            for (_, _, dst, ops) in run:
                for s in ops:
                    if s not in slots:
                        slots.append(s)
                        loads.append(s)
                if dst not in slots:
                    slots.append(dst)
                if dst not in stores:
                    stores.append(dst)
            groups.append(dict(sched=name, row0=run[0][0], row1=run[-1][0], run=run,
                               slots=slots, loads=loads, stores=stores))
    maxs = max(len(g["slots"]) for g in groups)
    maxi = max(len(g["run"]) for g in groups)
    L = []
    w = L.append
    w("// GENERATED by gen_fusion.py from wm_schedule.cpp -- do not edit.")
    w("// One fused elementwise kernel per maximal run of block additions of each")
    w("// builtin schedule (schedule, rows row0..row1).")
    w("#pragma once")
    w("#include <cstdint>")
    w('#include "wm_device.h"')
    w("namespace wm {")
    w("namespace fused {")
    w(f"constexpr int kMaxSlots = {maxs};")
    w(f"constexpr int kMaxIns = {maxi};")
    w(f"constexpr int kNumGroups = {len(groups)};")
    w("struct GroupDesc {")
    w("    const char* sched;")
    w("    int row0, row1, nslots, nins, nload, nstore;")
    w("    // per instruction: dst slot, a slot, b slot (-1 for copies)")
    w("    int ins[kMaxIns][3];")
    w("};")
    w("static const GroupDesc kGroups[kNumGroups] = {")
    for g in groups:
        idx = {s: i for i, s in enumerate(g["slots"])}
        ins = []
        for (_, kind, dst, ops) in g["run"]:
            a = idx[ops[0]]
            b = idx[ops[1]] if kind == "add" else -1
            ins.append("{%d, %d, %d}" % (idx[dst], a, b))
        ins += ["{-1, -1, -1}"] * (maxi - len(ins))
        w('    {"%s", %d, %d, %d, %d, %d, %d, {%s}},' % (
            g["sched"], g["row0"], g["row1"], len(g["slots"]), len(g["run"]), len(g["loads"]),
            len(g["stores"]), ", ".join(ins)))
    w("};")
    w("")
    w("struct GroupParams {")
    w("    double* v[kMaxSlots];")
    w("    std::uint64_t ld[kMaxSlots];")
    w("    // instruction j: s_dst = ca[j] * s_a + cb[j] * s_b (cb = 0 for a one-term copy);")
    w("    // +-1 / 0 coefficients stay unreduced (lazy), bit j of `gen` marks a general")
    w("    // scalar whose result is reduced at once (MODP)")
    w("    double ca[kMaxIns], cb[kMaxIns];")
    w("    std::uint32_t gen;")
    w("    std::uint32_t rows, cols;  // cols even, all views 16-B aligned")
    w("    double p, pinv;")
    w("};")
    w("")
    w("// lazy modular reduction (wm_apply.cuh): a run's intermediate values stay")
    w("// unreduced (exact integers in float64); every stored slot is canonicalised once")
    w("template <bool REAL>")
    w("__device__ __forceinline__ double canon(double v, double p, double pinv);")
    w("template <bool REAL>")
    w("__device__ __forceinline__ double lin(const GroupParams& G, int j, double a, double b) {")
    w("    const double v = fma(G.ca[j], a, G.cb[j] * b);  // branch-free: no per-mode switch")
    w("    return (!REAL && ((G.gen >> j) & 1u)) ? canon<REAL>(v, G.p, G.pinv) : v;")
    w("}")
    w("")
    w("// LDG: read-only path for slots nothing in the kernel writes")
    w("template <bool LDG>")
    w("__device__ __forceinline__ double2 gld(const double* p) {")
    w("    return LDG ? __ldg(reinterpret_cast<const double2*>(p)) : *reinterpret_cast<const double2*>(p);")
    w("}")
    w("")
    for gi, g in enumerate(groups):
        idx = {s: i for i, s in enumerate(g["slots"])}
        w(f"// {g['sched']} rows {g['row0']}-{g['row1']}: reads "
          f"{' '.join(g['loads'])}; writes {' '.join(g['stores'])}")
        w("template <bool REAL, bool LDG>")
        w(f"__device__ __forceinline__ void group_body_{gi}(const GroupParams& G, std::uint64_t r,"
          " std::uint64_t c) {")
        for s in g["loads"]:
            i = idx[s]
            w(f"    double2 s{i} = gld<LDG>(G.v[{i}] + r * G.ld[{i}] + c);")
        for s in g["slots"]:
            if s not in g["loads"]:
                w(f"    double2 s{idx[s]};")
        for j, (_, kind, dst, ops) in enumerate(g["run"]):
            d, a = idx[dst], idx[ops[0]]
            b = idx[ops[1]] if kind == "add" else a
            w(f"    s{d} = make_double2(lin<REAL>(G, {j}, s{a}.x, s{b}.x), "
              f"lin<REAL>(G, {j}, s{a}.y, s{b}.y));")
        for s in g["stores"]:
            i = idx[s]
            w(f"    *reinterpret_cast<double2*>(G.v[{i}] + r * G.ld[{i}] + c) = "
              f"make_double2(canon<REAL>(s{i}.x, G.p, G.pinv), canon<REAL>(s{i}.y, G.p, G.pinv));")
        w("}")
        w("")
    w("// one kernel per run (wm_kernels.cu instantiates k_group<REAL, G> for every G):")
    w("// each launch runs only its own compact body -- no dispatch switch, no jump table")
    w("template <bool REAL, int G>")
    w("struct GroupBody;")
    for gi in range(len(groups)):
        w(f"template <bool REAL> struct GroupBody<REAL, {gi}> {{")
        w("    static __device__ __forceinline__ void run(const GroupParams& P, std::uint64_t r,"
          " std::uint64_t c) {")
        w(f"        group_body_{gi}<REAL, true>(P, r, c);")
        w("    }")
        w("};")
    w("#define WM_FUSED_GROUP_IDS(X) " + " ".join(f"X({gi})" for gi in range(len(groups))))
    w("}  // namespace fused")
    w("}  // namespace wm")
    text = "\n".join(L) + "\n"
    if not os.path.exists(OUT) or open(OUT).read() != text:
        open(OUT, "w").write(text)
    return len(groups)


if __name__ == "__main__":
    print(main(), "groups ->", OUT)
