// Builtin Winograd schedules (paper Tables 1-8) in the compact notation of
// wm_schedule.h.  Row numbers and the paper's value labels are given in the
// trailing comments so each line can be checked against the reference texts
// (/root/reference/proj/include/winomem/schedule.hpp:692-1000).
#include "wm_schedule.h"

#include <map>
#include <sstream>

namespace wm {

const char* slot_name(Slot s) {
    static const char* n[] = {"A11", "A12", "A21", "A22", "B11", "B12", "B21", "B22",
                              "C11", "C12", "C21", "C22", "X",   "Y",   "Z"};
    return n[static_cast<int>(s)];
}

std::uint64_t eval_dim(Dim d, std::uint64_t m, std::uint64_t k, std::uint64_t n) {
    switch (d) {
        case Dim::M2: return m / 2;
        case Dim::K2: return k / 2;
        case Dim::N2: return n / 2;
        case Dim::MaxK2N2: return (k > n ? k : n) / 2;
        case Dim::MaxM2K2: return (m > k ? m : k) / 2;
    }
    return 0;
}

const char* contract_name(Contract c) {
    switch (c) {
        case Contract::ReadOnly: return "read-only";
        case Contract::OverwriteA: return "overwrite-A";
        case Contract::OverwriteB: return "overwrite-B";
        case Contract::OverwriteBoth: return "overwrite-both";
    }
    return "?";
}

bool slot_writable(Slot s, Contract c) {
    switch (slot_role(s)) {
        case Role::InputA: return c == Contract::OverwriteA || c == Contract::OverwriteBoth;
        case Role::InputB: return c == Contract::OverwriteB || c == Contract::OverwriteBoth;
        default: return true;
    }
}

int Schedule::product_count() const {
    int c = 0;
    for (const auto& i : ins) c += i.kind == Instr::Product;
    return c;
}

namespace {

Slot parse_slot(const std::string& t, int line) {
    for (int i = 0; i < NSLOT; ++i)
        if (t == slot_name(static_cast<Slot>(i))) return static_cast<Slot>(i);
    fail(E_PARSE, "line " + std::to_string(line) + ": unknown slot '" + t + "'");
}

struct Cursor {
    std::vector<std::string> tok;
    std::size_t i = 0;
    bool done() const { return i >= tok.size(); }
    const std::string& peek() const {
        static const std::string e;
        return done() ? e : tok[i];
    }
    std::string next() { return done() ? std::string() : tok[i++]; }
};

// [+|-] [a|b] -- the sign/scalar prefix of one term
Sym parse_sym(Cursor& c, bool first, int line) {
    Sym s;
    if (c.peek() == "+" || c.peek() == "-") {
        s.neg = c.next() == "-";
    } else if (!first) {
        fail(E_PARSE, "line " + std::to_string(line) + ": expected + or - between terms");
    }
    if (c.peek() == "a") {
        s.sym = 1;
        c.next();
    } else if (c.peek() == "b") {
        s.sym = 2;
        c.next();
    }
    return s;
}

}  // namespace

Schedule compile_program(const std::string& name, Contract contract, bool accumulating,
                         bool square_only, const std::vector<TempDecl>& temps,
                         const char* program) {
    Schedule s;
    s.name = name;
    s.contract = contract;
    s.accumulating = accumulating;
    s.square_only = square_only;
    s.temps = temps;
    std::istringstream is(program);
    std::string raw;
    int line = 0;
    while (std::getline(is, raw)) {
        ++line;
        auto hash = raw.find('#');
        if (hash != std::string::npos) raw = raw.substr(0, hash);
        Cursor c;
        {
            std::istringstream ls(raw);
            std::string t;
            while (ls >> t) c.tok.push_back(t);
        }
        if (c.done()) continue;
        Instr in;
        in.dst = parse_slot(c.next(), line);
        if (c.next() != "=") fail(E_PARSE, "line " + std::to_string(line) + ": expected '='");
        std::string tag;
        if (!c.peek().empty() && c.peek().back() == ':') {
            tag = c.next();
            tag.pop_back();
        }
        in.s0 = parse_sym(c, true, line);
        in.o0 = parse_slot(c.next(), line);
        if (c.peek() == "*") {
            c.next();
            in.kind = Instr::Product;
            in.o1 = parse_slot(c.next(), line);
            if (!c.done()) {
                in.has_acc = true;
                in.sacc = parse_sym(c, false, line);
                in.oacc = parse_slot(c.next(), line);
            }
            in.tag = tag.empty() ? (in.has_acc ? "acc3" : "std2") : tag;
        } else if (c.done()) {
            in.kind = Instr::Copy1;
        } else {
            in.kind = Instr::Add2;
            in.s1 = parse_sym(c, false, line);
            in.o1 = parse_slot(c.next(), line);
        }
        if (!c.done()) fail(E_PARSE, "line " + std::to_string(line) + ": trailing tokens");
        // a schedule may only write the slots its contract allows (schedule.hpp:587-590)
        if (!slot_writable(in.dst, contract))
            fail(E_CONTRACT_VIOLATION, name + ": writing " + slot_name(in.dst) +
                                           " violates contract " + contract_name(contract));
        if (slot_role(in.dst) == Role::Temporary) {
            bool declared = false;
            for (const auto& t : s.temps) declared |= t.slot == in.dst;
            if (!declared) s.temps.push_back({in.dst, Dim::N2, Dim::N2});
        }
        s.ins.push_back(in);
    }
    return s;
}

namespace {

// ---- Table 1: C <- AB, 2 temporaries, read-only inputs (schedule.hpp:692-720)
const char* kStd2 = R"(
X = A11 - A21            # 1  S3
Y = B22 - B12            # 2  T3
C21 = X * Y              # 3  P7
X = A21 + A22            # 4  S1
Y = B12 - B11            # 5  T1
C22 = X * Y              # 6  P5
X = X - A11              # 7  S2 = S1 - A11
Y = B22 - Y              # 8  T2 = B22 - T1
C12 = X * Y              # 9  P6
X = A12 - X              # 10 S4 = A12 - S2
C11 = X * B22            # 11 P3
X = A11 * B11            # 12 P1
C12 = X + C12            # 13 U2 = P1 + P6
C21 = C12 + C21          # 14 U3 = U2 + P7
C12 = C12 + C22          # 15 U4 = U2 + P5
C22 = C21 + C22          # 16 U7 = U3 + P5
C12 = C12 + C11          # 17 U5 = U4 + P3
Y = Y - B21              # 18 T4 = T2 - B21
C11 = A22 * Y            # 19 P4
C21 = C21 - C11          # 20 U6 = U3 - P4
C11 = A12 * B21          # 21 P2
C11 = X + C11            # 22 U1 = P1 + P2
)";

// ---- Table 2: C <- alpha AB + beta C, 3 temporaries (schedule.hpp:722-750)
const char* kAcc3 = R"(
X = A21 + A22            # 1  S1
Y = B12 - B11            # 2  T1
Z = a X * Y              # 3  P5 = alpha S1 T1
C22 = Z + b C22          # 4
C12 = Z + b C12          # 5
X = X - A11              # 6  S2
Y = B22 - Y              # 7  T2
Z = a A11 * B11          # 8  P1
C11 = Z + b C11          # 9
Z = a X * Y + Z          # 10 U2 = alpha S2 T2 + P1
C11 = a A12 * B21 + C11  # 11 U1
X = A12 - X              # 12 S4
Y = Y - B21              # 13 T4
C12 = a X * B22 + C12    # 14
C12 = Z + C12            # 15 U5 = U2 + C12
C21 = a A22 * Y - b C21  # 16 P4 = alpha A22 T4 - beta C21
X = A11 - A21            # 17 S3
Y = B22 - B12            # 18 T3
Z = a X * Y + Z          # 19 U3 = alpha S3 T3 + U2
C22 = Z + C22            # 20 U7
C21 = Z - C21            # 21 U6 = U3 - C21
)";

// ---- Table 3: C <- AB overwriting A and B, no temporary (schedule.hpp:752-778)
const char* kIp = R"(
C11 = A11 - A21          # 1  S3
A21 = A21 + A22          # 2  S1
C22 = B12 - B11          # 3  T1
B12 = B22 - B12          # 4  T3
C21 = ip: C11 * B12      # 5  P7 = S3 T3
C12 = A21 - A11          # 6  S2 = S1 - A11
C11 = ip: A11 * B11      # 7  P1
B11 = B22 - C22          # 8  T2 = B22 - T1
A11 = ip: A21 * C22      # 9  P5 = S1 T1
C22 = B11 - B21          # 10 T4 = T2 - B21
A21 = ip: A22 * C22      # 11 P4 = A22 T4
A22 = A12 - C12          # 12 S4 = A12 - S2
C22 = ip: C12 * B11      # 13 P6 = S2 T2
C22 = C11 + C22          # 14 U2 = P1 + P6
C12 = ip: A12 * B21      # 15 P2
C11 = C11 + C12          # 16 U1 = P1 + P2
C12 = C22 + A11          # 17 U4 = U2 + P5
C22 = C22 + C21          # 18 U3 = U2 + P7
C21 = C22 - A21          # 19 U6 = U3 - P4
C22 = C22 + A11          # 20 U7 = U3 + P5
A12 = ip: A22 * B22      # 21 P3 = S4 B22
C12 = C12 + A12          # 22 U5 = U4 + P3
)";

// ---- Table 4: C <- AB overwriting A, one temporary (schedule.hpp:780-807)
const char* kOvlHead = R"(
C22 = A11 - A21          # 1  S3
A21 = A21 + A22          # 2  S1
C12 = A21 - A11          # 3  S2 = S1 - A11
C21 = B12 - B11          # 4  T1
C11 = ovl: A11 * B11     # 5  P1
A11 = B22 - B12          # 6  T3
X = ip: C22 * A11        # 7  P7 = S3 T3
A11 = B22 - C21          # 8  T2 = B22 - T1
C22 = ip: A21 * C21      # 9  P5 = S1 T1
C21 = A12 - C12          # 10 S4 = A12 - S2
A21 = ovl: C21 * B22     # 11 P3 = S4 B22
C21 = ovl: C12 * A11     # 12 P6 = S2 T2
A11 = A11 - B21          # 13 T4 = T2 - B21
C21 = C11 + C21          # 14 U2 = P1 + P6
C12 = C21 + C22          # 15 U4 = U2 + P5
C21 = C21 + X            # 16 U3 = U2 + P7
C22 = C21 + C22          # 17 U7 = U3 + P5
C12 = C12 + A21          # 18 U5 = U4 + P3
)";
const char* kOvlTail = R"(
X = ovl: A12 * B21       # 19 P2
C11 = C11 + X            # 20 U1 = P1 + P2
A21 = ip: A22 * A11      # 21 P4 = A22 T4
C21 = C21 - A21          # 22 U6 = U3 - P4
)";
// ovl2 (schedule.hpp:812-841): A12 is backed up into A21 around the P2 call
// and the last product uses OvR, so only two blocks of A are clobbered.
const char* kOvl2Tail = R"(
A21 = A12                # 19 backup A12
X = ovl: A12 * B21       # 20 P2
A12 = A21                # 21 restore A12
C11 = C11 + X            # 22 U1 = P1 + P2
A21 = ovr: A22 * A11     # 23 P4 = A22 T4
C21 = C21 - A21          # 24 U6 = U3 - P4
)";

// ---- Table 5: C <- AB overwriting B, one temporary (schedule.hpp:843-870)
const char* kOvr = R"(
C22 = A11 - A21          # 1  S3
C21 = A21 + A22          # 2  S1
C12 = B12 - B11          # 3  T1
C11 = ovr: A11 * B11     # 4  P1
B11 = C21 - A11          # 5  S2 = S1 - A11
B12 = B22 - B12          # 6  T3
X = ip: C22 * B12        # 7  P7 = S3 T3
B12 = B22 - C12          # 8  T2 = B22 - T1
C22 = ip: C21 * C12      # 9  P5 = S1 T1
C12 = B12 - B21          # 10 T4 = T2 - B21
C21 = ovr: B11 * B12     # 11 P6 = S2 T2
B12 = ovr: A22 * C12     # 12 P4 = A22 T4
B11 = A12 - B11          # 13 S4 = A12 - S2
C21 = C11 + C21          # 14 U2 = P1 + P6
C12 = C21 + C22          # 15 U4 = U2 + P5
C21 = C21 + X            # 16 U3 = U2 + P7
C22 = C21 + C22          # 17 U7 = U3 + P5
C21 = C21 - B12          # 18 U6 = U3 - P4
B12 = ip: B11 * B22      # 19 P3 = S4 B22
C12 = C12 + B12          # 20 U5 = U4 + P3
B12 = ovr: A12 * B21     # 21 P2
C11 = C11 + B12          # 22 U1 = P1 + P2
)";

// ---- Table 6: C <- alpha AB + beta C overwriting A and B, 2 temporaries
// (schedule.hpp:872-902)
const char* kAclr = R"(
C22 = C22 - C12               # 1  Z1
X = A21 + A22                 # 2  S1
Y = B12 - B11                 # 3  T1
C21 = C21 - C22               # 4  Z2 = C21 - Z1
B12 = B22 - B12               # 5  T3
A21 = A11 - A21               # 6  S3
C22 = aclr: a A21 * B12 + b C22   # 7  P7 = alpha S3 T3 + beta Z1
A21 = X - A11                 # 8  S2 = S1 - A11
B12 = B22 - Y                 # 9  T2 = B22 - T1
C12 = aclr: a X * Y + b C12   # 10 P5
Y = ip: a A11 * B11           # 11 P1
X = B12 - B21                 # 12 T4 = T2 - B21
C21 = aclr: a A22 * X - b C21 # 13 P4 = alpha A22 T4 - beta Z2
A22 = A12 - A21               # 14 S4 = A12 - S2
X = ip: a A21 * B12           # 15 P6 = alpha S2 T2
C11 = aclr: a A12 * B21 + b C11   # 16 P2
C11 = Y + C11                 # 17 U1 = P1 + P2
X = Y + X                     # 18 U2 = P1 + P6
C22 = X + C22                 # 19 U3 = U2 + P7
X = X + C12                   # 20 U4 = U2 + P5
C21 = C22 - C21               # 21 U6 = U3 - P4
C22 = C22 + C12               # 22 U7 = U3 + P5
C12 = ip: a A22 * B22         # 23 P3 = alpha S4 B22
C12 = X + C12                 # 24 U5 = U4 + P3
)";

// ---- Table 7 (right-overwriting accumulation), 2 temporaries
// (schedule.hpp:904-934)
const char* kAccr = R"(
C22 = C22 - C12               # 1  Z1
X = B12 - B11                 # 2  T1
C21 = C21 - C22               # 3  Z2
B12 = B22 - B12               # 4  T3
Y = A11 - A21                 # 5  S3
C22 = accr: a Y * B12 + b C22 # 6  P7
Y = A21 + A22                 # 7  S1
B12 = B22 - X                 # 8  T2 = B22 - T1
C12 = accr: a Y * X + b C12   # 9  P5
X = B12 - B21                 # 10 T4 = T2 - B21
C21 = accr: a A22 * X - b C21 # 11 P4
X = ovr: a A11 * B11          # 12 P1
C11 = accr: a A12 * B21 + b C11   # 13 P2
Y = Y - A11                   # 14 S2 = S1 - A11
B21 = ovr: a Y * B12          # 15 P6 = alpha S2 T2
Y = A12 - Y                   # 16 S4 = A12 - S2
B21 = X + B21                 # 17 U2 = P1 + P6
C22 = B21 + C22               # 18 U3 = U2 + P7
B21 = B21 + C12               # 19 U4 = U2 + P5
C21 = C22 - C21               # 20 U6 = U3 - P4
C11 = X + C11                 # 21 U1 = P1 + P2
C22 = C22 + C12               # 22 U7 = U3 + P5
C12 = ip: a Y * B22           # 23 P3 = alpha S4 B22
C12 = B21 + C12               # 24 U5 = U4 + P3
)";

// ---- Table 7 hybrid: C <- alpha AB + beta C with constant inputs, 2 temporaries
// (schedule.hpp:939-969); rows 19 and 24 accumulate into the destination's
// current value and T2 is recomputed on purpose (rows 21-23).
const char* kAcc2 = R"(
C22 = C22 - C12               # 1  Z1
C12 = C12 - C21               # 2  Z3
X = A21 + A22                 # 3  S1
Y = B12 - B11                 # 4  T1
C12 = acc2: a X * Y + b C12   # 5  P5 = alpha S1 T1 + beta Z3
X = X - A11                   # 6  S2
Y = B22 - Y                   # 7  T2
C21 = acc2: a X * Y + b C21   # 8  P6
X = A12 - X                   # 9  S4
C22 = C12 + b C22             # 10 W1 = P5 + beta Z1
C12 = acc2: a X * B22 + C12   # 11 P3 = alpha S4 B22 + P5
X = a A11 * B11               # 12 P1
C21 = C21 + X                 # 13 U2 = P6 + P1
C11 = acc2: a A12 * B21 + b C11   # 14 P2
C11 = X + C11                 # 15 U1 = P1 + P2
C12 = C21 + C12               # 16 U5 = U2 + P3
X = A11 - A21                 # 17 S3
Y = B22 - B12                 # 18 T3
C21 = aclr: a X * Y + C21     # 19 U3 = alpha S3 T3 + U2
C22 = C21 + C22               # 20 U7 = U3 + W1
Y = B12 - B11                 # 21 T1'
Y = B22 - Y                   # 22 T2'
Y = Y - B21                   # 23 T4
C21 = accr: - a A22 * Y + C21 # 24 U6 = -alpha A22 T4 + U3
)";

// ---- Table 8: rectangular accumulation overwriting B (schedule.hpp:971-1000)
const char* kAcr = R"(
C22 = C22 - C12               # 1  Z1
X = B12 - B11                 # 2  T1
C21 = C21 - C22               # 3  Z2
B12 = B22 - B12               # 4  T3
Y = A11 - A21                 # 5  S3
C22 = acr: a Y * B12 + b C22  # 6  P7
Y = A21 + A22                 # 7  S1
B12 = B22 - X                 # 8  T2
C12 = acr: a Y * X + b C12    # 9  P5
X = B12 - B21                 # 10 T4
C21 = acr: a A22 * X - b C21  # 11 P4
X = a A11 * B11               # 12 P1
C11 = acr: a A12 * B21 + b C11    # 13 P2
C11 = X + C11                 # 14 U1
Y = Y - A11                   # 15 S2
X = acr: a Y * B12 + X        # 16 U2 = alpha S2 T2 + P1
C22 = X + C22                 # 17 U3 = U2 + P7
C21 = C22 - C21               # 18 U6 = U3 - P4
C22 = C22 + C12               # 19 U7 = U3 + P5
X = X + C12                   # 20 U4 = U2 + P5
Y = A12 - Y                   # 21 S4
C12 = a Y * B22               # 22 P3
C12 = X + C12                 # 23 U5 = U4 + P3
)";

std::map<std::string, Schedule> make_catalog() {
    using D = Dim;
    using C = Contract;
    std::map<std::string, Schedule> m;
    m["std2"] = compile_program("std2", C::ReadOnly, false, false,
                                {{SX, D::M2, D::MaxK2N2}, {SY, D::K2, D::N2}}, kStd2);
    m["acc3"] = compile_program("acc3", C::ReadOnly, true, false,
                                {{SX, D::M2, D::K2}, {SY, D::K2, D::N2}, {SZ, D::M2, D::N2}},
                                kAcc3);
    m["ip"] = compile_program("ip", C::OverwriteBoth, false, true, {}, kIp);
    m["ovl"] = compile_program("ovl", C::OverwriteA, false, true, {{SX, D::N2, D::N2}},
                               (std::string(kOvlHead) + kOvlTail).c_str());
    m["ovl2"] = compile_program("ovl2", C::OverwriteA, false, true, {{SX, D::N2, D::N2}},
                                (std::string(kOvlHead) + kOvl2Tail).c_str());
    m["ovr"] = compile_program("ovr", C::OverwriteB, false, true, {{SX, D::N2, D::N2}}, kOvr);
    m["aclr"] = compile_program("aclr", C::OverwriteBoth, true, true,
                                {{SX, D::N2, D::N2}, {SY, D::N2, D::N2}}, kAclr);
    m["accr"] = compile_program("accr", C::OverwriteB, true, true,
                                {{SX, D::N2, D::N2}, {SY, D::N2, D::N2}}, kAccr);
    m["acc2"] = compile_program("acc2", C::ReadOnly, true, true,
                                {{SX, D::N2, D::N2}, {SY, D::N2, D::N2}}, kAcc2);
    m["acr"] = compile_program("acr", C::OverwriteB, true, false,
                               {{SX, D::MaxM2K2, D::N2}, {SY, D::M2, D::K2}}, kAcr);
    return m;
}

}  // namespace

const std::vector<std::string>& builtin_names() {
    static const std::vector<std::string> n = {"std2", "acc3", "ip",   "ovl",  "ovl2",
                                               "ovr",  "aclr", "accr", "acc2", "acr"};
    return n;
}

bool is_builtin(const std::string& name) {
    for (const auto& n : builtin_names())
        if (n == name) return true;
    return false;
}

const Schedule& builtin(const std::string& name) {
    static const std::map<std::string, Schedule> catalog = make_catalog();
    auto it = catalog.find(name);
    if (it == catalog.end()) fail(E_UNKNOWN_SCHEDULE, "unknown schedule: " + name);
    return it->second;
}

}  // namespace wm
