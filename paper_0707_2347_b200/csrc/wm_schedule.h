// Schedule IR and builtin catalog.
//
// A schedule is the ordered program of one Winograd frame over 15 symbolic
// slots (A11..A22, B11..B22, C11..C22 and the temporaries X, Y, Z) -- the
// representation of /root/reference/proj/include/winomem/schedule.hpp:45-239.
// The builtins are the paper's Tables 1-8 (PAPER.md; reference texts
// schedule.hpp:692-1000), re-encoded in the compact notation parsed by
// `compile_program` below.  Labels (S1, T3, P5, U2, ...) are documentation in the
// reference; only slot locations drive execution, so they are kept as comments.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "wm_types.h"

namespace wm {

enum Slot : std::uint8_t {
    A11, A12, A21, A22, B11, B12, B21, B22, C11, C12, C21, C22, SX, SY, SZ, NSLOT
};
const char* slot_name(Slot s);

enum class Role { InputA, InputB, InoutC, Temporary };
inline Role slot_role(Slot s) {
    int i = static_cast<int>(s);
    if (i < 4) return Role::InputA;
    if (i < 8) return Role::InputB;
    if (i < 12) return Role::InoutC;
    return Role::Temporary;
}

// schedule.hpp:72-107: temporary dimensions over half-sizes
enum class Dim : std::uint8_t { M2, K2, N2, MaxK2N2, MaxM2K2 };
std::uint64_t eval_dim(Dim d, std::uint64_t m, std::uint64_t k, std::uint64_t n);

// schedule.hpp:185-211
enum class Contract : std::uint8_t { ReadOnly, OverwriteA, OverwriteB, OverwriteBoth };
const char* contract_name(Contract c);
bool slot_writable(Slot s, Contract c);

// scalar symbol of a term: (+/-)(1 | alpha | beta)
struct Sym {
    bool neg = false;
    std::uint8_t sym = 0;  // 0 one, 1 alpha, 2 beta
};

struct Instr {
    enum Kind : std::uint8_t { Add2, Copy1, Product } kind = Add2;
    Slot dst = SX;
    // Add2: s0*o0 + s1*o1; Copy1: s0*o0; Product: s0 * o0 * o1 (+ s1*o1acc)
    Sym s0, s1;
    Slot o0 = SX, o1 = SX;
    bool has_acc = false;
    Sym sacc;
    Slot oacc = SX;
    std::string tag;  // recursion target for products ("std2", "ip", ..., "classic")
};

struct TempDecl {
    Slot slot;
    Dim rows, cols;
};

struct Schedule {
    std::string name;
    Contract contract = Contract::ReadOnly;
    bool accumulating = false;
    bool square_only = true;
    std::vector<TempDecl> temps;
    std::vector<Instr> ins;
    int product_count() const;
};

// The builtin catalog (schedule.hpp:1002-1028); throws E_UNKNOWN_SCHEDULE.
const Schedule& builtin(const std::string& name);
const std::vector<std::string>& builtin_names();
bool is_builtin(const std::string& name);

// Compact program notation (one instruction per line):
//   DST = [+|-] [a|b] SLOT (+|-) [a|b] SLOT          two-term addition
//   DST = [+|-] [a|b] SLOT                            copy / negate / scale
//   DST = [TAG:] [+|-] [a|b] SLOT * SLOT [(+|-) [a|b] DST]
// An untagged product recurses into std2 (no accumulator) or acc3 (with one),
// the DSL default of schedule.hpp:583-585.
Schedule compile_program(const std::string& name, Contract c, bool accumulating,
                         bool square_only, const std::vector<TempDecl>& temps,
                         const char* program);

// Schedule DSL (wm_dsl.cpp; the reference's text form, schedule.hpp:261-684):
// parse_schedule throws E_PARSE / E_CONTRACT_VIOLATION; render_schedule emits
// text that parses back to the same schedule (labels V1, V2, ...).
Schedule parse_schedule(const std::string& text);
std::string render_schedule(const Schedule& s);
bool same_schedule(const Schedule& a, const Schedule& b);

}  // namespace wm
