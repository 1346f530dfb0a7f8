// Schedule DSL: the text form of a schedule that the reference reads from files
// and emits from its pebble search (schedule.hpp:261-684), parsed into and
// rendered from this build's Schedule IR, so that hand-written or generated
// schedules run on the device (run_parsed_schedule, executor.hpp:304-342).
//
//   schedule NAME
//   contract read-only | overwrite-A | overwrite-B | overwrite-both
//   accumulating true | false
//   shape square | rectangular
//   temp SLOT RDIM CDIM          (m/2, k/2, n/2, max(k/2,n/2), max(m/2,k/2))
//   IDX: LABEL = RHS @ SLOT
//
// RHS terms are [+|-] [alpha*|beta*|INT*] followed by an operand, a product
// `L*R`, or a recursion call `Tag(inner terms)`.  Operands name a slot or the
// label of an earlier result (which resolves to the slot it was written to).
// Untagged products recurse into std2 (no accumulator term) or acc3.  The
// device executes scalars +-1, alpha and beta; an integer literal other than 1
// is rejected at parse time.
#include <cctype>
#include <map>
#include <sstream>

#include "wm_schedule.h"

namespace wm {
namespace {

struct Tok {
    enum Kind { Ident, Int, Sym, End } kind = End;
    std::string text;
    long long value = 0;
};

class Lexer {
  public:
    Lexer(const std::string& s, int line) : s_(s), line_(line) {}
    Tok peek() {
        if (!has_) cur_ = lex(), has_ = true;
        return cur_;
    }
    Tok next() {
        Tok t = peek();
        has_ = false;
        return t;
    }
    [[noreturn]] void error(const std::string& m) const {
        fail(E_PARSE, "line " + std::to_string(line_) + ": " + m);
    }
    int line() const { return line_; }

  private:
    Tok lex() {
        while (pos_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[pos_]))) ++pos_;
        if (pos_ >= s_.size() || s_[pos_] == '#') return {};
        const char c = s_[pos_];
        const std::size_t b = pos_;
        if (std::isdigit(static_cast<unsigned char>(c))) {
            while (pos_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[pos_]))) ++pos_;
            const std::string t = s_.substr(b, pos_ - b);
            return {Tok::Int, t, std::stoll(t)};
        }
        if (std::isalpha(static_cast<unsigned char>(c))) {
            while (pos_ < s_.size() && (std::isalnum(static_cast<unsigned char>(s_[pos_])) ||
                                        s_[pos_] == '_' || s_[pos_] == '\''))
                ++pos_;
            return {Tok::Ident, s_.substr(b, pos_ - b), 0};
        }
        ++pos_;
        return {Tok::Sym, std::string(1, c), 0};
    }
    std::string s_;
    int line_;
    std::size_t pos_ = 0;
    Tok cur_;
    bool has_ = false;
};

// recursion tags (schedule.hpp:109-121) -> this build's schedule names
const char* const kTagNames[] = {"Classic", "Std2", "Acc3", "IP",   "OvL", "OvR",
                                 "AcLR",    "AccR", "Acc2", "AcR", "Self"};
const char* const kTagTargets[] = {"classic", "std2", "acc3", "ip",  "ovl", "ovr",
                                   "aclr",    "accr", "acc2", "acr", "self"};

const char* tag_target(const std::string& t) {
    for (int i = 0; i < 11; ++i)
        if (t == kTagNames[i]) return kTagTargets[i];
    return nullptr;
}

const char* tag_display(const std::string& target) {
    for (int i = 0; i < 11; ++i)
        if (target == kTagTargets[i]) return kTagNames[i];
    return nullptr;
}

bool slot_by_name(const std::string& t, Slot* out) {
    for (int i = 0; i < NSLOT; ++i)
        if (t == slot_name(static_cast<Slot>(i))) {
            *out = static_cast<Slot>(i);
            return true;
        }
    return false;
}

bool dim_by_name(const std::string& t, Dim* d) {
    if (t == "m/2") *d = Dim::M2;
    else if (t == "k/2") *d = Dim::K2;
    else if (t == "n/2") *d = Dim::N2;
    else if (t == "max(k/2,n/2)") *d = Dim::MaxK2N2;
    else if (t == "max(m/2,k/2)") *d = Dim::MaxM2K2;
    else return false;
    return true;
}

const char* dim_text(Dim d) {
    switch (d) {
        case Dim::M2: return "m/2";
        case Dim::K2: return "k/2";
        case Dim::N2: return "n/2";
        case Dim::MaxK2N2: return "max(k/2,n/2)";
        case Dim::MaxM2K2: return "max(m/2,k/2)";
    }
    return "?";
}

struct Term {
    Sym sym;
    bool is_prod = false;
    Slot a = SX, b = SX;
    std::string tag;            // recursion call (empty: none)
    std::vector<Term> inner;    // its terms
    bool scalar_outside = false;
};

using Labels = std::map<std::string, Slot>;

Slot resolve(const Labels& L, const std::string& t, const Lexer& lx) {
    auto it = L.find(t);
    if (it == L.end())
        fail(E_UNKNOWN_SLOT, "line " + std::to_string(lx.line()) + ": unknown operand '" + t + "'");
    return it->second;
}

std::vector<Term> parse_terms(const Labels& L, Lexer& lx) {
    std::vector<Term> out;
    bool first = true;
    for (;;) {
        Tok t = lx.peek();
        if (t.kind == Tok::End || (t.kind == Tok::Sym && (t.text == "@" || t.text == ")"))) break;
        Term term;
        if (t.kind == Tok::Sym && (t.text == "+" || t.text == "-")) {
            term.sym.neg = t.text == "-";
            lx.next();
        } else if (!first) {
            lx.error("expected '+' or '-' between terms");
        }
        first = false;
        Tok u = lx.peek();
        bool scaled = false;
        if (u.kind == Tok::Int) {
            if (u.value != 1) lx.error("integer scalars other than 1 are not supported on the device path");
            lx.next();
            scaled = true;
        } else if (u.kind == Tok::Ident && (u.text == "alpha" || u.text == "beta")) {
            term.sym.sym = u.text == "alpha" ? 1 : 2;
            lx.next();
            scaled = true;
        }
        if (scaled) {
            Tok star = lx.next();
            if (star.kind != Tok::Sym || star.text != "*") lx.error("expected '*' after scalar");
        }
        Tok id = lx.next();
        if (id.kind != Tok::Ident) lx.error("expected operand");
        const char* target = tag_target(id.text);
        Tok paren = lx.peek();
        if (target && paren.kind == Tok::Sym && paren.text == "(") {
            lx.next();
            term.tag = target;
            term.scalar_outside = scaled;
            term.inner = parse_terms(L, lx);
            Tok close = lx.next();
            if (close.kind != Tok::Sym || close.text != ")") lx.error("expected ')'");
        } else {
            term.a = resolve(L, id.text, lx);
            Tok star = lx.peek();
            if (star.kind == Tok::Sym && star.text == "*") {
                lx.next();
                Tok id2 = lx.next();
                if (id2.kind != Tok::Ident) lx.error("expected operand after '*'");
                term.b = resolve(L, id2.text, lx);
                term.is_prod = true;
            }
        }
        out.push_back(term);
    }
    return out;
}

bool parse_directive(Schedule& s, Lexer& lx, const std::string& raw) {
    const std::string kw = lx.peek().text;
    if (kw != "schedule" && kw != "contract" && kw != "accumulating" && kw != "shape" && kw != "temp")
        return false;
    lx.next();
    if (kw == "schedule") {
        s.name = lx.next().text;
    } else if (kw == "contract") {
        std::string v;
        for (Tok t = lx.next(); t.kind != Tok::End; t = lx.next()) v += t.text;
        if (v == "read-only") s.contract = Contract::ReadOnly;
        else if (v == "overwrite-A") s.contract = Contract::OverwriteA;
        else if (v == "overwrite-B") s.contract = Contract::OverwriteB;
        else if (v == "overwrite-both") s.contract = Contract::OverwriteBoth;
        else lx.error("unknown contract: " + v);
    } else if (kw == "accumulating") {
        const std::string v = lx.next().text;
        if (v != "true" && v != "false") lx.error("accumulating expects true|false");
        s.accumulating = v == "true";
    } else if (kw == "shape") {
        const std::string v = lx.next().text;
        if (v == "square") s.square_only = true;
        else if (v == "rectangular") s.square_only = false;
        else lx.error("shape expects square|rectangular");
    } else {
        std::istringstream ts(raw);
        std::string w, slot, rd, cd;
        ts >> w >> slot >> rd >> cd;
        Slot sl;
        Dim r, c;
        if (!slot_by_name(slot, &sl) || slot_role(sl) != Role::Temporary)
            lx.error("temp expects a temporary slot name");
        if (!dim_by_name(rd, &r) || !dim_by_name(cd, &c)) lx.error("bad temp dimension");
        s.temps.push_back({sl, r, c});
    }
    return true;
}

void parse_instruction(Schedule& s, Labels& L, Lexer& lx) {
    Tok idx = lx.next();
    if (idx.kind != Tok::Int) lx.error("expected instruction index");
    if (idx.value != static_cast<long long>(s.ins.size()) + 1)
        lx.error("instruction indices must be sequential from 1");
    Tok colon = lx.next();
    if (colon.kind != Tok::Sym || colon.text != ":") lx.error("expected ':'");
    Tok lbl = lx.next();
    if (lbl.kind != Tok::Ident) lx.error("expected result label");
    Tok eq = lx.next();
    if (eq.kind != Tok::Sym || eq.text != "=") lx.error("expected '='");
    std::vector<Term> terms = parse_terms(L, lx);
    Tok at = lx.next();
    if (at.kind != Tok::Sym || at.text != "@") lx.error("expected '@ SLOT'");
    Tok dt = lx.next();
    Slot dst;
    if (dt.kind != Tok::Ident || !slot_by_name(dt.text, &dst))
        fail(E_UNKNOWN_SLOT, "line " + std::to_string(lx.line()) + ": unknown destination slot");
    if (lx.peek().kind != Tok::End) lx.error("trailing tokens");

    Instr in;
    in.dst = dst;
    bool have_prod = false;
    std::vector<Term> adds;
    for (const Term& t : terms) {
        if (!t.tag.empty()) {
            if (have_prod) lx.error("more than one product term");
            bool found = false;
            for (const Term& u : t.inner) {
                if (!u.tag.empty()) lx.error("nested recursion tags");
                if (u.is_prod) {
                    if (found) lx.error("two products in one call");
                    found = true;
                    Sym ps = u.sym;
                    if (t.scalar_outside) {
                        if (t.inner.size() != 1)
                            lx.error("a scalar before a tagged call needs a pure product inside");
                        if (t.sym.neg) ps.neg = !ps.neg;
                        if (t.sym.sym) {
                            if (ps.sym) lx.error("conflicting scalars");
                            ps.sym = t.sym.sym;
                        }
                    } else if (t.sym.neg) {
                        ps.neg = !ps.neg;
                    }
                    in.s0 = ps;
                    in.o0 = u.a;
                    in.o1 = u.b;
                } else {
                    adds.push_back(u);
                }
            }
            if (!found) lx.error("tagged call without a product");
            in.tag = t.tag;
            have_prod = true;
        } else if (t.is_prod) {
            if (have_prod) lx.error("more than one product term");
            in.s0 = t.sym;
            in.o0 = t.a;
            in.o1 = t.b;
            have_prod = true;
        } else {
            adds.push_back(t);
        }
    }
    if (!have_prod && adds.empty()) lx.error("empty right-hand side");
    if (adds.size() > 2) lx.error("more than two slot terms");
    if (have_prod && adds.size() > 1) lx.error("a product allows at most one accumulator term");
    if (have_prod) {
        in.kind = Instr::Product;
        if (!adds.empty()) {
            in.has_acc = true;
            in.sacc = adds[0].sym;
            in.oacc = adds[0].a;
        }
        if (in.tag.empty()) in.tag = in.has_acc ? "acc3" : "std2";  // schedule.hpp:583-585
    } else if (adds.size() == 2) {
        in.kind = Instr::Add2;
        in.s0 = adds[0].sym;
        in.o0 = adds[0].a;
        in.s1 = adds[1].sym;
        in.o1 = adds[1].a;
    } else {
        in.kind = Instr::Copy1;
        in.s0 = adds[0].sym;
        in.o0 = adds[0].a;
    }
    if (!slot_writable(in.dst, s.contract))
        fail(E_CONTRACT_VIOLATION, "line " + std::to_string(lx.line()) + ": writing " +
                                       slot_name(in.dst) + " violates contract " +
                                       contract_name(s.contract));
    if (slot_role(in.dst) == Role::Temporary) {
        bool declared = false;
        for (const auto& t : s.temps) declared |= t.slot == in.dst;
        if (!declared) s.temps.push_back({in.dst, Dim::N2, Dim::N2});
    }
    L[lbl.text] = in.dst;
    s.ins.push_back(in);
}

std::string sym_text(const Sym& s) {
    std::string t = s.neg ? "-" : "";
    if (s.sym == 1) t += "alpha*";
    if (s.sym == 2) t += "beta*";
    return t;
}

}  // namespace

Schedule parse_schedule(const std::string& text) {
    Schedule s;  // defaults of schedule.hpp:219-224
    s.name = "anonymous";
    s.square_only = true;
    Labels L;
    for (int i = 0; i < NSLOT; ++i) L[slot_name(static_cast<Slot>(i))] = static_cast<Slot>(i);
    std::istringstream is(text);
    std::string raw;
    int line = 0;
    bool saw_ins = false;
    while (std::getline(is, raw)) {
        Lexer lx(raw, ++line);
        const Tok first = lx.peek();
        if (first.kind == Tok::End) continue;
        if (first.kind == Tok::Ident && !saw_ins && parse_directive(s, lx, raw)) continue;
        saw_ins = true;
        parse_instruction(s, L, lx);
    }
    return s;
}

std::string render_schedule(const Schedule& s) {
    std::ostringstream os;
    os << "schedule " << s.name << "\n"
       << "contract " << contract_name(s.contract) << "\n"
       << "accumulating " << (s.accumulating ? "true" : "false") << "\n"
       << "shape " << (s.square_only ? "square" : "rectangular") << "\n";
    for (const auto& t : s.temps)
        os << "temp " << slot_name(t.slot) << " " << dim_text(t.rows) << " " << dim_text(t.cols) << "\n";
    // an operand is written as the label of the value its slot holds (the
    // slot's own name while it still holds the frame's input)
    std::string held[NSLOT];
    for (int i = 0; i < NSLOT; ++i) held[i] = slot_name(static_cast<Slot>(i));
    int idx = 0;
    for (const auto& in : s.ins) {
        ++idx;
        const std::string label = "V" + std::to_string(idx);
        os << idx << ": " << label << " = ";
        if (in.kind == Instr::Product) {
            const bool dflt = in.tag == (in.has_acc ? "acc3" : "std2");
            const char* disp = tag_display(in.tag);
            if (!disp) fail(E_UNKNOWN_SCHEDULE, "cannot render recursion target " + in.tag);
            if (!dflt) os << disp << "(";
            os << sym_text(in.s0) << held[in.o0] << "*" << held[in.o1];
            if (in.has_acc)
                os << (in.sacc.neg ? " - " : " + ") << sym_text(Sym{false, in.sacc.sym})
                   << held[in.oacc];
            if (!dflt) os << ")";
        } else {
            os << sym_text(in.s0) << held[in.o0];
            if (in.kind == Instr::Add2)
                os << (in.s1.neg ? " - " : " + ") << sym_text(Sym{false, in.s1.sym}) << held[in.o1];
        }
        os << " @ " << slot_name(in.dst) << "\n";
        held[in.dst] = label;
    }
    return os.str();
}

bool same_schedule(const Schedule& a, const Schedule& b) {
    if (a.name != b.name || a.contract != b.contract || a.accumulating != b.accumulating ||
        a.square_only != b.square_only || a.temps.size() != b.temps.size() ||
        a.ins.size() != b.ins.size())
        return false;
    for (std::size_t i = 0; i < a.temps.size(); ++i)
        if (a.temps[i].slot != b.temps[i].slot || a.temps[i].rows != b.temps[i].rows ||
            a.temps[i].cols != b.temps[i].cols)
            return false;
    auto eq = [](const Sym& x, const Sym& y) { return x.neg == y.neg && x.sym == y.sym; };
    for (std::size_t i = 0; i < a.ins.size(); ++i) {
        const Instr &x = a.ins[i], &y = b.ins[i];
        if (x.kind != y.kind || x.dst != y.dst || !eq(x.s0, y.s0) || x.o0 != y.o0) return false;
        if (x.kind != Instr::Copy1 && x.o1 != y.o1) return false;
        if (x.kind == Instr::Add2 && !eq(x.s1, y.s1)) return false;
        if (x.kind == Instr::Product) {
            if (x.tag != y.tag || x.has_acc != y.has_acc) return false;
            if (x.has_acc && (!eq(x.sacc, y.sacc) || x.oacc != y.oacc)) return false;
        }
    }
    return true;
}

}  // namespace wm
