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
#include <algorithm>
#include <cctype>
#include <map>
#include <sstream>

#include "wm_schedule.h"

namespace wm {
namespace {

// ------------------------------------------------------------------ tables

// recursion tags (schedule.hpp:109-121) <-> this build's schedule names
struct TagName {
    const char* text;
    const char* target;
};
constexpr TagName kTags[] = {{"Classic", "classic"}, {"Std2", "std2"}, {"Acc3", "acc3"},
                             {"IP", "ip"},           {"OvL", "ovl"},   {"OvR", "ovr"},
                             {"AcLR", "aclr"},       {"AccR", "accr"}, {"Acc2", "acc2"},
                             {"AcR", "acr"},         {"Self", "self"}};

const char* tag_target(const std::string& t) {
    for (const TagName& e : kTags)
        if (t == e.text) return e.target;
    return nullptr;
}

const char* tag_display(const std::string& target) {
    for (const TagName& e : kTags)
        if (target == e.target) return e.text;
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

struct DimName {
    Dim d;
    const char* text;
};
constexpr DimName kDims[] = {{Dim::M2, "m/2"},
                             {Dim::K2, "k/2"},
                             {Dim::N2, "n/2"},
                             {Dim::MaxK2N2, "max(k/2,n/2)"},
                             {Dim::MaxM2K2, "max(m/2,k/2)"}};

bool dim_by_name(const std::string& t, Dim* d) {
    for (const DimName& e : kDims)
        if (t == e.text) {
            *d = e.d;
            return true;
        }
    return false;
}

const char* dim_text(Dim d) {
    for (const DimName& e : kDims)
        if (e.d == d) return e.text;
    return "?";
}

// ------------------------------------------------------------------ tokens

// One source line cut into words (identifiers, integers) and single-character
// punctuation; everything after '#' is a comment.
struct Piece {
    enum Kind : std::uint8_t { Word, Number, Punct } kind;
    std::string text;
};

std::vector<Piece> cut_line(const std::string& line) {
    std::vector<Piece> out;
    std::size_t i = 0;
    auto is_word = [](char ch) {
        return std::isalnum(static_cast<unsigned char>(ch)) || ch == '_' || ch == '\'';
    };
    while (i < line.size()) {
        const char ch = line[i];
        if (ch == '#') break;
        if (std::isspace(static_cast<unsigned char>(ch))) {
            ++i;
            continue;
        }
        std::size_t j = i + 1;
        if (std::isdigit(static_cast<unsigned char>(ch))) {
            while (j < line.size() && std::isdigit(static_cast<unsigned char>(line[j]))) ++j;
            out.push_back({Piece::Number, line.substr(i, j - i)});
        } else if (std::isalpha(static_cast<unsigned char>(ch))) {
            while (j < line.size() && is_word(line[j])) ++j;
            out.push_back({Piece::Word, line.substr(i, j - i)});
        } else {
            out.push_back({Piece::Punct, std::string(1, ch)});
        }
        i = j;
    }
    return out;
}

// ------------------------------------------------------------------ header

// Header lines precede the first instruction; the dimension expressions of a
// `temp` line are whitespace-separated words of the raw line.
bool read_header_line(Schedule& s, const std::string& raw, int line) {
    std::istringstream words(raw);
    std::string key;
    words >> key;
    auto bad = [&](const std::string& m) { fail(E_PARSE, "line " + std::to_string(line) + ": " + m); };
    if (key == "schedule") {
        words >> s.name;
    } else if (key == "contract") {
        std::string v;
        words >> v;
        const Contract all[] = {Contract::ReadOnly, Contract::OverwriteA, Contract::OverwriteB,
                                Contract::OverwriteBoth};
        bool known = false;
        for (Contract c : all)
            if (v == contract_name(c)) s.contract = c, known = true;
        if (!known) bad("unknown contract: " + v);
    } else if (key == "accumulating") {
        std::string v;
        words >> v;
        if (v != "true" && v != "false") bad("accumulating expects true|false");
        s.accumulating = v == "true";
    } else if (key == "shape") {
        std::string v;
        words >> v;
        if (v != "square" && v != "rectangular") bad("shape expects square|rectangular");
        s.square_only = v == "square";
    } else if (key == "temp") {
        std::string slot, rows, cols;
        words >> slot >> rows >> cols;
        TempDecl t{};
        if (!slot_by_name(slot, &t.slot) || slot_role(t.slot) != Role::Temporary)
            bad("temp expects a temporary slot name");
        if (!dim_by_name(rows, &t.rows) || !dim_by_name(cols, &t.cols)) bad("bad temp dimension");
        s.temps.push_back(t);
    } else {
        return false;
    }
    return true;
}

// ------------------------------------------------------------------ body

// A right-hand side is a signed sum of terms; a term is an operand, a product
// of two operands, or a recursion call Tag(...) around such a sum.
struct Term {
    Sym sym;
    enum Form : std::uint8_t { Operand, Product, Call } form = Operand;
    Slot lhs = SX, rhs = SX;
    std::string target;        // Call: recursion target
    std::vector<Term> inside;  // Call: its terms
    bool prefixed = false;     // Call: scalar written before the tag
};

class InstructionReader {
  public:
    InstructionReader(std::vector<Piece> pieces, int line, std::map<std::string, Slot>& names)
        : p_(std::move(pieces)), line_(line), names_(names) {}

    void read_into(Schedule& s) {
        const long long index = number("expected instruction index");
        if (index != static_cast<long long>(s.ins.size()) + 1)
            error("instruction indices must be sequential from 1");
        punct(':', "expected ':'");
        const std::string label = word("expected result label");
        punct('=', "expected '='");
        const std::vector<Term> sum = terms();
        punct('@', "expected '@ SLOT'");
        Slot dst;
        if (!looking_at(Piece::Word) || !slot_by_name(p_[i_].text, &dst))
            fail(E_UNKNOWN_SLOT, "line " + std::to_string(line_) + ": unknown destination slot");
        ++i_;
        if (i_ != p_.size()) error("trailing tokens");

        Instr in = lower(sum);
        in.dst = dst;
        if (!slot_writable(dst, s.contract))
            fail(E_CONTRACT_VIOLATION, "line " + std::to_string(line_) + ": writing " +
                                           slot_name(dst) + " violates contract " +
                                           contract_name(s.contract));
        if (slot_role(dst) == Role::Temporary &&
            std::none_of(s.temps.begin(), s.temps.end(), [&](const TempDecl& t) { return t.slot == dst; }))
            s.temps.push_back({dst, Dim::N2, Dim::N2});
        names_[label] = dst;
        s.ins.push_back(in);
    }

  private:
    [[noreturn]] void error(const std::string& m) const {
        fail(E_PARSE, "line " + std::to_string(line_) + ": " + m);
    }
    bool looking_at(Piece::Kind k, char ch = 0) const {
        return i_ < p_.size() && p_[i_].kind == k && (!ch || p_[i_].text[0] == ch);
    }
    void punct(char ch, const char* m) {
        if (!looking_at(Piece::Punct, ch)) error(m);
        ++i_;
    }
    std::string word(const char* m) {
        if (!looking_at(Piece::Word)) error(m);
        return p_[i_++].text;
    }
    long long number(const char* m) {
        if (!looking_at(Piece::Number)) error(m);
        return std::stoll(p_[i_++].text);
    }
    Slot operand(const std::string& name) const {
        const auto it = names_.find(name);
        if (it == names_.end())
            fail(E_UNKNOWN_SLOT, "line " + std::to_string(line_) + ": unknown operand '" + name + "'");
        return it->second;
    }

    std::vector<Term> terms() {
        std::vector<Term> out;
        while (i_ < p_.size() && !looking_at(Piece::Punct, '@') && !looking_at(Piece::Punct, ')')) {
            Term t;
            if (looking_at(Piece::Punct, '+') || looking_at(Piece::Punct, '-'))
                t.sym.neg = p_[i_++].text[0] == '-';
            else if (!out.empty())
                error("expected '+' or '-' between terms");
            bool scaled = false;
            if (looking_at(Piece::Number)) {
                if (p_[i_].text != "1") error("integer scalars other than 1 are not supported on the device path");
                ++i_;
                scaled = true;
            } else if (looking_at(Piece::Word) && (p_[i_].text == "alpha" || p_[i_].text == "beta")) {
                t.sym.sym = p_[i_++].text == "alpha" ? 1 : 2;
                scaled = true;
            }
            if (scaled) punct('*', "expected '*' after scalar");
            const std::string head = word("expected operand");
            const char* target = tag_target(head);
            if (target && looking_at(Piece::Punct, '(')) {
                ++i_;
                t.form = Term::Call;
                t.target = target;
                t.prefixed = scaled;
                t.inside = terms();
                punct(')', "expected ')'");
            } else {
                t.lhs = operand(head);
                if (looking_at(Piece::Punct, '*')) {
                    ++i_;
                    t.rhs = operand(word("expected operand after '*'"));
                    t.form = Term::Product;
                }
            }
            out.push_back(std::move(t));
        }
        return out;
    }

    // Terms -> one instruction: at most one product (tagged or not) with at most
    // one accumulator term, or one / two slot terms.
    Instr lower(const std::vector<Term>& sum) const {
        Instr in;
        const Term* product = nullptr;
        std::string target;
        Sym product_sym;
        std::vector<const Term*> slots;
        auto take_product = [&](const Term& t, Sym sym, const std::string& tag) {
            if (product) error("more than one product term");
            product = &t;
            product_sym = sym;
            target = tag;
        };
        for (const Term& t : sum) {
            if (t.form == Term::Operand) {
                slots.push_back(&t);
            } else if (t.form == Term::Product) {
                take_product(t, t.sym, "");
            } else {
                if (product) error("more than one product term");
                const Term* inner_product = nullptr;
                for (const Term& u : t.inside) {
                    if (u.form == Term::Call) error("nested recursion tags");
                    if (u.form == Term::Operand) {
                        slots.push_back(&u);
                        continue;
                    }
                    if (inner_product) error("two products in one call");
                    inner_product = &u;
                }
                if (!inner_product) error("tagged call without a product");
                // the call's own sign / scalar distributes onto its product
                Sym sym = inner_product->sym;
                if (t.prefixed && t.inside.size() != 1)
                    error("a scalar before a tagged call needs a pure product inside");
                sym.neg = sym.neg != t.sym.neg;
                if (t.prefixed && t.sym.sym) {
                    if (sym.sym) error("conflicting scalars");
                    sym.sym = t.sym.sym;
                }
                take_product(*inner_product, sym, t.target);
            }
        }
        if (!product && slots.empty()) error("empty right-hand side");
        if (slots.size() > 2) error("more than two slot terms");
        if (product) {
            if (slots.size() > 1) error("a product allows at most one accumulator term");
            in.kind = Instr::Product;
            in.s0 = product_sym;
            in.o0 = product->lhs;
            in.o1 = product->rhs;
            in.has_acc = !slots.empty();
            if (in.has_acc) {
                in.sacc = slots[0]->sym;
                in.oacc = slots[0]->lhs;
            }
            // untagged products: std2, or acc3 with an accumulator (schedule.hpp:583-585)
            in.tag = !target.empty() ? target : in.has_acc ? "acc3" : "std2";
            return in;
        }
        in.kind = slots.size() == 2 ? Instr::Add2 : Instr::Copy1;
        in.s0 = slots[0]->sym;
        in.o0 = slots[0]->lhs;
        if (slots.size() == 2) {
            in.s1 = slots[1]->sym;
            in.o1 = slots[1]->lhs;
        }
        return in;
    }

    std::vector<Piece> p_;
    std::size_t i_ = 0;
    int line_;
    std::map<std::string, Slot>& names_;
};

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
    std::map<std::string, Slot> names;  // slot names, then result labels
    for (int i = 0; i < NSLOT; ++i) names[slot_name(static_cast<Slot>(i))] = static_cast<Slot>(i);
    std::istringstream lines(text);
    std::string raw;
    int line = 0;
    bool in_body = false;
    while (std::getline(lines, raw)) {
        ++line;
        std::vector<Piece> pieces = cut_line(raw);
        if (pieces.empty()) continue;
        if (!in_body && pieces[0].kind == Piece::Word && read_header_line(s, raw, line)) continue;
        in_body = true;
        InstructionReader(std::move(pieces), line, names).read_into(s);
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
