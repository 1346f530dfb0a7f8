// Cost model: the mults / adds / word moves / peak and total temporary words a
// variant will meter, predicted without executing anything.
//
// The reference keeps one hand-derived recurrence per schedule
// (models.hpp:33-229).  Here the prediction is read off the schedule IR
// itself, so any builtin -- and any future schedule in the catalog -- gets its
// model for free: a frame is abstractly interpreted over value *shapes* only
// (no views, no device ops), counting each two-term instruction's elements as
// additions, each one-term instruction's as moves, and folding in the cost of
// each product's recursion target.  Temporaries are acquired when a frame
// starts and released when it ends (run_schedule, executor.hpp:126-131,204),
// so a frame's peak is its own temporary words plus the deepest child peak.
// Frames are memoised per (schedule, m, k, n): one evaluation per recursion
// level, whatever the cutoff.
//
// Drivers (ipmm, ipovmm, iprect, blocked_acc) are predicted by tallying the
// schedule calls they issue (drivers.hpp:52-209 and the iprect composition of
// DESIGN.md) and summing the tallies.  Pinned against the reference's own
// expected_costs and meter in tests/test_oracle.py and tests/test_planner.py.
#include <algorithm>
#include <map>
#include <tuple>

#include "wm_planner.h"

namespace wm {
namespace {

struct Shape {
    std::uint64_t r = 0, c = 0;
    std::uint64_t words() const { return r * c; }
};

// classical_mul's meter (ring.hpp:375-383) at unit scalars
Costs leaf_costs(std::uint64_t m, std::uint64_t k, std::uint64_t n, bool accumulate) {
    Costs out;
    out.mults = m * k * n;
    out.adds = m * n * (k - 1) + (accumulate ? m * n : 0);
    return out;
}

void add_scaled(Costs& into, const Costs& c, std::uint64_t times) {
    into.mults += times * c.mults;
    into.adds += times * c.adds;
    into.moves += times * c.moves;
}

class IrCostModel {
  public:
    explicit IrCostModel(std::uint64_t cutoff) : cutoff_(cutoff) {}

    // One call of builtin `name` on (m x k) * (k x n), as multiply_into issues it.
    Costs call(const std::string& name, std::uint64_t m, std::uint64_t k, std::uint64_t n) {
        const auto key = std::make_tuple(name, m, k, n);
        const auto hit = cache_.find(key);
        if (hit != cache_.end()) return hit->second;
        Costs out;
        if (name == "classic") {
            out = leaf_costs(m, k, n, false);
        } else {
            const Schedule& s = builtin(name);  // unknown names throw E_UNKNOWN_SCHEDULE
            out = std::min({m, k, n}) <= cutoff_ ? leaf_costs(m, k, n, s.accumulating)
                                                 : frame(s, m, k, n);
        }
        cache_.emplace(key, out);
        return out;
    }

    std::uint64_t cutoff() const { return cutoff_; }

  private:
    Costs frame(const Schedule& s, std::uint64_t m, std::uint64_t k, std::uint64_t n) {
        Shape value[NSLOT];
        for (int q = 0; q < 4; ++q) {
            value[A11 + q] = {m / 2, k / 2};
            value[B11 + q] = {k / 2, n / 2};
            value[C11 + q] = {m / 2, n / 2};
        }
        std::uint64_t own = 0;
        for (const TempDecl& t : s.temps) own += eval_dim(t.rows, m, k, n) * eval_dim(t.cols, m, k, n);

        Costs out;
        std::uint64_t deepest_child = 0;
        for (const Instr& in : s.ins) {
            switch (in.kind) {
                case Instr::Add2:
                    value[in.dst] = value[in.o0];
                    out.adds += value[in.dst].words();
                    break;
                case Instr::Copy1:
                    value[in.dst] = value[in.o0];
                    out.moves += value[in.dst].words();
                    break;
                case Instr::Product: {
                    const Shape lhs = value[in.o0], rhs = value[in.o1];
                    const std::string target = in.tag == "self" ? s.name : in.tag;
                    const Costs child = target == "classic"
                                            ? leaf_costs(lhs.r, lhs.c, rhs.c, in.has_acc)
                                            : call(target, lhs.r, lhs.c, rhs.c);
                    add_scaled(out, child, 1);
                    out.total += child.total;
                    deepest_child = std::max(deepest_child, child.peak);
                    value[in.dst] = {lhs.r, rhs.c};
                    break;
                }
            }
        }
        out.peak = own + deepest_child;
        out.total += own;
        return out;
    }

    std::uint64_t cutoff_;
    std::map<std::tuple<std::string, std::uint64_t, std::uint64_t, std::uint64_t>, Costs> cache_;
};

// A driver's schedule calls, with multiplicities; scratch lives in the operands.
struct Tally {
    std::map<std::tuple<std::string, std::uint64_t, std::uint64_t, std::uint64_t>, std::uint64_t> calls;
    void add(const std::string& name, std::uint64_t m, std::uint64_t k, std::uint64_t n,
             std::uint64_t times) {
        if (times) calls[std::make_tuple(name, m, k, n)] += times;
    }
    Costs sum(IrCostModel& model) const {
        Costs out;
        for (const auto& [key, times] : calls)
            add_scaled(out, model.call(std::get<0>(key), std::get<1>(key), std::get<2>(key),
                                       std::get<3>(key)),
                       times);
        return out;
    }
};

}  // namespace

Costs expected_costs(const std::string& variant, std::uint64_t m, std::uint64_t k,
                     std::uint64_t n, int cutoff) {
    IrCostModel model(static_cast<std::uint64_t>(cutoff));
    Tally tally;
    int t = 0;
    std::string base;
    if (variant == "ipmm") {
        // ipmm_rec (drivers.hpp:105-134): per level 3 std2 + 3(q-1) acc3 on s^3
        // blocks, then the C22 stream one level down; a long-K leaf at the end
        std::uint64_t side = n;
        Costs out;
        while (side > model.cutoff()) {
            const std::uint64_t s = side / 2, q = k / s;
            tally.add("std2", s, s, s, 3);
            tally.add("acc3", s, s, s, 3 * (q - 1));
            side = s;
        }
        out = tally.sum(model);
        add_scaled(out, leaf_costs(side, k, side, false), 1);
        return out;
    }
    if (variant == "ipovmm") {  // drivers.hpp:52-99
        const std::uint64_t mb = m / n, kb = k / n;
        tally.add("std2", n, n, n, 1);
        tally.add("ovl", n, n, n, mb - 1);
        tally.add("acc3", n, n, n, (kb - 1) * mb);
        return tally.sum(model);
    }
    if (variant == "iprect") {  // config-3 composition over k x k squares
        const std::uint64_t mb = m / k, nb = n / k;
        for (std::uint64_t i = 0; i < mb; ++i)
            for (std::uint64_t j = 0; j < nb; ++j) tally.add(iprect_block_variant(i, j, mb, nb), k, k, k, 1);
        return tally.sum(model);
    }
    if (parse_blocked(variant, &t, &base)) {  // drivers.hpp:163-209
        const std::uint64_t s = n / static_cast<std::uint64_t>(t), tt = static_cast<std::uint64_t>(t);
        tally.add(base, s, s, s, tt * tt * tt);
        Costs out = tally.sum(model);
        // one shared scratch chunk, allocated once
        out.peak = out.total = base == "acc2" ? 2 * (s * s - 1) / 3 : s * s;
        return out;
    }
    return model.call(variant, m, k, n);
}

}  // namespace wm
