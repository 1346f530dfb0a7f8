// Host planner -- see wm_planner.h.  Function-by-function restatement of the
// reference interpreter and drivers, emitting device operations instead of
// executing them.
#include "wm_planner.h"

#include <algorithm>
#include <functional>
#include <map>
#include <tuple>

namespace wm {

// ----------------------------------------------------------------- views

bool View::overlaps(const View& o) const {
    // MatView::overlaps (ring.hpp:148-174)
    if (empty() || o.empty()) return false;
    if (region != o.region || origin != o.origin) return false;
    if (ld == o.ld) {
        const std::int64_t s = static_cast<std::int64_t>(ld);
        const std::int64_t delta = static_cast<std::int64_t>(o.off) - static_cast<std::int64_t>(off);
        const std::int64_t lo = delta - static_cast<std::int64_t>(cols);
        const std::int64_t hi = delta + static_cast<std::int64_t>(o.cols);
        // rows i of *this and j of o overlap iff (i - j) * s lies in (lo, hi)
        const std::int64_t kmin = lo / s - 2, kmax = hi / s + 2;
        for (std::int64_t kk = kmin; kk <= kmax; ++kk)
            if (kk * s > lo && kk * s < hi && kk > -static_cast<std::int64_t>(o.rows) &&
                kk < static_cast<std::int64_t>(rows))
                return true;
        return false;
    }
    return first_word() <= o.last_word() && o.first_word() <= last_word();
}

bool View::phys_overlaps(const View& o) const {
    if (empty() || o.empty() || region != o.region) return false;
    View a = *this, b = o;
    a.origin = b.origin = 0;
    a.base = b.base = 0;
    return a.overlaps(b);
}

std::array<View, 4> quad_split(const View& v) {
    if (v.rows % 2 || v.cols % 2) fail(E_ODD_DIMENSION, "quad_split requires even dimensions");
    const std::uint64_t r = v.rows / 2, c = v.cols / 2;
    return {v.window(0, 0, r, c), v.window(0, c, r, c), v.window(r, 0, r, c),
            v.window(r, c, r, c)};
}

// ------------------------------------------------------------ workspaces

void ArenaWorkspace::push_frame() {
    marks_.push_back(used_);
    words_.emplace_back();
}

View ArenaWorkspace::acquire(std::uint64_t rows, std::uint64_t cols, int depth, const char* slot) {
    if (marks_.empty()) fail(E_WORKSPACE, "acquire outside a frame");
    // 256-byte aligned placement keeps every temporary 16-B vector / TMA aligned;
    // at the BASELINE sizes (temporaries >= 128 x 128) it adds no padding.
    const std::uint64_t off = (used_ + 31) & ~std::uint64_t(31);
    used_ = off + rows * cols;
    high_ = std::max(high_, used_);
    words_.back().push_back(rows * cols);
    if (meter_) meter_->on_alloc(rows * cols, depth, slot);
    View v;
    v.region = R_T;
    v.origin = next_origin_++;
    v.base = off;
    v.off = off;
    v.rows = rows;
    v.cols = cols;
    v.ld = cols;
    return v;
}

void ArenaWorkspace::pop_frame() {
    if (marks_.empty()) fail(E_WORKSPACE, "pop without frame");
    if (meter_)
        for (auto w : words_.back()) meter_->on_free(w);
    words_.pop_back();
    used_ = marks_.back();
    marks_.pop_back();
}

View BumpWorkspace::acquire(std::uint64_t rows, std::uint64_t cols, int, const char*) {
    if (marks_.empty()) fail(E_WORKSPACE, "acquire outside a frame");
    const std::uint64_t need = rows * cols;
    if (used_ + need > chunk_.cols)
        fail(E_WORKSPACE, "scratch chunk exhausted: need " + std::to_string(need) +
                              " words, free " + std::to_string(chunk_.cols - used_));
    View v = chunk_;
    v.off = chunk_.off + used_;
    v.rows = rows;
    v.cols = cols;
    v.ld = cols;
    used_ += need;
    return v;
}

void BumpWorkspace::pop_frame() {
    if (marks_.empty()) fail(E_WORKSPACE, "pop without frame");
    used_ = marks_.back();
    marks_.pop_back();
}

QuadrantWorkspace::QuadrantWorkspace(View donor) {
    if (donor.rows != donor.cols) fail(E_WORKSPACE, "quadrant workspace donor must be square");
    frames_.push_back({donor, 0});
}

void QuadrantWorkspace::push_frame() {
    Frame& top = frames_.back();
    View region = top.region;
    if (top.used > 0) {
        if (region.rows < 2) fail(E_WORKSPACE, "scratch region exhausted");
        region = quad_split(region)[3];
    }
    frames_.push_back({region, 0});
}

View QuadrantWorkspace::acquire(std::uint64_t rows, std::uint64_t cols, int, const char* slot) {
    Frame& f = frames_.back();
    if (f.region.rows < 2 || rows > f.region.rows / 2 || cols > f.region.cols / 2)
        fail(E_WORKSPACE, std::string("temporary ") + slot + " does not fit the scratch region");
    if (f.used >= 3) fail(E_WORKSPACE, "more than three temporaries in a frame");
    View q = quad_split(f.region)[f.used++];
    return q.window(0, 0, rows, cols);
}

void QuadrantWorkspace::pop_frame() {
    if (frames_.size() <= 1) fail(E_WORKSPACE, "pop without frame");
    frames_.pop_back();
}

// ------------------------------------------------------------ driver helpers

bool parse_blocked(const std::string& v, int* t, std::string* base) {
    const std::string pre = "blocked_acc_t";
    if (v.rfind(pre, 0) != 0) return false;
    std::string rest = v.substr(pre.size());
    std::size_t i = 0;
    while (i < rest.size() && rest[i] >= '0' && rest[i] <= '9') ++i;
    if (i == 0) return false;
    *t = std::stoi(rest.substr(0, i));
    const std::string tail = rest.substr(i);
    if (tail.empty()) *base = "acc3";
    else if (tail == "_acc2") *base = "acc2";
    else return false;
    return true;
}

// iprect (config 3): block (i, j) of C = A_i * B_j over squares of side k.
const char* iprect_block_variant(std::uint64_t i, std::uint64_t j, std::uint64_t mb,
                                 std::uint64_t nb) {
    const bool last_i = i + 1 == mb, last_j = j + 1 == nb;
    if (last_i && last_j) return "ip";   // A_i and B_j both dead afterwards
    if (last_j) return "ovl";            // A_i's last use
    if (last_i) return "ovr";            // B_j's last use
    return "std2";
}

bool variant_accumulates(const std::string& v) {
    int t;
    std::string base;
    if (v == "ipmm" || v == "ipovmm" || v == "iprect" || v == "classic") return false;
    if (parse_blocked(v, &t, &base)) return true;
    return builtin(v).accumulating;
}

Contract variant_contract(const std::string& v) {
    int t;
    std::string base;
    if (v == "ipovmm" || v == "iprect") return Contract::OverwriteBoth;
    if (v == "ipmm" || v == "classic" || parse_blocked(v, &t, &base)) return Contract::ReadOnly;
    return builtin(v).contract;
}

// ------------------------------------------------------------ interpreter

namespace {

inline bool is_pow2(std::uint64_t x) { return x && (x & (x - 1)) == 0; }

struct Ctx {
    Field f;
    int cutoff = 1;
    Meter* meter = nullptr;
    Workspace* ws = nullptr;
    Contract policy = Contract::ReadOnly;
    Scalar alpha_v, beta_v;
    int depth = 0;
    bool peel = false;
    bool emit = true;
    std::vector<Op>* out = nullptr;
    const PlanOptions* opt = nullptr;
    int* frame_counter = nullptr;
    std::vector<View>* capture_temps = nullptr;  // dry run of a fused frame
    int frame = -1;
    const char* sched = nullptr;
    int row = 0;

    // ExecCtx::check_write (executor.hpp:40-49): region of the top-level call
    void check_write(const View& v, const char* what) const {
        if (v.origin == 0 &&
            !(policy == Contract::OverwriteA || policy == Contract::OverwriteBoth))
            fail(E_CONTRACT, std::string(what) + ": write into constant A");
        if (v.origin == 1 &&
            !(policy == Contract::OverwriteB || policy == Contract::OverwriteBoth))
            fail(E_CONTRACT, std::string(what) + ": write into constant B");
    }
    Scalar resolve(const Sym& s) const {
        Scalar v = s.sym == 1 ? alpha_v : s.sym == 2 ? beta_v : f.one();
        return s.neg ? f.neg(v) : v;
    }
    void emit_op(OpKind kind, const View& d, const View& a, const View& b, Scalar sa,
                 Scalar sb) const {
        if (!emit || !out) return;
        Op op;
        op.kind = kind;
        op.d = d;
        op.a = a;
        op.b = b;
        op.sa = sa;
        op.sb = sb;
        op.depth = depth;
        op.frame = frame;
        op.sched = sched;
        op.row = row;
        out->push_back(op);
    }
};

// block_addsub (ring.hpp:241-278)
void block_addsub(const Ctx& ctx, const View& dst, const View& a, const View& b, Scalar sa,
                  Scalar sb) {
    if (a.rows != b.rows || a.cols != b.cols || dst.rows != a.rows || dst.cols != a.cols)
        fail(E_DIMENSION, "block_addsub dimension mismatch");
    if (!dst.same_window(a) && dst.overlaps(a))
        fail(E_PARTIAL_OVERLAP, "block_addsub: dst partially overlaps a");
    if (!dst.same_window(b) && dst.overlaps(b))
        fail(E_PARTIAL_OVERLAP, "block_addsub: dst partially overlaps b");
    ctx.emit_op(OP_ADDSUB, dst, a, b, sa, sb);
    if (ctx.meter) {
        const std::uint64_t rc = dst.words();
        ctx.meter->add2_elems += rc;
        ctx.meter->adds += rc;
        if (!ctx.f.trivial(sa)) ctx.meter->mults += rc;
        if (!ctx.f.trivial(sb)) ctx.meter->mults += rc;
    }
}

// block_scale_copy (ring.hpp:282-310)
void block_scale_copy(const Ctx& ctx, const View& dst, const View& src, Scalar s) {
    if (dst.rows != src.rows || dst.cols != src.cols)
        fail(E_DIMENSION, "block_scale_copy dimension mismatch");
    if (!dst.same_window(src) && dst.overlaps(src))
        fail(E_PARTIAL_OVERLAP, "block_scale_copy: dst partially overlaps src");
    if (ctx.meter && !(ctx.f.is_one(s) && dst.same_window(src)))
        ctx.meter->copy_elems += dst.words();
    if (ctx.f.is_one(s)) {
        if (!dst.same_window(src)) ctx.emit_op(OP_COPY, dst, src, View{}, s, ctx.f.zero());
        if (ctx.meter) ctx.meter->word_moves += dst.words();
        return;
    }
    ctx.emit_op(OP_COPY, dst, src, View{}, s, ctx.f.zero());
    if (ctx.meter) {
        if (ctx.f.is_minus_one(s)) ctx.meter->word_moves += dst.words();
        else ctx.meter->mults += dst.words();
    }
}

// classical_mul (ring.hpp:315-384): the base case
void classical_mul(const Ctx& ctx, const View& C, const View& A, const View& B, Scalar alpha,
                   Scalar beta) {
    const std::uint64_t m = A.rows, k = A.cols, n = B.cols;
    if (B.rows != k || C.rows != m || C.cols != n)
        fail(E_DIMENSION, "classical_mul dimension mismatch");
    if (C.overlaps(A) || C.overlaps(B))
        fail(E_ALIAS, "classical_mul: C must be disjoint from A and B");
    ctx.emit_op(OP_MUL, C, A, B, alpha, beta);
    if (ctx.meter) {
        Meter& mt = *ctx.meter;
        ++mt.classical_calls;
        mt.leaf_flops += 2 * m * k * n;
        mt.mults += m * k * n;
        mt.adds += m * n * (k - 1);
        if (!ctx.f.is_zero(beta)) mt.adds += m * n;
        if (!ctx.f.trivial(alpha)) mt.mults += m * n;
        if (!ctx.f.trivial(beta)) mt.mults += m * n;
    }
}

void run_schedule(const Schedule& s, const View& A, const View& B, const View& C, Scalar alpha,
                  Scalar beta, Ctx ctx);
void peel_multiply(const View& A, const View& B, const View& C, Scalar alpha, Scalar beta,
                   const std::string& base, Ctx ctx);

// Can this frame run fused (wm_frame.cu)?  Every product must be a classical
// leaf, the frame square with the leaf size a multiple of the GEMM tile, the
// output disjoint from the operands (the kernels tile C), the field Z/pZ, and
// the frame must own two c x c blocks to host the seven product planes: two of
// its temporaries, or -- when its contract lets it overwrite A / B -- the
// A21 / B12 blocks (whose raw values the fused products never read).
bool frame_fusable(const std::string& variant, const View& A, const View& B, const View& C,
                   const Ctx& ctx) {
    if (!ctx.opt || !ctx.opt->fuse_frames || !ctx.emit || ctx.f.real) return false;
    if (ctx.peel || !is_builtin(variant)) return false;
    const std::uint64_t m = A.rows, k = A.cols, n = B.cols;
    if (m != k || k != n || m % 2) return false;
    const std::uint64_t c = m / 2;
    if (c > static_cast<std::uint64_t>(ctx.cutoff)) return false;  // children recurse
    if (c % static_cast<std::uint64_t>(ctx.opt->frame_align)) return false;
    if (c > static_cast<std::uint64_t>(ctx.opt->frame_max_leaf)) return false;
    if (C.phys_overlaps(A) || C.phys_overlaps(B)) return false;
    const Schedule& s = builtin(variant);
    int big = 0;
    for (const auto& t : s.temps)
        big += eval_dim(t.rows, m, k, n) >= c && eval_dim(t.cols, m, k, n) >= c;
    const bool ovA = s.contract == Contract::OverwriteA || s.contract == Contract::OverwriteBoth;
    const bool ovB = s.contract == Contract::OverwriteB || s.contract == Contract::OverwriteBoth;
    return big + (ovA ? 1 : 0) + (ovB ? 1 : 0) >= 2;
}

// multiply_into (executor.hpp:71-80)
void multiply_into(const std::string& variant, const View& A, const View& B, const View& C,
                   Scalar alpha, Scalar beta, Ctx& ctx) {
    if (variant == "classic" ||
        std::min({A.rows, A.cols, B.cols}) <= static_cast<std::uint64_t>(ctx.cutoff)) {
        ctx.check_write(C, "classical");
        classical_mul(ctx, C, A, B, alpha, beta);
        return;
    }
    if (frame_fusable(variant, A, B, C, ctx)) {
        // meter and validate the frame exactly as the reference walks it
        // (capturing its temporaries), then issue it fused
        std::vector<View> temps;
        Ctx dry = ctx;
        dry.emit = false;
        dry.capture_temps = &temps;
        run_schedule(builtin(variant), A, B, C, alpha, beta, dry);
        ctx.check_write(C, "frame");
        const Schedule& s = builtin(variant);
        const std::uint64_t c = A.rows / 2;
        std::vector<View> hosts;
        for (const View& t : temps)
            if (t.rows >= c && t.cols >= c && hosts.size() < 3) hosts.push_back(t.window(0, 0, c, c));
        const bool ovA = s.contract == Contract::OverwriteA || s.contract == Contract::OverwriteBoth;
        const bool ovB = s.contract == Contract::OverwriteB || s.contract == Contract::OverwriteBoth;
        if (hosts.size() < 2 && ovA) hosts.push_back(quad_split(A)[2]);
        if (hosts.size() < 2 && ovB) hosts.push_back(quad_split(B)[1]);
        if (hosts.size() < 2) fail(E_INVALID, "fused frame without plane hosts");
        if (ctx.emit && ctx.out) {
            Op op;
            op.kind = OP_FRAME;
            op.d = C;
            op.a = A;
            op.b = B;
            op.sa = alpha;
            op.sb = beta;
            op.depth = ctx.depth + 1;
            op.frame = ctx.frame;
            op.sched = s.name.c_str();
            op.row = ctx.row;
            op.h0 = hosts[0];
            op.h1 = hosts[1];
            if (hosts.size() > 2) op.h2 = hosts[2];
            ctx.out->push_back(op);
        }
        return;
    }
    run_schedule(builtin(variant), A, B, C, alpha, beta, ctx);
}

// run_schedule (executor.hpp:82-205)
void run_schedule(const Schedule& s, const View& A, const View& B, const View& C, Scalar alpha,
                  Scalar beta, Ctx ctx) {
    const std::uint64_t m = A.rows, k = A.cols, n = B.cols;
    if (B.rows != k || C.rows != m || C.cols != n)
        fail(E_DIMENSION, "schedule operands do not conform");
    if (m % 2 || k % 2 || n % 2) fail(E_ODD_DIMENSION, "schedule requires even dimensions");
    if (s.square_only && !(m == k && k == n)) fail(E_SHAPE, s.name + " supports square matrices only");
    if (!s.accumulating && !ctx.f.is_zero(beta))
        fail(E_DIMENSION, s.name + " is a plain product; beta must be 0");

    if (ctx.meter) ++ctx.meter->schedule_calls[s.name];
    ctx.frame = ctx.frame_counter ? (*ctx.frame_counter)++ : -1;
    ctx.sched = s.name.c_str();
    ctx.alpha_v = alpha;
    ctx.beta_v = beta;
    ctx.depth += 1;

    const auto aq = quad_split(A), bq = quad_split(B), cq = quad_split(C);
    struct Bound {
        View buf;
        std::uint64_t vr = 0, vc = 0;
        bool init = false, quadrant = false;
    };
    Bound slot[NSLOT];
    for (int i = 0; i < 4; ++i) {
        slot[A11 + i] = {aq[i], aq[i].rows, aq[i].cols, true, true};
        slot[B11 + i] = {bq[i], bq[i].rows, bq[i].cols, true, true};
        slot[C11 + i] = {cq[i], cq[i].rows, cq[i].cols, s.accumulating, true};
    }
    ctx.ws->push_frame();
    for (const auto& t : s.temps) {
        const std::uint64_t r = eval_dim(t.rows, m, k, n), c = eval_dim(t.cols, m, k, n);
        slot[t.slot] = {ctx.ws->acquire(r, c, ctx.depth, slot_name(t.slot)), 0, 0, false, false};
        if (ctx.capture_temps) ctx.capture_temps->push_back(slot[t.slot].buf);
    }
    ctx.capture_temps = nullptr;  // only the fused frame's own temporaries

    auto operand = [&](Slot id, const char* what) -> View {
        Bound& b = slot[id];
        if (!b.init)
            fail(E_CONTRACT, std::string(what) + ": slot " + slot_name(id) + " read before first write");
        return b.quadrant ? b.buf : b.buf.window(0, 0, b.vr, b.vc);
    };
    auto dst_view = [&](Slot id, std::uint64_t r, std::uint64_t c) -> View {
        Bound& b = slot[id];
        if (b.quadrant) {
            if (b.buf.rows != r || b.buf.cols != c)
                fail(E_DIMENSION, "value shape does not match quadrant slot");
            return b.buf;
        }
        if (r > b.buf.rows || c > b.buf.cols)
            fail(E_DIMENSION, std::string("value does not fit temporary ") + slot_name(id));
        return b.buf.window(0, 0, r, c);
    };
    auto mark = [&](Slot id, std::uint64_t r, std::uint64_t c) {
        slot[id].init = true;
        slot[id].vr = r;
        slot[id].vc = c;
    };

    int rowno = 0;
    for (const auto& in : s.ins) {
        ctx.row = ++rowno;
        if (in.kind == Instr::Product) {
            const View lv = operand(in.o0, "product"), rv = operand(in.o1, "product");
            if (lv.cols != rv.rows) fail(E_DIMENSION, "product inner dimensions disagree in " + s.name);
            const View dv = dst_view(in.dst, lv.rows, rv.cols);
            ctx.check_write(dv, "product");
            Scalar a_eff = ctx.resolve(in.s0);
            if (!s.accumulating) a_eff = ctx.f.mul(a_eff, alpha);
            Scalar b_eff = ctx.f.zero();
            if (in.has_acc) {
                if (in.oacc != in.dst) fail(E_CONTRACT, "accumulator term must alias destination");
                b_eff = ctx.resolve(in.sacc);
            }
            const std::string target = in.tag == "self" ? s.name : in.tag;
            if (ctx.peel && target != "classic")
                peel_multiply(lv, rv, dv, a_eff, b_eff, target, ctx);
            else
                multiply_into(target, lv, rv, dv, a_eff, b_eff, ctx);
            mark(in.dst, dv.rows, dv.cols);
        } else if (in.kind == Instr::Add2) {
            const View av = operand(in.o0, "addsub"), bv = operand(in.o1, "addsub");
            if (av.rows != bv.rows || av.cols != bv.cols)
                fail(E_DIMENSION, "addition operands disagree in " + s.name);
            const View dv = dst_view(in.dst, av.rows, av.cols);
            ctx.check_write(dv, "addsub");
            block_addsub(ctx, dv, av, bv, ctx.resolve(in.s0), ctx.resolve(in.s1));
            mark(in.dst, dv.rows, dv.cols);
        } else {
            const View sv = operand(in.o0, "copy");
            const View dv = dst_view(in.dst, sv.rows, sv.cols);
            ctx.check_write(dv, "copy");
            block_scale_copy(ctx, dv, sv, ctx.resolve(in.s0));
            mark(in.dst, dv.rows, dv.cols);
        }
    }
    ctx.ws->pop_frame();
}

// peel_multiply (executor.hpp:210-236)
void peel_multiply(const View& A, const View& B, const View& C, Scalar alpha, Scalar beta,
                   const std::string& base, Ctx ctx) {
    const std::uint64_t m = A.rows, k = A.cols, n = B.cols;
    if (B.rows != k || C.rows != m || C.cols != n) fail(E_DIMENSION, "peel operands do not conform");
    if (std::min({m, k, n}) <= static_cast<std::uint64_t>(ctx.cutoff)) {
        ctx.check_write(C, "classical");
        classical_mul(ctx, C, A, B, alpha, beta);
        return;
    }
    const std::uint64_t m0 = m & ~std::uint64_t(1), k0 = k & ~std::uint64_t(1),
                        n0 = n & ~std::uint64_t(1);
    ctx.peel = true;
    run_schedule(builtin(base), A.window(0, 0, m0, k0), B.window(0, 0, k0, n0),
                 C.window(0, 0, m0, n0), alpha, beta, ctx);
    if (k % 2) {
        ctx.check_write(C, "peel");
        classical_mul(ctx, C.window(0, 0, m0, n0), A.window(0, k0, m0, 1), B.window(k0, 0, 1, n0),
                      alpha, ctx.f.one());
    }
    if (n % 2)
        classical_mul(ctx, C.window(0, n0, m0, 1), A.window(0, 0, m0, k), B.window(0, n0, k, 1),
                      alpha, beta);
    if (m % 2) classical_mul(ctx, C.window(m0, 0, 1, n), A.window(m0, 0, 1, k), B, alpha, beta);
}

// assert_scratch_fits (drivers.hpp:38-46)
void assert_scratch_fits(std::uint64_t block, int cutoff, std::uint64_t region_words) {
    const std::uint64_t demand =
        std::max({expected_costs("std2", block, block, block, cutoff).peak,
                  expected_costs("acc3", block, block, block, cutoff).peak,
                  expected_costs("ovl", block, block, block, cutoff).peak});
    if (demand > region_words) fail(E_WORKSPACE, "scratch region smaller than schedule demand");
}

// ipmm_rec (drivers.hpp:105-134)
void ipmm_rec(const View& A, const View& B, const View& C, Ctx ctx) {
    const std::uint64_t n = C.rows, k = A.cols;
    if (n <= static_cast<std::uint64_t>(ctx.cutoff)) {
        classical_mul(ctx, C, A, B, ctx.f.one(), ctx.f.zero());
        return;
    }
    const std::uint64_t s = n / 2, q = k / s;
    const auto cq = quad_split(C);
    auto ablk = [&](std::uint64_t r, std::uint64_t i) { return A.window(r * s, i * s, s, s); };
    auto bblk = [&](std::uint64_t i, std::uint64_t c) { return B.window(i * s, c * s, s, s); };
    assert_scratch_fits(s, ctx.cutoff, s * s);
    {
        QuadrantWorkspace ws(cq[3]);
        ctx.ws = &ws;
        const Scalar one = ctx.f.one(), zero = ctx.f.zero();
        multiply_into("std2", ablk(0, 0), bblk(0, 0), cq[0], one, zero, ctx);
        multiply_into("std2", ablk(0, 0), bblk(0, 1), cq[1], one, zero, ctx);
        multiply_into("std2", ablk(1, 0), bblk(0, 0), cq[2], one, zero, ctx);
        for (std::uint64_t i = 1; i < q; ++i) {
            multiply_into("acc3", ablk(0, i), bblk(i, 0), cq[0], one, one, ctx);
            multiply_into("acc3", ablk(0, i), bblk(i, 1), cq[1], one, one, ctx);
            multiply_into("acc3", ablk(1, i), bblk(i, 0), cq[2], one, one, ctx);
        }
        ctx.ws = nullptr;
    }
    ipmm_rec(A.window(s, 0, s, k), B.window(0, s, k, s), cq[3], ctx);
}

View region_view(Region r, std::uint64_t rows, std::uint64_t cols, std::uint64_t ld) {
    View v;
    v.region = r;
    v.origin = static_cast<std::int32_t>(r);
    v.base = 0;
    v.off = 0;
    v.rows = rows;
    v.cols = cols;
    v.ld = ld;
    return v;
}

}  // namespace

Plan plan_variant(const std::string& variant, Field f, std::uint64_t m, std::uint64_t k,
                  std::uint64_t n, std::uint64_t lda, std::uint64_t ldb, std::uint64_t ldc,
                  Scalar alpha, Scalar beta, int cutoff, const PlanOptions& opt) {
    Plan plan;
    plan.variant = variant;
    plan.m = m;
    plan.k = k;
    plan.n = n;
    plan.cutoff = cutoff;
    plan.field = f;
    if (m == 0 || k == 0 || n == 0) fail(E_DIMENSION, "matrix dimensions must be positive");
    if (lda < k || ldb < n || ldc < n) fail(E_DIMENSION, "leading dimension smaller than columns");
    if (cutoff < 1) fail(E_DIMENSION, "cutoff must be >= 1");
    if (!f.real && (f.p <= 2 || f.p >= (1u << 16)))
        fail(E_DIMENSION, "the device path supports odd primes p < 2^16 (lazy exact path)");

    const View A = region_view(R_A, m, k, lda), B = region_view(R_B, k, n, ldb),
               C = region_view(R_C, m, n, ldc);
    ArenaWorkspace heap(&plan.meter);
    Ctx ctx;
    ctx.f = f;
    ctx.cutoff = cutoff;
    ctx.meter = &plan.meter;
    ctx.ws = &heap;
    ctx.out = &plan.ops;
    {  // unit-size recursions emit ~10^5-10^6 operations: reserve instead of regrowing
        std::uint64_t side = std::min({m, k, n}), leaves = 1;
        while (side > static_cast<std::uint64_t>(std::max(cutoff, 1)) && leaves < (1u << 22)) {
            side /= 2;
            leaves *= 7;
        }
        plan.ops.reserve(static_cast<std::size_t>(4 * leaves));
    }
    ctx.opt = &opt;
    int frame_counter = 0;
    ctx.frame_counter = &frame_counter;
    int t;
    std::string base;

    if (opt.parsed) {
        // run_parsed_schedule (executor.hpp:304-342)
        const Schedule& s = *opt.parsed;
        if (s.square_only && !(m == k && k == n && is_pow2(n)))
            fail(E_SHAPE, s.name + " requires square power-of-two dimensions");
        ctx.policy = s.contract;
        if (std::min({m, k, n}) <= static_cast<std::uint64_t>(cutoff))
            classical_mul(ctx, C, A, B, alpha, beta);
        else
            run_schedule(s, A, B, C, alpha, beta, ctx);
    } else if (variant == "ipmm") {
        // ipmm (drivers.hpp:137-158)
        if (B.cols != m || C.rows != m || C.cols != m || B.rows != k)
            fail(E_DIMENSION, "ipmm expects A n x k, B k x n, C n x n");
        if (!is_pow2(m) || !is_pow2(k)) fail(E_SHAPE, "ipmm requires power-of-two dimensions");
        if (k < m) fail(E_SHAPE, "ipmm requires k >= n; use the transpose");
        ctx.policy = Contract::ReadOnly;
        ipmm_rec(A, B, C, ctx);
    } else if (variant == "ipovmm") {
        // ipovmm (drivers.hpp:52-99)
        if (!is_pow2(m) || !is_pow2(k) || !is_pow2(n))
            fail(E_SHAPE, "ipovmm requires power-of-two dimensions");
        if (n >= std::min(m, k)) fail(E_SHAPE, "ipovmm requires n < min(m,k); transpose or use ipmm");
        ctx.policy = Contract::OverwriteBoth;
        const std::uint64_t m0 = m / n, k0 = k / n;
        auto ablk = [&](std::uint64_t i, std::uint64_t j) { return A.window(i * n, j * n, n, n); };
        auto bstripe = [&](std::uint64_t j) { return B.window(j * n, 0, n, n); };
        auto cstripe = [&](std::uint64_t i) { return C.window(i * n, 0, n, n); };
        assert_scratch_fits(n, cutoff, n * n);
        const Scalar one = f.one(), zero = f.zero();
        {
            QuadrantWorkspace ws(cstripe(1));
            ctx.ws = &ws;
            multiply_into("std2", ablk(0, 0), bstripe(0), cstripe(0), one, zero, ctx);
        }
        QuadrantWorkspace ws(ablk(0, 0));
        ctx.ws = &ws;
        for (std::uint64_t i = 1; i < m0; ++i)
            multiply_into("ovl", ablk(i, 0), bstripe(0), cstripe(i), one, zero, ctx);
        for (std::uint64_t j = 1; j < k0; ++j)
            for (std::uint64_t i = 0; i < m0; ++i)
                multiply_into("acc3", ablk(i, j), bstripe(j), cstripe(i), one, one, ctx);
    } else if (variant == "iprect") {
        // In-place rectangular product, k <= min(m, n) (config 3): the
        // composition of PAPER.md:588-598 -- squares of side k, read-only std2
        // while both operand blocks are still needed, ovl / ovr at the last use
        // of A_i / B_j, ip for the final block; scratch is carved from the
        // final, not-yet-written C block, so no temporary is allocated.
        if (!is_pow2(m) || !is_pow2(k) || !is_pow2(n))
            fail(E_SHAPE, "iprect requires power-of-two dimensions");
        if (k > std::min(m, n)) fail(E_SHAPE, "iprect requires k <= min(m,n)");
        ctx.policy = Contract::OverwriteBoth;
        const std::uint64_t mb = m / k, nb = n / k;
        if (std::min({m, k, n}) <= static_cast<std::uint64_t>(cutoff)) {
            classical_mul(ctx, C, A, B, alpha, f.zero());
        } else {
            if (mb * nb > 1) assert_scratch_fits(k, cutoff, k * k);
            QuadrantWorkspace ws(C.window((mb - 1) * k, (nb - 1) * k, k, k));
            ctx.ws = &ws;
            for (std::uint64_t i = 0; i < mb; ++i)
                for (std::uint64_t j = 0; j < nb; ++j)
                    multiply_into(iprect_block_variant(i, j, mb, nb), A.window(i * k, 0, k, k),
                                  B.window(0, j * k, k, k), C.window(i * k, j * k, k, k), alpha,
                                  f.zero(), ctx);
        }
    } else if (parse_blocked(variant, &t, &base)) {
        // blocked_acc (drivers.hpp:163-209)
        if (m != n || k != n) fail(E_DIMENSION, "blocked_acc expects square n x n operands");
        if (t < 1 || n % static_cast<std::uint64_t>(t) != 0) fail(E_DIMENSION, "t must divide n");
        const std::uint64_t s = n / static_cast<std::uint64_t>(t);
        if (!is_pow2(s)) fail(E_DIMENSION, "n/t must be a power of two");
        const std::uint64_t chunk = base == "acc2" ? 2 * (s * s - 1) / 3 : s * s;
        heap.push_frame();
        View scratch = heap.acquire(1, chunk, 0, "scratch");
        BumpWorkspace ws(scratch);
        ctx.ws = &ws;
        ctx.policy = Contract::ReadOnly;
        const std::uint64_t T = static_cast<std::uint64_t>(t);
        for (std::uint64_t i = 0; i < T; ++i)
            for (std::uint64_t j = 0; j < T; ++j)
                for (std::uint64_t l = 0; l < T; ++l)
                    multiply_into(base, A.window(i * s, l * s, s, s), B.window(l * s, j * s, s, s),
                                  C.window(i * s, j * s, s, s), alpha, l == 0 ? beta : f.one(), ctx);
        heap.pop_frame();
    } else if (variant == "classic") {
        ctx.policy = Contract::ReadOnly;
        classical_mul(ctx, C, A, B, alpha, beta);
    } else {
        // multiply (executor.hpp:240-299)
        const Schedule& s = builtin(variant);
        ctx.policy = s.contract;
        if (!s.accumulating && !f.is_zero(beta))
            fail(E_DIMENSION, variant + " is a plain product; beta must be 0");
        const bool pow2 = is_pow2(m) && is_pow2(k) && is_pow2(n);
        if (s.square_only && !(m == k && k == n && pow2))
            fail(E_SHAPE, variant + " requires square power-of-two dimensions");
        if (std::min({m, k, n}) <= static_cast<std::uint64_t>(cutoff)) {
            classical_mul(ctx, C, A, B, alpha, beta);
        } else if (!pow2) {
            if (variant != "std2" && variant != "acc3")
                fail(E_SHAPE, variant + " requires power-of-two dimensions (peeling wraps std2/acc3 only)");
            peel_multiply(A, B, C, alpha, beta, variant, ctx);
        } else {
            multiply_into(variant, A, B, C, alpha, beta, ctx);
        }
    }
    plan.arena_words = heap.high_water();
    plan.alloc_log = std::make_shared<const std::vector<Meter::AllocEvent>>(
        std::move(plan.meter.alloc_log));
    return plan;
}

}  // namespace wm
