// winomem-b200 C++ drop-in: the reference winomem API (namespace winomem,
// /root/reference/proj/include/winomem/) re-declared over the C-ABI in
// winomem_b200.h.  Code written against the reference's run_variant / multiply /
// ipmm / classical_mul / block_addsub / models::expected_costs compiles
// unchanged against this header and runs on the B200; link with
// libwinomem_b200.so.
//
// Matrices stay host-resident uint32 residues exactly as in the reference
// (ring.hpp:180-219); every call uploads, runs on the device and writes back the
// matrices the variant's contract allows it to change.  Errors are thrown as
// the reference's exception types.  There is no CPU path: without a CUDA
// device the calls throw.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <istream>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "winomem_b200.h"

namespace winomem {

using Elem = std::uint32_t;

// ---- exception taxonomy (ring.hpp:23-43, workspace.hpp:20-22, schedule.hpp:30-43)
struct dimension_error : std::runtime_error {
    explicit dimension_error(const std::string& w) : std::runtime_error(w) {}
};
struct odd_dimension_error : dimension_error {
    explicit odd_dimension_error(const std::string& w) : dimension_error(w) {}
};
struct partial_overlap_error : std::runtime_error {
    explicit partial_overlap_error(const std::string& w) : std::runtime_error(w) {}
};
struct alias_error : std::runtime_error {
    explicit alias_error(const std::string& w) : std::runtime_error(w) {}
};
struct shape_error : std::runtime_error {
    explicit shape_error(const std::string& w) : std::runtime_error(w) {}
};
struct contract_error : std::runtime_error {
    explicit contract_error(const std::string& w) : std::runtime_error(w) {}
};
struct io_error : std::runtime_error {
    explicit io_error(const std::string& w) : std::runtime_error(w) {}
};
struct workspace_error : std::runtime_error {
    explicit workspace_error(const std::string& w) : std::runtime_error(w) {}
};
struct unknown_slot_error : std::runtime_error {
    explicit unknown_slot_error(const std::string& w) : std::runtime_error(w) {}
};
struct unknown_schedule_error : std::runtime_error {
    explicit unknown_schedule_error(const std::string& w) : std::runtime_error(w) {}
};
struct parse_error : std::runtime_error {
    explicit parse_error(const std::string& w) : std::runtime_error(w) {}
};
struct contract_violation_error : std::runtime_error {
    explicit contract_violation_error(const std::string& w) : std::runtime_error(w) {}
};
struct device_error : std::runtime_error {
    explicit device_error(const std::string& w) : std::runtime_error(w) {}
};

namespace b200 {
inline void check(int rc) {
    if (rc == WM_OK) return;
    const std::string w = wm_last_error();
    switch (rc) {
        case WM_E_DIMENSION: throw dimension_error(w);
        case WM_E_ODD_DIMENSION: throw odd_dimension_error(w);
        case WM_E_PARTIAL_OVERLAP: throw partial_overlap_error(w);
        case WM_E_ALIAS: throw alias_error(w);
        case WM_E_SHAPE: throw shape_error(w);
        case WM_E_CONTRACT: throw contract_error(w);
        case WM_E_IO: throw io_error(w);
        case WM_E_WORKSPACE: throw workspace_error(w);
        case WM_E_UNKNOWN_SCHEDULE: throw unknown_schedule_error(w);
        case WM_E_PARSE: throw parse_error(w);
        case WM_E_CONTRACT_VIOLATION: throw contract_violation_error(w);
        case WM_E_UNKNOWN_SLOT: throw unknown_slot_error(w);
        default: throw device_error(w);
    }
}

inline int& device_ordinal() {
    static int d = 0;
    return d;
}
inline void set_device(int d) { device_ordinal() = d; }

// one context per modulus, created on first use
inline wm_ctx* context(std::uint32_t p) {
    static std::mutex mu;
    static std::map<std::uint32_t, wm_ctx*> ctxs;
    std::lock_guard<std::mutex> g(mu);
    auto it = ctxs.find(p);
    if (it != ctxs.end()) return it->second;
    wm_ctx* c = nullptr;
    check(wm_ctx_create(device_ordinal(), p, WM_FIELD_MODP, nullptr, &c));
    ctxs[p] = c;
    return c;
}
}  // namespace b200

// ---- ring (ring.hpp:47-228) ----------------------------------------------
class Modulus {
  public:
    explicit Modulus(std::uint32_t p) : p_(p) {
        if (p <= 2 || p >= (1u << 31) || !is_prime(p))
            throw dimension_error("modulus must be an odd prime in (2, 2^31): " + std::to_string(p));
    }
    std::uint32_t p() const { return p_; }
    Elem minus_one() const { return p_ - 1; }
    Elem reduce_u64(std::uint64_t x) const { return static_cast<Elem>(x % p_); }
    Elem reduce_i64(std::int64_t x) const {
        const std::int64_t r = x % static_cast<std::int64_t>(p_);
        return static_cast<Elem>(r < 0 ? r + p_ : r);
    }
    Elem add(Elem a, Elem b) const { std::uint32_t s = a + b; return s >= p_ ? s - p_ : s; }
    Elem sub(Elem a, Elem b) const { return a >= b ? a - b : a + p_ - b; }
    Elem neg(Elem a) const { return a ? p_ - a : 0; }
    Elem mul(Elem a, Elem b) const {
        return static_cast<Elem>(static_cast<std::uint64_t>(a) * b % p_);
    }
    bool operator==(const Modulus& o) const { return p_ == o.p_; }
    static bool is_prime(std::uint32_t n) {
        if (n < 2) return false;
        if (n % 2 == 0) return n == 2;
        for (std::uint64_t d = 3; d * d <= n; d += 2)
            if (n % d == 0) return false;
        return true;
    }

  private:
    std::uint32_t p_;
};

inline constexpr std::uint32_t kDefaultModulus = 65521;

class SplitMix64 {
  public:
    explicit SplitMix64(std::uint64_t seed) : state_(seed) {}
    std::uint64_t next() {
        std::uint64_t z = (state_ += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }

  private:
    std::uint64_t state_;
};

inline std::uint64_t fnv1a64(const Elem* data, std::size_t count) {
    return wm_fnv1a64_u32(data, count);
}

// Non-owning window {ptr, rows, cols, stride, origin} into a row-major host
// buffer (ring.hpp:122-177); `origin` names the owning buffer.
struct MatView {
    Elem* ptr = nullptr;
    std::size_t rows = 0, cols = 0, stride = 0;
    const Elem* origin = nullptr;
    Elem& at(std::size_t i, std::size_t j) const { return ptr[i * stride + j]; }
    bool empty() const { return rows == 0 || cols == 0; }
    std::size_t words() const { return rows * cols; }
    MatView window(std::size_t r0, std::size_t c0, std::size_t r, std::size_t c) const {
        if (r0 + r > rows || c0 + c > cols) throw dimension_error("window exceeds view bounds");
        return MatView{ptr + r0 * stride + c0, r, c, stride, origin};
    }
    bool same_window(const MatView& o) const {
        return ptr == o.ptr && rows == o.rows && cols == o.cols && stride == o.stride;
    }
    std::size_t first_word() const { return static_cast<std::size_t>(ptr - origin); }
    std::size_t last_word() const { return first_word() + (rows - 1) * stride + cols - 1; }
    // Do the two windows share an element?  Same buffer and stride: row i of
    // this and row j of o meet iff (i - j) * stride falls strictly inside
    // (d - cols, d + o.cols), d = o.ptr - ptr; the admissible t = i - j form an
    // integer interval, intersected with (-o.rows, rows).  Other strides: word
    // spans (only provably disjoint temporaries have them).
    bool overlaps(const MatView& o) const {
        if (empty() || o.empty() || origin != o.origin) return false;
        if (stride != o.stride) return first_word() <= o.last_word() && o.first_word() <= last_word();
        const std::int64_t s = static_cast<std::int64_t>(stride);
        const std::int64_t d = static_cast<std::int64_t>(o.ptr - ptr);
        const std::int64_t lo = d - static_cast<std::int64_t>(cols) + 1;   // t*s >= lo
        const std::int64_t hi = d + static_cast<std::int64_t>(o.cols) - 1; // t*s <= hi
        auto floor_div = [](std::int64_t a, std::int64_t b) {
            return a / b - ((a % b != 0) && ((a < 0) != (b < 0)));
        };
        const std::int64_t tmin = std::max(-floor_div(-lo, s), 1 - static_cast<std::int64_t>(o.rows));
        const std::int64_t tmax = std::min(floor_div(hi, s), static_cast<std::int64_t>(rows) - 1);
        return tmin <= tmax;
    }
    bool disjoint(const MatView& o) const { return !overlaps(o); }
};

// quad_split (ring.hpp:222-228): the four half-size windows, no data moves
inline std::array<MatView, 4> quad_split(const MatView& v) {
    if (v.rows % 2 || v.cols % 2) throw odd_dimension_error("quad_split requires even dimensions");
    const std::size_t r = v.rows / 2, c = v.cols / 2;
    return {v.window(0, 0, r, c), v.window(0, c, r, c), v.window(r, 0, r, c),
            v.window(r, c, r, c)};
}

class Matrix {
  public:
    Matrix(std::size_t rows, std::size_t cols, Modulus mod)
        : rows_(rows), cols_(cols), mod_(mod), data_(rows * cols, 0) {
        if (rows == 0 || cols == 0) throw dimension_error("matrix dimensions must be positive");
    }
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    const Modulus& mod() const { return mod_; }
    Elem* data() { return data_.data(); }
    const Elem* data() const { return data_.data(); }
    std::size_t size() const { return data_.size(); }
    Elem& at(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
    Elem at(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
    MatView view() { return MatView{data_.data(), rows_, cols_, cols_, data_.data()}; }
    void fill_random(std::uint64_t seed) {
        SplitMix64 g(seed);
        for (auto& x : data_) x = static_cast<Elem>(g.next() % mod_.p());
    }
    void fill_zero() { std::fill(data_.begin(), data_.end(), 0); }
    std::uint64_t hash() const { return fnv1a64(data_.data(), data_.size()); }
    bool operator==(const Matrix& o) const {
        return rows_ == o.rows_ && cols_ == o.cols_ && mod_ == o.mod_ && data_ == o.data_;
    }

  private:
    std::size_t rows_, cols_;
    Modulus mod_;
    std::vector<Elem> data_;
};

// ---- meter (meter.hpp) -----------------------------------------------------
struct AllocEvent {
    std::uint64_t words = 0;
    int depth = 0;
    std::string slot;
};

class CostMeter {
  public:
    std::uint64_t mults = 0, adds = 0, word_moves = 0;
    std::uint64_t live_extra_words = 0, peak_extra_words = 0, total_alloc_words = 0;
    std::uint64_t classical_calls = 0;
    std::vector<AllocEvent> alloc_log;  // every temporary the schedule acquired
    std::map<std::string, std::uint64_t> schedule_calls;
    // device figures of the last call
    std::uint64_t peak_extra_bytes = 0, launches = 0;

    void count_mults(std::uint64_t n) { mults += n; }
    void count_adds(std::uint64_t n) { adds += n; }
    void count_moves(std::uint64_t n) { word_moves += n; }
    void on_alloc(std::uint64_t words, int depth, const std::string& slot) {
        live_extra_words += words;
        peak_extra_words = std::max(peak_extra_words, live_extra_words);
        total_alloc_words += words;
        alloc_log.push_back({words, depth, slot});
    }
    void on_free(std::uint64_t words) { live_extra_words -= words; }
    void on_classical() { ++classical_calls; }
    void on_schedule(const std::string& name) { ++schedule_calls[name]; }
};

// ---- workspaces (workspace.hpp:24-147) --------------------------------------
// The host-side scratch providers of the reference interface.  The device
// multiply plans its own HBM arena (the same LIFO frames, reported through
// CostMeter); these serve host code written against the Workspace plug-in.
class Workspace {
  public:
    virtual ~Workspace() = default;
    virtual void push_frame() = 0;
    virtual MatView acquire(std::size_t rows, std::size_t cols, int depth, const char* slot) = 0;
    virtual void pop_frame() = 0;
};

class HeapWorkspace : public Workspace {
  public:
    explicit HeapWorkspace(CostMeter* meter) : meter_(meter) {}
    void push_frame() override { frames_.emplace_back(); }
    MatView acquire(std::size_t rows, std::size_t cols, int depth, const char* slot) override {
        if (frames_.empty()) throw workspace_error("acquire outside a frame");
        frames_.back().emplace_back(rows * cols, 0);
        Elem* p = frames_.back().back().data();
        if (meter_) meter_->on_alloc(rows * cols, depth, slot ? slot : "");
        return MatView{p, rows, cols, cols, p};
    }
    void pop_frame() override {
        if (frames_.empty()) throw workspace_error("pop without frame");
        if (meter_)
            for (const auto& b : frames_.back()) meter_->on_free(b.size());
        frames_.pop_back();
    }

  private:
    CostMeter* meter_;
    std::vector<std::vector<std::vector<Elem>>> frames_;
};

class BumpWorkspace : public Workspace {
  public:
    BumpWorkspace(Elem* base, std::size_t words) : base_(base), cap_(words) {}
    void push_frame() override { marks_.push_back(used_); }
    MatView acquire(std::size_t rows, std::size_t cols, int, const char*) override {
        if (marks_.empty()) throw workspace_error("acquire outside a frame");
        const std::size_t need = rows * cols;
        if (need > cap_ - used_)
            throw workspace_error("scratch chunk exhausted: need " + std::to_string(need) +
                                  " words, free " + std::to_string(cap_ - used_));
        Elem* p = base_ + used_;
        used_ += need;
        high_ = std::max(high_, used_);
        return MatView{p, rows, cols, cols, base_};
    }
    void pop_frame() override {
        if (marks_.empty()) throw workspace_error("pop without frame");
        used_ = marks_.back();
        marks_.pop_back();
    }
    std::size_t high_water() const { return high_; }

  private:
    Elem* base_;
    std::size_t cap_, used_ = 0, high_ = 0;
    std::vector<std::size_t> marks_;
};

class QuadrantWorkspace : public Workspace {
  public:
    explicit QuadrantWorkspace(MatView donor) {
        if (donor.rows != donor.cols) throw workspace_error("quadrant workspace donor must be square");
        regions_.push_back({donor, 0});
    }
    void push_frame() override {
        Region next = {regions_.back().view, 0};
        if (regions_.back().taken) {  // descend into the free fourth quadrant
            if (next.view.rows < 2) throw workspace_error("scratch region exhausted");
            next.view = quad_split(next.view)[3];
        }
        regions_.push_back(next);
    }
    MatView acquire(std::size_t rows, std::size_t cols, int, const char* slot) override {
        Region& r = regions_.back();
        if (r.view.rows < 2 || rows > r.view.rows / 2 || cols > r.view.cols / 2)
            throw workspace_error(std::string("temporary ") + (slot ? slot : "") +
                                  " does not fit the scratch region");
        if (r.taken == 3) throw workspace_error("more than three temporaries in a frame");
        return quad_split(r.view)[r.taken++].window(0, 0, rows, cols);
    }
    void pop_frame() override {
        if (regions_.size() < 2) throw workspace_error("pop without frame");
        regions_.pop_back();
    }

  private:
    struct Region {
        MatView view;
        int taken;
    };
    std::vector<Region> regions_;
};

struct CostReport {
    std::string variant;
    std::size_t m = 0, k = 0, n = 0;
    int cutoff = 1;
    std::uint64_t mults = 0, adds = 0, peak_extra_words = 0, total_alloc_words = 0,
                  word_moves = 0;
    std::uint64_t ops() const { return mults + adds; }
    static const char* csv_header() { return "variant,m,k,n,cutoff,mults,adds,peak_extra,total_alloc"; }
    std::string csv_row() const {
        std::ostringstream os;
        os << variant << ',' << m << ',' << k << ',' << n << ',' << cutoff << ',' << mults << ','
           << adds << ',' << peak_extra_words << ',' << total_alloc_words;
        return os.str();
    }
};

struct DiffReport {
    std::vector<std::string> diffs;
    bool empty() const { return diffs.empty(); }
};

inline DiffReport compare(const CostReport& a, const CostReport& b) {
    DiffReport r;
    auto chk = [&](const char* f, std::uint64_t x, std::uint64_t y) {
        if (x != y) r.diffs.push_back(std::string(f) + ": measured=" + std::to_string(x) +
                                      " expected=" + std::to_string(y));
    };
    chk("mults", a.mults, b.mults);
    chk("adds", a.adds, b.adds);
    chk("peak_extra_words", a.peak_extra_words, b.peak_extra_words);
    chk("total_alloc_words", a.total_alloc_words, b.total_alloc_words);
    return r;
}

struct MultiplyOptions {
    Elem alpha = 1;
    Elem beta = 0;
    int cutoff = 1;
};

namespace b200 {
inline CostReport to_report(const std::string& v, std::size_t m, std::size_t k, std::size_t n,
                            int cutoff, const wm_report& r, CostMeter* meter) {
    CostReport rep;
    rep.variant = v;
    rep.m = m;
    rep.k = k;
    rep.n = n;
    rep.cutoff = cutoff;
    rep.mults = r.mults;
    rep.adds = r.adds;
    rep.peak_extra_words = r.peak_extra_words;
    rep.total_alloc_words = r.total_alloc_words;
    rep.word_moves = r.word_moves;
    if (meter) {
        meter->mults += r.mults;
        meter->adds += r.adds;
        meter->word_moves += r.word_moves;
        meter->peak_extra_words = std::max(meter->peak_extra_words, r.peak_extra_words);
        meter->total_alloc_words += r.total_alloc_words;
        meter->classical_calls += r.classical_calls;
        meter->peak_extra_bytes = r.peak_extra_bytes;
        meter->launches = r.n_launches;
        const int need = wm_plan_alloc_log(nullptr, 0);
        std::string log(static_cast<std::size_t>(need) + 1, '\0');
        wm_plan_alloc_log(&log[0], need + 1);
        log.resize(static_cast<std::size_t>(need));
        std::istringstream ls(log);
        std::string ev;
        while (std::getline(ls, ev, ';')) {
            const auto c1 = ev.find(':'), c2 = ev.find(':', c1 + 1);
            if (c1 == std::string::npos || c2 == std::string::npos) continue;
            meter->alloc_log.push_back({std::stoull(ev.substr(0, c1)),
                                        std::stoi(ev.substr(c1 + 1, c2 - c1 - 1)), ev.substr(c2 + 1)});
        }
        char buf[4096];
        wm_plan_schedule_calls(buf, sizeof(buf));
        std::string s(buf), item;
        std::istringstream is(s);
        while (std::getline(is, item, ',')) {
            auto c = item.find(':');
            if (c != std::string::npos)
                meter->schedule_calls[item.substr(0, c)] += std::stoull(item.substr(c + 1));
        }
    }
    return rep;
}
}  // namespace b200

// run_variant (drivers.hpp:213-222) -- executes on the B200
inline CostReport run_variant(const std::string& variant, Matrix& A, Matrix& B, Matrix& C,
                              const MultiplyOptions& opt = {}, CostMeter* meter = nullptr) {
    if (!(A.mod() == B.mod()) || !(A.mod() == C.mod()))
        throw dimension_error("operands use different moduli");
    if (B.rows() != A.cols() || C.rows() != A.rows() || C.cols() != B.cols())
        throw dimension_error("multiply dimensions do not conform");
    wm_report r{};
    b200::check(wm_run_variant_host_u32(b200::context(A.mod().p()), variant.c_str(), A.rows(),
                                        A.cols(), B.cols(), A.data(), B.data(), C.data(),
                                        opt.alpha, opt.beta, opt.cutoff, &r));
    return b200::to_report(variant, A.rows(), A.cols(), B.cols(), opt.cutoff, r, meter);
}

// multiply (executor.hpp:240-299)
inline CostReport multiply(const std::string& variant, Matrix& A, Matrix& B, Matrix& C,
                           const MultiplyOptions& opt = {}, CostMeter* meter = nullptr) {
    return run_variant(variant, A, B, C, opt, meter);
}

// ipmm / ipovmm (drivers.hpp:52-158)
inline CostReport ipmm(Matrix& A, Matrix& B, Matrix& C, int cutoff = 1, CostMeter* meter = nullptr) {
    return run_variant("ipmm", A, B, C, {1, 0, cutoff}, meter);
}
inline CostReport ipovmm(Matrix& A, Matrix& B, Matrix& C, int cutoff = 1,
                         CostMeter* meter = nullptr) {
    return run_variant("ipovmm", A, B, C, {1, 0, cutoff}, meter);
}
inline CostReport blocked_acc(Matrix& A, Matrix& B, Matrix& C, Elem alpha, Elem beta, int t,
                              const std::string& base = "acc3", int cutoff = 1,
                              CostMeter* meter = nullptr) {
    const std::string v = "blocked_acc_t" + std::to_string(t) + (base == "acc2" ? "_acc2" : "");
    if (base != "acc3" && base != "acc2")
        throw unknown_schedule_error("blocked_acc base must be acc3 or acc2");
    return run_variant(v, A, B, C, {alpha, beta, cutoff}, meter);
}

// classical_mul (ring.hpp:315-384) on whole matrices
inline void classical_mul(Matrix& C, Matrix& A, Matrix& B, Elem alpha, Elem beta) {
    run_variant("classic", A, B, C, {alpha, beta, 1});
}

// ---- the primitive operators on host views (ring.hpp:241-384) ---------------
// Each call checks the reference's aliasing rules on the host views, stages the
// windows on the device (one strided copy each; a window that exactly aliases
// another shares its device copy), runs the sm_100a kernel and writes the
// destination window back.  Metering follows the reference call for call.
namespace b200 {
struct DeviceWindow {
    wm_dmat d{};
    explicit DeviceWindow(const MatView& v, bool upload, wm_ctx* ctx) {
        check(wm_dev_alloc(ctx, v.rows * v.cols, &d.ptr));
        d.rows = v.rows;
        d.cols = v.cols;
        d.ld = v.cols;
        if (upload) check(wm_upload_u32(ctx, d, v.ptr, v.stride));
    }
    void download(const MatView& v, wm_ctx* ctx) const {
        check(wm_download_u32(ctx, v.ptr, v.stride, d));
    }
    DeviceWindow(const DeviceWindow&) = delete;
    DeviceWindow& operator=(const DeviceWindow&) = delete;
    ~DeviceWindow() { wm_dev_free(d.ptr); }
};
inline bool trivial_scalar(Elem s, const Modulus& mod) {
    return s == 0 || s == 1 || s == mod.minus_one();
}
}  // namespace b200

inline void block_addsub(MatView dst, MatView a, MatView b, Elem sa, Elem sb, const Modulus& mod,
                         CostMeter* meter = nullptr) {
    if (a.rows != b.rows || a.cols != b.cols || dst.rows != a.rows || dst.cols != a.cols)
        throw dimension_error("block_addsub dimension mismatch");
    if (!dst.same_window(a) && dst.overlaps(a))
        throw partial_overlap_error("block_addsub: dst partially overlaps a");
    if (!dst.same_window(b) && dst.overlaps(b))
        throw partial_overlap_error("block_addsub: dst partially overlaps b");
    wm_ctx* ctx = b200::context(mod.p());
    b200::DeviceWindow da(a, true, ctx);
    std::optional<b200::DeviceWindow> db, dd;
    if (!b.same_window(a)) db.emplace(b, true, ctx);
    const wm_dmat& bd = db ? db->d : da.d;
    const wm_dmat* dstd = dst.same_window(a) ? &da.d : dst.same_window(b) ? &bd : nullptr;
    if (!dstd) {
        dd.emplace(dst, false, ctx);
        dstd = &dd->d;
    }
    b200::check(wm_block_addsub(ctx, *dstd, da.d, bd, sa, sb));
    b200::check(wm_download_u32(ctx, dst.ptr, dst.stride, *dstd));
    if (meter) {
        meter->count_adds(dst.words());
        if (!b200::trivial_scalar(sa, mod)) meter->count_mults(dst.words());
        if (!b200::trivial_scalar(sb, mod)) meter->count_mults(dst.words());
    }
}

inline void block_scale_copy(MatView dst, MatView src, Elem s, const Modulus& mod,
                             CostMeter* meter = nullptr) {
    if (dst.rows != src.rows || dst.cols != src.cols)
        throw dimension_error("block_scale_copy dimension mismatch");
    if (!dst.same_window(src) && dst.overlaps(src))
        throw partial_overlap_error("block_scale_copy: dst partially overlaps src");
    wm_ctx* ctx = b200::context(mod.p());
    b200::DeviceWindow ds(src, true, ctx);
    std::optional<b200::DeviceWindow> dd;
    if (!dst.same_window(src)) dd.emplace(dst, false, ctx);
    const wm_dmat& dstd = dd ? dd->d : ds.d;
    b200::check(wm_block_scale_copy(ctx, dstd, ds.d, s));
    b200::check(wm_download_u32(ctx, dst.ptr, dst.stride, dstd));
    if (meter) {
        if (s == 1 || s == mod.minus_one()) meter->count_moves(dst.words());
        else meter->count_mults(dst.words());
    }
}

inline void classical_mul(MatView C, MatView A, MatView B, Elem alpha, Elem beta,
                          const Modulus& mod, CostMeter* meter = nullptr) {
    const std::size_t m = A.rows, k = A.cols, n = B.cols;
    if (B.rows != k || C.rows != m || C.cols != n)
        throw dimension_error("classical_mul dimension mismatch");
    if (C.overlaps(A) || C.overlaps(B))
        throw alias_error("classical_mul: C must be disjoint from A and B");
    wm_ctx* ctx = b200::context(mod.p());
    b200::DeviceWindow da(A, true, ctx), dc(C, beta != 0, ctx);
    std::optional<b200::DeviceWindow> db;
    if (!B.same_window(A)) db.emplace(B, true, ctx);
    b200::check(wm_classical_mul(ctx, dc.d, da.d, db ? db->d : da.d, alpha, beta));
    dc.download(C, ctx);
    if (meter) {
        meter->on_classical();
        meter->count_mults(static_cast<std::uint64_t>(m) * k * n);
        meter->count_adds(static_cast<std::uint64_t>(m) * n * (k - 1));
        if (beta != 0) meter->count_adds(static_cast<std::uint64_t>(m) * n);
        if (!b200::trivial_scalar(alpha, mod)) meter->count_mults(static_cast<std::uint64_t>(m) * n);
        if (!b200::trivial_scalar(beta, mod)) meter->count_mults(static_cast<std::uint64_t>(m) * n);
    }
}

// ---- schedule DSL (schedule.hpp:261-684, executor.hpp:304-342) -------------
// A parsed schedule is carried as its validated text; the device planner
// re-reads it (it is small) at each run.
// schedule.hpp:185-211
enum class Contract : std::uint8_t { ReadOnly, OverwriteA, OverwriteB, OverwriteBoth };
inline const char* contract_name(Contract c) {
    switch (c) {
        case Contract::ReadOnly: return "read-only";
        case Contract::OverwriteA: return "overwrite-A";
        case Contract::OverwriteB: return "overwrite-B";
        case Contract::OverwriteBoth: return "overwrite-both";
    }
    return "?";
}

struct Schedule {
    std::string name;
    std::string text;       // canonical rendering (parses back to the same schedule)
    bool builtin_match = false;
    // header fields of the rendering (schedule.hpp:219-224)
    Contract contract = Contract::ReadOnly;
    bool accumulating = false;
    bool square_only = true;
};

namespace b200 {
inline Schedule from_rendering(const std::string& text) {
    Schedule s;
    s.text = text;
    std::istringstream is(text);
    std::string line;
    while (std::getline(is, line)) {
        std::istringstream ls(line);
        std::string key, val;
        ls >> key >> val;
        if (key == "schedule") s.name = val;
        else if (key == "accumulating") s.accumulating = val == "true";
        else if (key == "shape") s.square_only = val == "square";
        else if (key == "contract")
            for (Contract c : {Contract::ReadOnly, Contract::OverwriteA, Contract::OverwriteB,
                               Contract::OverwriteBoth})
                if (val == contract_name(c)) s.contract = c;
    }
    return s;
}
}  // namespace b200

inline Schedule parse_schedule(const std::string& text) {
    int need = 0, match = 0;
    b200::check(wm_parse_schedule(text.c_str(), nullptr, 0, &need, &match));
    std::string out(static_cast<std::size_t>(need) + 1, '\0');
    b200::check(wm_parse_schedule(text.c_str(), &out[0], need + 1, &need, &match));
    out.resize(static_cast<std::size_t>(need));
    Schedule s = b200::from_rendering(out);
    s.builtin_match = match != 0;
    return s;
}

inline std::string render_schedule(const Schedule& s) { return s.text; }

inline Schedule builtin(const std::string& name) {
    int need = 0;
    b200::check(wm_render_schedule(name.c_str(), nullptr, 0, &need));
    std::string out(static_cast<std::size_t>(need) + 1, '\0');
    b200::check(wm_render_schedule(name.c_str(), &out[0], need + 1, &need));
    out.resize(static_cast<std::size_t>(need));
    Schedule s = b200::from_rendering(out);
    s.builtin_match = true;
    return s;
}

inline CostReport run_parsed_schedule(const Schedule& s, Matrix& A, Matrix& B, Matrix& C,
                                      const MultiplyOptions& opt = {},
                                      CostMeter* meter = nullptr) {
    if (B.rows() != A.cols() || C.rows() != A.rows() || C.cols() != B.cols())
        throw dimension_error("multiply dimensions do not conform");
    wm_report r{};
    b200::check(wm_run_parsed_schedule_host_u32(b200::context(A.mod().p()), s.text.c_str(),
                                                A.rows(), A.cols(), B.cols(), A.data(), B.data(),
                                                C.data(), opt.alpha, opt.beta, opt.cutoff, &r));
    return b200::to_report(s.name, A.rows(), A.cols(), B.cols(), opt.cutoff, r, meter);
}

// ---- matrix file formats (ring.hpp:386-449), on the host Matrix --------------
// Text: "rows cols p" then rows*cols residues; binary: little-endian u64
// (rows, cols, p) then u64 residues.  io_error on a bad header, truncation or
// a non-canonical entry.  (wm_matrix_read_device / _write_device move files
// straight to and from device matrices.)
inline void write_text(const Matrix& a, std::ostream& os) {
    os << a.rows() << ' ' << a.cols() << ' ' << a.mod().p() << '\n';
    for (std::size_t i = 0; i < a.rows(); ++i) {
        for (std::size_t j = 0; j < a.cols(); ++j) os << (j ? " " : "") << a.at(i, j);
        os << '\n';
    }
}

inline Matrix read_text(std::istream& is) {
    std::uint64_t r, c, p;
    if (!(is >> r >> c >> p)) throw io_error("bad matrix text header");
    Matrix a(r, c, Modulus(static_cast<std::uint32_t>(p)));
    for (std::size_t i = 0; i < r; ++i)
        for (std::size_t j = 0; j < c; ++j) {
            std::uint64_t v;
            if (!(is >> v)) throw io_error("matrix text truncated");
            if (v >= p) throw io_error("matrix entry not a canonical residue");
            a.at(i, j) = static_cast<Elem>(v);
        }
    return a;
}

namespace b200 {
inline void put_le(std::ostream& os, std::uint64_t v) {
    char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<char>(v >> (8 * i));
    os.write(b, 8);
}
inline std::uint64_t get_le(std::istream& is) {
    unsigned char b[8];
    is.read(reinterpret_cast<char*>(b), 8);
    if (!is) throw io_error("matrix binary truncated");
    std::uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<std::uint64_t>(b[i]) << (8 * i);
    return v;
}
}  // namespace b200

inline void write_binary(const Matrix& a, std::ostream& os) {
    b200::put_le(os, a.rows());
    b200::put_le(os, a.cols());
    b200::put_le(os, a.mod().p());
    for (std::size_t i = 0; i < a.rows() * a.cols(); ++i) b200::put_le(os, a.data()[i]);
}

inline Matrix read_binary(std::istream& is) {
    const std::uint64_t r = b200::get_le(is), c = b200::get_le(is), p = b200::get_le(is);
    Matrix a(r, c, Modulus(static_cast<std::uint32_t>(p)));
    for (std::size_t i = 0; i < r * c; ++i) {
        const std::uint64_t v = b200::get_le(is);
        if (v >= p) throw io_error("matrix entry not a canonical residue");
        a.data()[i] = static_cast<Elem>(v);
    }
    return a;
}

namespace models {
// "blocked_acc_t<T>[_acc2]" (models.hpp:180-200)
struct BlockedSpec {
    int t = 1;
    std::string base = "acc3";
};
inline std::optional<BlockedSpec> parse_blocked(const std::string& v) {
    const std::string pre = "blocked_acc_t";
    if (v.compare(0, pre.size(), pre) != 0) return std::nullopt;
    std::size_t i = pre.size();
    while (i < v.size() && v[i] >= '0' && v[i] <= '9') ++i;
    if (i == pre.size()) return std::nullopt;
    BlockedSpec b;
    b.t = std::stoi(v.substr(pre.size(), i - pre.size()));
    const std::string tail = v.substr(i);
    if (tail == "_acc2") b.base = "acc2";
    else if (!tail.empty()) return std::nullopt;
    return b;
}

// expected_costs (models.hpp:202-229)
inline CostReport expected_costs(const std::string& variant, std::size_t m, std::size_t k,
                                 std::size_t n, int cutoff) {
    wm_report r{};
    b200::check(wm_expected_costs(variant.c_str(), m, k, n, cutoff, &r));
    return b200::to_report(variant, m, k, n, cutoff, r, nullptr);
}
}  // namespace models

// Host-only plan: the exact CostReport the reference meter would produce.
inline CostReport plan_only(const std::string& variant, std::size_t m, std::size_t k,
                            std::size_t n, const MultiplyOptions& opt = {},
                            std::uint32_t p = kDefaultModulus) {
    wm_report r{};
    b200::check(wm_plan_report(variant.c_str(), WM_FIELD_MODP, p, m, k, n, opt.alpha, opt.beta,
                               opt.cutoff, 0, &r));
    return b200::to_report(variant, m, k, n, opt.cutoff, r, nullptr);
}

inline const std::vector<std::string>& builtin_names() {
    static const std::vector<std::string> n = {"std2", "acc3", "ip",   "ovl",  "ovl2",
                                               "ovr",  "aclr", "accr", "acc2", "acr"};
    return n;
}

inline bool variant_accumulates(const std::string& v) {
    if (v == "ipmm" || v == "ipovmm" || v == "iprect" || v == "classic") return false;
    if (v.rfind("blocked_acc_t", 0) == 0) return true;
    for (const char* a : {"acc3", "aclr", "accr", "acc2", "acr"})
        if (v == a) return true;
    for (const auto& b : builtin_names())
        if (v == b) return false;
    throw unknown_schedule_error("unknown schedule: " + v);
}

}  // namespace winomem
