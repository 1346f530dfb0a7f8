// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// A C-ABI shim over the UNMODIFIED reference headers (winomem, header-only
// C++20, /root/reference/proj/include).  The Makefile in this directory
// compiles it with the reference's own Release flags (-O3 -DNDEBUG,
// proj/CMakeLists.txt:9-11) into oracle/_ref/libwinomem_ref.so.  Tests use it
// to pin the CPU restatement (wm_oracle.c) and the product planner's metering;
// bench.py's cpu_baseline / --impl reference legs time it.
//
// Entry points mirror the reference API they wrap:
//   ref_run_variant      -> winomem::run_variant   (inc/drivers.hpp:213-222)
//   ref_expected_costs   -> models::expected_costs (inc/models.hpp:202-229)
//   ref_classical_mul    -> winomem::classical_mul (inc/ring.hpp:315-384)
//   ref_block_addsub     -> winomem::block_addsub  (inc/ring.hpp:241-278)
//   ref_fill_random      -> Matrix::fill_random    (inc/ring.hpp:202-205)
//   ref_hash             -> fnv1a64                (inc/ring.hpp:107-114)
#include <fstream>
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>

#include "winomem/winomem.hpp"

using namespace winomem;

namespace {
// status codes shared with include/winomem_b200.h (WM_E_*)
int code_of(const std::exception& e) {
    if (dynamic_cast<const odd_dimension_error*>(&e)) return 2;
    if (dynamic_cast<const dimension_error*>(&e)) return 1;
    if (dynamic_cast<const partial_overlap_error*>(&e)) return 3;
    if (dynamic_cast<const alias_error*>(&e)) return 4;
    if (dynamic_cast<const shape_error*>(&e)) return 5;
    if (dynamic_cast<const contract_error*>(&e)) return 6;
    if (dynamic_cast<const io_error*>(&e)) return 7;
    if (dynamic_cast<const workspace_error*>(&e)) return 8;
    if (dynamic_cast<const unknown_schedule_error*>(&e)) return 9;
    if (dynamic_cast<const parse_error*>(&e)) return 10;
    if (dynamic_cast<const contract_violation_error*>(&e)) return 11;
    return 99;
}
void put_err(char* err, int len, const char* msg) {
    if (err && len > 0) {
        std::strncpy(err, msg, static_cast<std::size_t>(len) - 1);
        err[len - 1] = 0;
    }
}
void fill_report(const CostReport& r, const CostMeter* m, std::uint64_t* out) {
    if (!out) return;
    out[0] = r.mults;
    out[1] = r.adds;
    out[2] = r.peak_extra_words;
    out[3] = r.total_alloc_words;
    out[4] = r.word_moves;
    out[5] = m ? m->classical_calls : 0;
}
}  // namespace

extern "C" {

// report_out[6] = {mults, adds, peak_extra_words, total_alloc_words,
//                  word_moves, classical_calls}
// sched_out (optional) receives "name:count,name:count" of schedule_calls.
int ref_run_variant(const char* variant, std::uint64_t m, std::uint64_t k,
                    std::uint64_t n, std::uint32_t p, std::uint32_t* A,
                    std::uint32_t* B, std::uint32_t* C, std::uint32_t alpha,
                    std::uint32_t beta, int cutoff, std::uint64_t* report_out,
                    char* sched_out, int sched_len, char* err, int errlen) {
    try {
        Modulus mod(p);
        Matrix Am(m, k, mod), Bm(k, n, mod), Cm(m, n, mod);
        std::memcpy(Am.data(), A, m * k * sizeof(Elem));
        std::memcpy(Bm.data(), B, k * n * sizeof(Elem));
        std::memcpy(Cm.data(), C, m * n * sizeof(Elem));
        CostMeter meter;
        MultiplyOptions opt;
        opt.alpha = alpha;
        opt.beta = beta;
        opt.cutoff = cutoff;
        CostReport r = run_variant(variant, Am, Bm, Cm, opt, &meter);
        std::memcpy(A, Am.data(), m * k * sizeof(Elem));
        std::memcpy(B, Bm.data(), k * n * sizeof(Elem));
        std::memcpy(C, Cm.data(), m * n * sizeof(Elem));
        fill_report(r, &meter, report_out);
        if (sched_out && sched_len > 0) {
            std::string s;
            for (const auto& kv : meter.schedule_calls) {
                if (!s.empty()) s += ",";
                s += kv.first + ":" + std::to_string(kv.second);
            }
            put_err(sched_out, sched_len, s.c_str());
        }
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return code_of(e);
    }
}

// run_parsed_schedule (executor.hpp:304-342) of a DSL text with the reference's
// own parser (schedule.hpp:679-684) on u32 matrices.
int ref_run_parsed(const char* text, std::uint64_t m, std::uint64_t k, std::uint64_t n,
                   std::uint32_t p, std::uint32_t* A, std::uint32_t* B, std::uint32_t* C,
                   std::uint32_t alpha, std::uint32_t beta, int cutoff, std::uint64_t* report_out,
                   char* err, int errlen) {
    try {
        Modulus mod(p);
        Matrix Am(m, k, mod), Bm(k, n, mod), Cm(m, n, mod);
        std::memcpy(Am.data(), A, m * k * sizeof(Elem));
        std::memcpy(Bm.data(), B, k * n * sizeof(Elem));
        std::memcpy(Cm.data(), C, m * n * sizeof(Elem));
        CostMeter meter;
        MultiplyOptions opt;
        opt.alpha = alpha;
        opt.beta = beta;
        opt.cutoff = cutoff;
        Schedule s = parse_schedule(text);
        CostReport r = run_parsed_schedule(s, Am, Bm, Cm, opt, &meter);
        std::memcpy(A, Am.data(), m * k * sizeof(Elem));
        std::memcpy(B, Bm.data(), k * n * sizeof(Elem));
        std::memcpy(C, Cm.data(), m * n * sizeof(Elem));
        fill_report(r, &meter, report_out);
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return code_of(e);
    }
}

int ref_expected_costs(const char* variant, std::uint64_t m, std::uint64_t k,
                       std::uint64_t n, int cutoff, std::uint64_t* report_out,
                       char* err, int errlen) {
    try {
        CostReport r = models::expected_costs(variant, m, k, n, cutoff);
        fill_report(r, nullptr, report_out);
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return code_of(e);
    }
}

int ref_classical_mul(std::uint64_t m, std::uint64_t k, std::uint64_t n,
                      std::uint32_t p, const std::uint32_t* A, const std::uint32_t* B,
                      std::uint32_t* C, std::uint32_t alpha, std::uint32_t beta) {
    try {
        Modulus mod(p);
        Matrix Am(m, k, mod), Bm(k, n, mod), Cm(m, n, mod);
        std::memcpy(Am.data(), A, m * k * sizeof(Elem));
        std::memcpy(Bm.data(), B, k * n * sizeof(Elem));
        std::memcpy(Cm.data(), C, m * n * sizeof(Elem));
        classical_mul(Cm.view(), Am.view(), Bm.view(), alpha, beta, mod);
        std::memcpy(C, Cm.data(), m * n * sizeof(Elem));
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_block_addsub(std::uint64_t r, std::uint64_t c, std::uint32_t p,
                     const std::uint32_t* a, const std::uint32_t* b, std::uint32_t* dst,
                     std::uint32_t sa, std::uint32_t sb) {
    try {
        Modulus mod(p);
        Matrix Am(r, c, mod), Bm(r, c, mod), Dm(r, c, mod);
        std::memcpy(Am.data(), a, r * c * sizeof(Elem));
        std::memcpy(Bm.data(), b, r * c * sizeof(Elem));
        block_addsub(Dm.view(), Am.view(), Bm.view(), sa, sb, mod);
        std::memcpy(dst, Dm.data(), r * c * sizeof(Elem));
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// One primitive on windows of ONE buffer (rows x cols, row-major): the
// aliasing / overlap rules of block_addsub, block_scale_copy and classical_mul
// (ring.hpp:241-384) need views that share storage.  op 0 = block_addsub(dst, a,
// b, s0, s1), 1 = block_scale_copy(dst, a, s0), 2 = classical_mul(dst, a, b, s0,
// s1); win = {r0, c0, rows, cols} for dst, a, b.  The buffer is updated in place.
int ref_primitive_on_windows(int op, std::uint64_t rows, std::uint64_t cols, std::uint32_t p,
                             std::uint32_t* buf, const std::uint64_t* win, std::uint32_t s0,
                             std::uint32_t s1, char* err, int errlen) {
    try {
        Modulus mod(p);
        Matrix M(rows, cols, mod);
        std::memcpy(M.data(), buf, rows * cols * sizeof(Elem));
        auto w = [&](int i) { return M.view().window(win[4 * i], win[4 * i + 1], win[4 * i + 2],
                                                     win[4 * i + 3]); };
        if (op == 0) block_addsub(w(0), w(1), w(2), s0, s1, mod);
        else if (op == 1) block_scale_copy(w(0), w(1), s0, mod);
        else classical_mul(w(0), w(1), w(2), s0, s1, mod);
        std::memcpy(buf, M.data(), rows * cols * sizeof(Elem));
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return code_of(e);
    }
}

// run_variant with a CostMeter: its alloc_log (meter.hpp:15-19, 40-45) as
// "words:depth:slot;..." (returns the full length, or -code on an exception)
int ref_alloc_log(const char* variant, std::uint64_t m, std::uint64_t k, std::uint64_t n,
                  std::uint32_t alpha, std::uint32_t beta, int cutoff, char* out, int len) {
    try {
        Modulus mod(65521);
        Matrix A(m, k, mod), B(k, n, mod), C(m, n, mod);
        A.fill_random(1);
        B.fill_random(2);
        C.fill_random(3);
        CostMeter meter;
        MultiplyOptions opt;
        opt.alpha = alpha;
        opt.beta = beta;
        opt.cutoff = cutoff;
        run_variant(variant, A, B, C, opt, &meter);
        std::string text;
        for (const auto& e : meter.alloc_log)
            text += std::to_string(e.words) + ":" + std::to_string(e.depth) + ":" + e.slot + ";";
        put_err(out, len, text.c_str());
        return static_cast<int>(text.size());
    } catch (const std::exception& e) {
        return -code_of(e);
    }
}

void ref_fill_random(std::uint32_t* out, std::uint64_t count, std::uint64_t seed,
                     std::uint32_t p) {
    SplitMix64 g(seed);
    for (std::uint64_t i = 0; i < count; ++i) out[i] = static_cast<Elem>(g.next() % p);
}

std::uint64_t ref_hash(const std::uint32_t* data, std::uint64_t count) {
    return fnv1a64(data, count);
}

// The builtin schedule catalog as the reference renders it (for the
// planner's catalog-equivalence test).
int ref_render_builtin(const char* name, char* out, int len) {
    try {
        std::string s = render_schedule(builtin(name));
        put_err(out, len, s.c_str());
        return static_cast<int>(s.size());
    } catch (const std::exception& e) {
        return -code_of(e);
    }
}

// Matrix file formats (ring.hpp:386-449): write a matrix with the reference's
// writers / read one back with its readers (status < 0: exception code).
int ref_write_matrix(const char* path, int binary, std::uint64_t rows, std::uint64_t cols,
                     std::uint32_t p, const std::uint32_t* data) {
    try {
        Matrix a(rows, cols, Modulus(p));
        std::copy(data, data + rows * cols, a.data());
        std::ofstream os(path, binary ? std::ios::binary : std::ios::out);
        if (binary) write_binary(a, os);
        else write_text(a, os);
        return 0;
    } catch (const std::exception& e) {
        return -code_of(e);
    }
}

int ref_read_matrix(const char* path, int binary, std::uint64_t* rows, std::uint64_t* cols,
                    std::uint32_t* p, std::uint32_t* out, std::uint64_t cap) {
    try {
        std::ifstream is(path, binary ? std::ios::binary : std::ios::in);
        Matrix a = binary ? read_binary(is) : read_text(is);
        *rows = a.rows();
        *cols = a.cols();
        *p = a.mod().p();
        if (out && a.size() <= cap) std::copy(a.data(), a.data() + a.size(), out);
        return 0;
    } catch (const std::exception& e) {
        return -code_of(e);
    }
}

}  // extern "C"
