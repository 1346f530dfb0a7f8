// Shared host types for the winomem-b200 planner and runtime.
//
// The planner is a restatement of the reference interpreter
// (/root/reference/proj/include/winomem/executor.hpp:82-205) that, instead of
// touching memory, emits a static list of device operations over four HBM
// regions: the caller's A, B, C (float64, row-major with a leading dimension)
// and one pre-sized temporary arena.  Views are therefore (region, element
// offset, rows, cols, ld) rather than raw pointers; the overlap rules of
// MatView (ring.hpp:122-177) are reproduced on those offsets.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace wm {

// Status codes: the reference exception taxonomy (ring.hpp:23-43,
// workspace.hpp:20-22, schedule.hpp:30-43) plus device/communication errors.
enum Status : int {
    S_OK = 0,
    E_DIMENSION = 1,
    E_ODD_DIMENSION = 2,
    E_PARTIAL_OVERLAP = 3,
    E_ALIAS = 4,
    E_SHAPE = 5,
    E_CONTRACT = 6,
    E_IO = 7,
    E_WORKSPACE = 8,
    E_UNKNOWN_SCHEDULE = 9,
    E_PARSE = 10,
    E_CONTRACT_VIOLATION = 11,
    E_CUDA = 12,
    E_NCCL = 13,
    E_INVALID = 14,
    E_UNKNOWN_SLOT = 15,  // unknown_slot_error (schedule.hpp:34-36)
};

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& what) { throw Error(code, what); }

// Field of the computation.  MODP: canonical residues mod an odd prime p < 2^16
// held exactly in float64 (BASELINE configs 1-4).  REAL64: plain float64
// (config 5).  Scalars carry both representations; the field picks one.
struct Scalar {
    std::uint32_t r = 0;  // residue (MODP)
    double d = 0.0;       // value (REAL64)
};

struct Field {
    bool real = false;
    std::uint32_t p = 65521;

    Scalar zero() const { return {0u, 0.0}; }
    Scalar one() const { return {1u, 1.0}; }
    Scalar neg(Scalar s) const { return {s.r ? p - s.r : 0u, -s.d}; }
    Scalar mul(Scalar a, Scalar b) const {
        return {static_cast<std::uint32_t>(static_cast<std::uint64_t>(a.r) * b.r % p),
                a.d * b.d};
    }
    bool is_zero(Scalar s) const { return real ? s.d == 0.0 : s.r == 0; }
    bool is_one(Scalar s) const { return real ? s.d == 1.0 : s.r == 1; }
    bool is_minus_one(Scalar s) const { return real ? s.d == -1.0 : s.r == p - 1; }
    // ring.hpp:232-236: magnitude-one and zero scalars cost no multiplication
    bool trivial(Scalar s) const { return is_zero(s) || is_one(s) || is_minus_one(s); }
};

enum Region : std::uint8_t { R_A = 0, R_B = 1, R_C = 2, R_T = 3, R_NONE = 255 };

// A window over one allocation.  `origin` identifies the allocation (the
// reference compares MatView::origin pointers): 0/1/2 for the caller's
// A/B/C, >= 3 for a metered heap temporary.  `base` is the element offset of
// that allocation inside its region, `off` the offset of element (0,0).
struct View {
    std::uint8_t region = R_NONE;
    std::int32_t origin = -1;
    std::uint64_t base = 0;
    std::uint64_t off = 0;
    std::uint64_t rows = 0, cols = 0, ld = 0;

    bool empty() const { return rows == 0 || cols == 0; }
    std::uint64_t words() const { return rows * cols; }
    View window(std::uint64_t r0, std::uint64_t c0, std::uint64_t r, std::uint64_t c) const {
        if (r0 + r > rows || c0 + c > cols) fail(E_DIMENSION, "window exceeds view bounds");
        View v = *this;
        v.off = off + r0 * ld + c0;
        v.rows = r;
        v.cols = c;
        return v;
    }
    bool same_window(const View& o) const {
        return region == o.region && origin == o.origin && off == o.off && rows == o.rows &&
               cols == o.cols && ld == o.ld;
    }
    std::uint64_t first_word() const { return off - base; }
    std::uint64_t last_word() const { return first_word() + (rows - 1) * ld + cols - 1; }
    // Exact index-set intersection for equal strides over one allocation,
    // conservative span test otherwise -- the semantics of MatView::overlaps.
    bool overlaps(const View& o) const;
    // Physical overlap in device memory (any allocations, same region):
    // used by the launch batcher for dependency analysis.
    bool phys_overlaps(const View& o) const;
};

std::array<View, 4> quad_split(const View& v);

enum OpKind : std::uint8_t {
    OP_ADDSUB = 0,  // d <- sa*a + sb*b           (block_addsub, ring.hpp:241-278)
    OP_COPY = 1,    // d <- sa*a                  (block_scale_copy, ring.hpp:282-310)
    OP_MUL = 2,     // d <- sa*a*b + sb*d          (classical_mul, ring.hpp:315-384)
    OP_FRAME = 3,   // one fused Winograd frame over classical leaves (same contract as MUL)
};

struct Op {
    OpKind kind;
    View d, a, b;
    Scalar sa, sb;
    int depth = 0;
    // provenance: the schedule frame instance and 1-based row that emitted it
    // (frame < 0: emitted by a driver outside any schedule frame)
    int frame = -1;
    const char* sched = nullptr;
    int row = 0;
    // OP_FRAME: c x c blocks free for residue planes: h0, h1 host the seven
    // product planes, h2 (optional, rows == 0 if absent) a third temporary
    View h0, h1, h2;
};

// CostMeter (meter.hpp:24-50)
struct Meter {
    std::uint64_t mults = 0, adds = 0, word_moves = 0;
    std::uint64_t live = 0, peak = 0, total = 0;
    std::uint64_t classical_calls = 0;
    std::map<std::string, std::uint64_t> schedule_calls;
    // algorithmic traffic / work, independent of fusion
    std::uint64_t add2_elems = 0;   // elements of two-term additions (3 words moved each)
    std::uint64_t copy_elems = 0;   // elements of copies / scalings (2 words each)
    std::uint64_t leaf_flops = 0;   // sum of 2*m*k*n over classical leaves
    // CostMeter::alloc_log (meter.hpp:15-19, 40-45): every metered temporary
    struct AllocEvent {
        std::uint64_t words;
        int depth;
        const char* slot;  // static slot name
    };
    std::vector<AllocEvent> alloc_log;
    void on_alloc(std::uint64_t w, int depth = 0, const char* slot = "") {
        alloc_log.push_back({w, depth, slot});
        live += w;
        if (live > peak) peak = live;
        total += w;
    }
    void on_free(std::uint64_t w) { live -= w; }
};

}  // namespace wm
