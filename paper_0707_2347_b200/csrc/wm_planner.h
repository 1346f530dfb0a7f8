// Host planner: restates the reference executor and drivers
// (/root/reference/proj/include/winomem/executor.hpp:22-299 and drivers.hpp:38-222)
// so that one call produces
//   * the exact CostMeter the reference would report (mults, adds, word moves,
//     peak / total temporary words, classical and per-schedule call counts);
//   * a static list of device operations (block additions, classical leaf
//     products, optionally fused leaf frames) over the regions A, B, C and the
//     temporary arena, in the schedule's execution order;
//   * the arena high-water mark, i.e. the HBM the schedule's temporaries need.
// Contract, aliasing and shape errors are raised with the reference taxonomy
// before any device work is issued.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "wm_schedule.h"
#include "wm_types.h"

namespace wm {

struct PlanOptions {
    // Emit one OP_FRAME for every schedule frame whose seven products are all
    // classical leaves (the fused pre-add / product / post-add kernel) instead of
    // its 15-17 additions and 7 leaf products.  Metering is unchanged: the frame
    // is still walked instruction by instruction and its temporaries are still
    // acquired in the arena.
    bool fuse_frames = false;
    // The FRAME kernels support leaf sizes that are multiples of this.
    int frame_align = 128;
    int frame_max_leaf = 1 << 20;
    // run_parsed_schedule (executor.hpp:304-342): execute this schedule at the
    // top frame instead of dispatching `variant` (recursion tags name builtins)
    const Schedule* parsed = nullptr;
};

struct Plan {
    std::string variant;
    std::uint64_t m = 0, k = 0, n = 0;
    int cutoff = 1;
    Field field;
    std::vector<Op> ops;
    Meter meter;
    std::uint64_t arena_words = 0;  // physical high-water of the temporary arena
    // the meter's allocation trace, shared (not copied) with every report of this plan
    std::shared_ptr<const std::vector<Meter::AllocEvent>> alloc_log;
};

struct Workspace {
    virtual ~Workspace() = default;
    virtual void push_frame() = 0;
    virtual View acquire(std::uint64_t rows, std::uint64_t cols, int depth, const char* slot) = 0;
    virtual void pop_frame() = 0;
};

// HeapWorkspace (workspace.hpp:34-64) over one pre-sized device arena: LIFO bump
// frames; every acquisition is metered and gets its own allocation identity.
class ArenaWorkspace : public Workspace {
  public:
    explicit ArenaWorkspace(Meter* m) : meter_(m) {}
    void push_frame() override;
    View acquire(std::uint64_t rows, std::uint64_t cols, int depth, const char* slot) override;
    void pop_frame() override;
    std::uint64_t high_water() const { return high_; }

  private:
    Meter* meter_;
    std::vector<std::uint64_t> marks_;
    std::vector<std::vector<std::uint64_t>> words_;
    std::uint64_t used_ = 0, high_ = 0;
    std::int32_t next_origin_ = 3;
};

// BumpWorkspace (workspace.hpp:68-101): LIFO over one preallocated chunk; not metered.
class BumpWorkspace : public Workspace {
  public:
    BumpWorkspace(View chunk) : chunk_(chunk) {}
    void push_frame() override { marks_.push_back(used_); }
    View acquire(std::uint64_t rows, std::uint64_t cols, int depth, const char* slot) override;
    void pop_frame() override;

  private:
    View chunk_;
    std::uint64_t used_ = 0;
    std::vector<std::uint64_t> marks_;
};

// QuadrantWorkspace (workspace.hpp:107-147): carves up to three half-quadrants of
// a square donor per frame and descends into the fourth.  Not metered.
class QuadrantWorkspace : public Workspace {
  public:
    explicit QuadrantWorkspace(View donor);
    void push_frame() override;
    View acquire(std::uint64_t rows, std::uint64_t cols, int depth, const char* slot) override;
    void pop_frame() override;

  private:
    struct Frame {
        View region;
        int used;
    };
    std::vector<Frame> frames_;
};

// Plan C <- alpha*A*B + beta*C for `variant` (a builtin schedule, "classic",
// "ipmm", "ipovmm", "iprect" or "blocked_acc_t<T>[_acc2]"), the dispatch of
// run_variant (drivers.hpp:213-222).  A is m x k (ld lda), B k x n, C m x n.
Plan plan_variant(const std::string& variant, Field f, std::uint64_t m, std::uint64_t k,
                  std::uint64_t n, std::uint64_t lda, std::uint64_t ldb, std::uint64_t ldc,
                  Scalar alpha, Scalar beta, int cutoff, const PlanOptions& opt);

// Expected costs of a variant (the reference's models.hpp:202-229 answers the
// same question); wm_costs.cpp derives them from the schedule IR.
struct Costs {
    std::uint64_t mults = 0, adds = 0, peak = 0, total = 0, moves = 0;
};
Costs expected_costs(const std::string& variant, std::uint64_t m, std::uint64_t k,
                     std::uint64_t n, int cutoff);

// "blocked_acc_t<T>[_acc2]" -> T and the base schedule (acc3 / acc2)
bool parse_blocked(const std::string& variant, int* t, std::string* base);
// Config-3 composition: the schedule for block (i, j) of an mb x nb grid of squares.
const char* iprect_block_variant(std::uint64_t i, std::uint64_t j, std::uint64_t mb,
                                 std::uint64_t nb);

bool variant_accumulates(const std::string& variant);
Contract variant_contract(const std::string& variant);

}  // namespace wm
