// Runtime and C-ABI (include/winomem_b200.h).
//
// A context owns one CUDA stream.  A call plans the multiplication on the host
// (wm_planner.cpp), lowers the operation list to launches -- consecutive
// independent additions are batched into one launch, leaves and fused frames
// are one launch each -- and issues them in order on the stream.  Lowered plans
// are cached per (variant, shape, scalars, pointers); with graphs enabled the
// launch sequence of a cached plan is captured once into a CUDA graph and
// replayed, which removes the per-launch host cost of the serial schedule chain.
// Each cached plan owns a temporary arena of exactly its high-water size.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/winomem_b200.h"
#include "wm_device.h"
#include "wm_frame.h"
#include "wm_io.h"
#include "wm_fused.h"
#include "wm_gemm.h"
#include "wm_launch.h"
#include "wm_micro.h"
#include "wm_planner.h"

namespace wm {
cudaError_t launch_leaf_i8(const MulParams& P, cudaStream_t s);      // wm_i8.cu
bool leaf_i8_supported(const MulParams& P);
cudaError_t leaf_i8_init();
GemmParams gemm_from_mul(const MulParams& P);
cudaError_t launch_leaf_i8_cfg(const MulParams& P, int bn, int split, cudaStream_t s);
bool frame_kernel_available();
}  // namespace wm

using namespace wm;

namespace {

thread_local std::string g_err;
thread_local std::string g_sched_calls;
// allocation trace of the last plan reported on this thread (shared with the plan)
thread_local std::shared_ptr<const std::vector<Meter::AllocEvent>> g_alloc_log;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define WM_CUDA(expr)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            fail(E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));             \
    } while (0)

struct Step {
    enum Kind : std::uint8_t { ADD, MUL, FRAME, GROUP, FPREP, FGEMM, FCOMB, UPLOAD, DOWNLOAD } kind;
    AddBatch add;
    unsigned blocks = 0;
    MulParams mul;
    int leaf = 0;  // MUL: 0 dmma, 1 i8
    int gid = -1;  // GROUP: fused schedule run
    fused::GroupParams grp;
    FramePrepParams fprep;  // fused leaf frame, three launches
    GemmParams fgemm;       // FGEMM, and MUL with leaf == 1 (int8 engine)
    FrameCombParams fcomb;
    int engine = 0;         // int8 GEMM: 0 cp.async, 1 TMA
    int bn = 32, split = 1;
    std::shared_ptr<TmaMaps> tmaps;
    unsigned long long* tl = nullptr;  // GROUP: measurement timeline slot
    // UPLOAD / DOWNLOAD (host u32 boundary): one block of a host matrix, staged
    // as u32 on the device and converted to / from the float64 operand
    std::uint32_t* hptr = nullptr;
    std::uint32_t* sptr = nullptr;
    double* dptr = nullptr;
    std::uint64_t hld = 0, sld = 0, dld = 0, io_rows = 0, io_cols = 0;
    std::uint32_t io_p = 0;
    std::int8_t lane_hint = -1;        // 0: the copy-in lane, 1: the copy-out lane
    // memory the launch reads / writes (dependency analysis for concurrent issue)
    std::vector<View> rd, wr;
};

// Read / write sets of one planned operation (a fused frame also writes the
// blocks hosting its planes).
void op_sets(const Op& o, std::vector<View>& rd, std::vector<View>& wr) {
    wr.push_back(o.d);
    rd.push_back(o.a);
    if (o.kind == OP_ADDSUB || o.kind == OP_MUL || o.kind == OP_FRAME) rd.push_back(o.b);
    if (o.kind == OP_MUL || o.kind == OP_FRAME) rd.push_back(o.d);
    if (o.kind == OP_FRAME)
        for (const View* h : {&o.h0, &o.h1, &o.h2})
            if (h->rows) wr.push_back(*h);
}

// Read / write sets of the three launches of a fused frame (lower_frame).  Only
// the prep reads the frame's operands: once it is done, the parent schedule's
// next additions (which overwrite the temporaries holding this frame's A / B)
// may run beside the GEMM and the combine.
//   prep:    reads A, B, C (C_in);  writes the plane hosts in C, and (accumulating
//            frames) raw planes in the third temporary / the spare h1 slot
//   GEMM:    reads the planes in C (accumulating: also h1 / h2 and the float64
//            B22 fallback in B);  writes the product planes in h0, h1
//   combine: reads h0, h1 and the packed beta*C_in in C;  writes C
void frame_sets(const Op& o, const Field& f, std::vector<Step>& steps, std::size_t first,
                const View* ext = nullptr) {
    const bool acc = !f.is_zero(o.sb);
    auto add = [](std::vector<View>& s, const View& v) {
        if (v.rows) s.push_back(v);
    };
    for (std::size_t j = first; j < steps.size(); ++j) {
        Step& s = steps[j];
        if (ext) {  // planes outside C: the prep never touches C
            if (s.kind == Step::FPREP) {
                add(s.rd, o.a), add(s.rd, o.b);
                for (int e = 0; e < 4; ++e) add(s.wr, ext[e]);
            } else if (s.kind == Step::FGEMM) {
                for (int e = 0; e < 4; ++e) add(s.rd, ext[e]);
                add(s.wr, o.h0), add(s.wr, o.h1);
            } else if (s.kind == Step::FCOMB) {
                add(s.rd, o.h0), add(s.rd, o.h1), add(s.rd, o.d), add(s.wr, o.d);
            }
            continue;
        }
        switch (s.kind) {
            case Step::FPREP:
                add(s.rd, o.a), add(s.rd, o.b), add(s.rd, o.d), add(s.wr, o.d);
                if (acc) add(s.wr, o.h1), add(s.wr, o.h2);
                break;
            case Step::FGEMM:
                add(s.rd, o.d), add(s.wr, o.h0), add(s.wr, o.h1);
                if (acc) add(s.rd, o.h2);
                if (acc && !o.h2.rows) add(s.rd, o.b);  // float64 B22 (no plane slot left)
                break;
            case Step::FCOMB:
                add(s.rd, o.h0), add(s.rd, o.h1), add(s.rd, o.d), add(s.wr, o.d);
                break;
            default: op_sets(o, s.rd, s.wr);
        }
    }
}

bool sets_conflict(const Step& a, const Step& b) {
    auto hit = [](const std::vector<View>& x, const std::vector<View>& y) {
        for (const View& u : x)
            for (const View& v : y)
                if (u.phys_overlaps(v)) return true;
        return false;
    };
    return hit(a.wr, b.rd) || hit(a.wr, b.wr) || hit(a.rd, b.wr);
}

struct DagPlan;
struct CachedPlan {
    Plan plan;
    std::vector<Step> steps;
    std::shared_ptr<DagPlan> dag;  // concurrent issue plan (lanes option)
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    unsigned long long* tl = nullptr;  // measurement timeline (trace option)
    MicroOp* micro = nullptr;          // tiny plans: the whole op list for one launch (wm_micro.cu)
    std::uint32_t micro_n = 0;
    MicroImage micro_img{};            // its shared-memory working set
    bool micro_small = false;          // every operation small: one warp walks it
    bool early_marked = false;         // mark_early_loads has run
    ~CachedPlan() {
        if (tl) cudaFree(tl);
        if (micro) cudaFree(micro);
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
    }
};

}  // namespace

constexpr int kLanes = 8;  // maximum; the "dag" option picks how many are used

struct Lanes {
    cudaStream_t s[kLanes] = {};
    std::vector<cudaEvent_t> ev;
    cudaEvent_t join[kLanes] = {};
    ~Lanes() {
        for (int l = 1; l < kLanes; ++l)
            if (s[l]) cudaStreamDestroy(s[l]);
        for (auto e : ev) cudaEventDestroy(e);
        for (auto e : join)
            if (e) cudaEventDestroy(e);
    }
};

struct wm_ctx {
    int device = 0;
    Field f;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // options
    bool fuse_frames = true;
    bool graphs = true;
    bool batch_adds = true;
    int leaf_kernel = 2;  // 0 dmma, 1 i8, 2 auto (i8 where the tiles fit, else dmma)
    int subset = 0;       // measurement: 0 all, 1 adds, 2 leaves, 3 frames, 4/5/6 frame prep/gemm/comb
    int gemm_engine = 0;  // int8 GEMM operand path: 0 cp.async ring, 1 TMA tensor maps
    bool fuse_adds = true;  // fused schedule runs (gen_fusion.py)
    bool direct_ok = false;  // direct-limb frame GEMM available (wm_direct.cu)
    bool direct_frames = true;  // use it for fused frames (limb-pair operand planes)
    int dag = 3;                // concurrent issue over this many streams (0/1: one stream;
                                // measured: 3 >= 2, 4 > 8 lanes)
    bool fold = true;           // fold a frame's operand-producing additions into its prep
    bool stream_io = true;      // host u32 boundary as quadrant copy steps inside the graph
    bool micro = true;          // plans of tiny operations as one micro launch (wm_micro.cu)
    bool dead_hosts = true;     // frame product planes in dead blocks (choose_product_hosts)
    int epoch = 512;            // launches per dependency epoch (all lanes join between epochs)
    bool wide_plain = true;     // plain frames' GEMM at BN = 64 (half the CTAs of BN = 32)
    bool cin_direct = true;     // accumulating frames: all planes in dead blocks, C_in read by the combine
    int early_loads = 3;        // (bit 0 prep, bit 1 combine) prep / combine read what their lane predecessor does not write
                                // before griddepcontrol.wait
    bool trace = false;         // measurement: per-launch start / end timeline (wm_diag_trace)
    const void* traced = nullptr;  // CachedPlan of the last traced run
    Lanes lanes;
    // plan cache (small LRU)
    std::list<std::pair<std::string, std::unique_ptr<CachedPlan>>> cache;
    // one arena of schedule temporaries for every plan of this context (plans
    // run one after the other on its stream), sized to the largest high-water
    // mark: the process holds exactly the schedule's peak extra memory
    double* arena = nullptr;
    std::uint64_t arena_words = 0;
    // boundary staging
    std::uint32_t* stage = nullptr;
    std::size_t stage_words = 0;
    double* hbuf[3] = {nullptr, nullptr, nullptr};
    std::size_t hbuf_words[3] = {0, 0, 0};

    ~wm_ctx() {
        cache.clear();
        if (arena) cudaFree(arena);
        if (stage) cudaFree(stage);
        for (auto* b : hbuf)
            if (b) cudaFree(b);
        if (own_stream && stream) cudaStreamDestroy(stream);
    }
};

namespace {

std::uint32_t modp_add_mode(const Field& f, Scalar sa, Scalar sb) {
    const bool a1 = f.is_one(sa), am = f.is_minus_one(sa), b1 = f.is_one(sb),
               bm = f.is_minus_one(sb);
    if (a1 && b1) return M_ADD;
    if (a1 && bm) return M_SUB;
    if (am && b1) return M_RSUB;
    if (am && bm) return M_NEGADD;
    return M_GEN;
}

bool aligned16(const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15u) == 0; }

AddItem make_item(const Op& op, const Field& f, double* const base[4]) {
    AddItem t{};
    t.d = base[op.d.region] + op.d.off;
    t.a = base[op.a.region] + op.a.off;
    t.ldd = op.d.ld;
    t.lda = op.a.ld;
    t.rows = static_cast<std::uint32_t>(op.d.rows);
    t.cols = static_cast<std::uint32_t>(op.d.cols);
    t.sa = op.sa.r;
    t.sb = op.sb.r;
    t.sad = op.sa.d;
    t.sbd = op.sb.d;
    bool vec = (t.cols % 2 == 0) && (t.ldd % 2 == 0) && (t.lda % 2 == 0) && aligned16(t.d) &&
               aligned16(t.a);
    if (op.kind == OP_ADDSUB) {
        t.b = base[op.b.region] + op.b.off;
        t.ldb = op.b.ld;
        t.mode = modp_add_mode(f, op.sa, op.sb);
        vec = vec && (t.ldb % 2 == 0) && aligned16(t.b);
    } else {
        t.b = t.a;
        t.ldb = t.lda;
        t.mode = f.is_one(op.sa) ? M_COPY : f.is_minus_one(op.sa) ? M_NEG : M_SCALE;
    }
    t.vec = vec ? 2 : 1;
    t.ca = f.real ? op.sa.d : static_cast<double>(op.sa.r);
    t.cb = op.kind != OP_ADDSUB ? 0.0 : f.real ? op.sb.d : static_cast<double>(op.sb.r);
    return t;
}

unsigned item_blocks(const AddItem& t) {
    const std::uint64_t units = static_cast<std::uint64_t>(t.rows) * t.cols / t.vec;
    const std::uint64_t per = static_cast<std::uint64_t>(kAddThreads) * kAddIlp;
    return static_cast<unsigned>((units + per - 1) / per);
}

MulParams make_mul(const Op& op, const Field& f, double* const base[4]) {
    MulParams P{};
    P.C = base[op.d.region] + op.d.off;
    P.A = base[op.a.region] + op.a.off;
    P.B = base[op.b.region] + op.b.off;
    P.ldc = op.d.ld;
    P.lda = op.a.ld;
    P.ldb = op.b.ld;
    P.m = static_cast<std::uint32_t>(op.a.rows);
    P.k = static_cast<std::uint32_t>(op.a.cols);
    P.n = static_cast<std::uint32_t>(op.b.cols);
    P.alpha = op.sa.r;
    P.beta = op.sb.r;
    P.alphad = op.sa.d;
    P.betad = op.sb.d;
    P.p = f.p;
    P.pd = static_cast<double>(f.p);
    P.pinv = 1.0 / static_cast<double>(f.p);
    return P;
}

void init_batch(AddBatch& b, const Field& f) {
    std::memset(&b, 0, sizeof(b));
    b.p = f.p;
    b.pd = static_cast<double>(f.p);
    b.pinv = 1.0 / static_cast<double>(f.p);
}

// The fused group (gen_fusion.py) for the run starting at plan op i: the
// longest one whose instructions are all still to be launched (a run whose
// operand-producing additions were folded into the next frame's prep uses the
// group generated for its remainder).
int find_group(const Plan& plan, std::size_t i, const std::vector<char>& folded) {
    const Op& op = plan.ops[i];
    if (op.frame < 0 || !op.sched) return -1;
    int best = -1;
    for (int g = 0; g < fused::kNumGroups; ++g) {
        const fused::GroupDesc& G = fused::kGroups[g];
        if (G.row0 != op.row || std::strcmp(G.sched, op.sched) != 0) continue;
        if (i + G.nins > plan.ops.size()) continue;
        bool clear = true;
        for (int j = 0; j < G.nins; ++j) clear = clear && !(i + j < folded.size() && folded[i + j]);
        if (clear && (best < 0 || G.nins > fused::kGroups[best].nins)) best = g;
    }
    return best;
}

// Bind the run of operations starting at ops[i] to fused group g: the rows must
// be the group's rows of one frame instance, every slot must map to one view,
// all views must share one shape, be pairwise disjoint and 16-B vectorisable.
bool try_group(const Plan& plan, std::size_t i, int g, double* const base[4], Step& st) {
    const fused::GroupDesc& G = fused::kGroups[g];
    if (i + G.nins > plan.ops.size()) return false;
    View slot[fused::kMaxSlots];
    bool bound[fused::kMaxSlots] = {};
    const Op& first = plan.ops[i];
    auto bind = [&](int s, const View& v) {
        if (!bound[s]) {
            slot[s] = v;
            bound[s] = true;
            return true;
        }
        return slot[s].same_window(v);
    };
    for (int j = 0; j < G.nins; ++j) {
        const Op& op = plan.ops[i + j];
        if (op.kind != OP_ADDSUB && op.kind != OP_COPY) return false;
        if (op.frame != first.frame || op.row != G.row0 + j) return false;
        const int ds = G.ins[j][0], as = G.ins[j][1], bs = G.ins[j][2];
        if ((bs < 0) != (op.kind == OP_COPY)) return false;
        if (op.d.rows != first.d.rows || op.d.cols != first.d.cols) return false;
        if (!bind(ds, op.d) || !bind(as, op.a) || (bs >= 0 && !bind(bs, op.b))) return false;
    }
    if (first.d.cols % 2) return false;
    for (int a = 0; a < G.nslots; ++a) {
        if (!bound[a]) return false;
        for (int b = a + 1; b < G.nslots; ++b)
            if (slot[a].phys_overlaps(slot[b])) return false;
    }
    const Field& f = plan.field;
    std::memset(&st.grp, 0, sizeof(st.grp));
    for (int a = 0; a < G.nslots; ++a) {
        double* ptr = base[slot[a].region] + slot[a].off;
        if (slot[a].ld % 2 || !aligned16(ptr)) return false;
        st.grp.v[a] = ptr;
        st.grp.ld[a] = slot[a].ld;
    }
    for (int j = 0; j < G.nins; ++j) {
        const Op& op = plan.ops[i + j];
        // s_dst = ca * s_a + cb * s_b: unit scalars as +-1 (lazy), others as residues
        // whose result is reduced at once
        auto coef = [&](Scalar v, bool* general) {
            if (f.real) return v.d;
            if (f.is_zero(v)) return 0.0;
            if (f.is_one(v)) return 1.0;
            if (f.is_minus_one(v)) return -1.0;
            *general = true;
            return static_cast<double>(v.r);
        };
        bool general = false;
        st.grp.ca[j] = coef(op.sa, &general);
        st.grp.cb[j] = op.kind == OP_ADDSUB ? coef(op.sb, &general) : 0.0;
        if (general) st.grp.gen |= 1u << j;
    }
    st.grp.rows = static_cast<std::uint32_t>(first.d.rows);
    st.grp.cols = static_cast<std::uint32_t>(first.d.cols);
    st.grp.p = static_cast<double>(f.p);
    st.grp.pinv = 1.0 / static_cast<double>(f.p);
    st.kind = Step::GROUP;
    st.gid = g;
    return true;
}

// Choose tiling and (TMA engine) encode the operand tensor maps for an int8 GEMM step.
void finish_gemm_step(Step& st, int engine, int force = 0) {
    gemm_choose(st.fgemm, &st.bn, &st.split);
    if (force) {
        st.bn = force / 100;
        st.split = force % 100;
    }
    st.engine = 0;
    if (engine == 1) {
        auto maps = std::make_shared<TmaMaps>();
        if (gemm_tma_encode(st.fgemm, st.bn, *maps)) {
            st.tmaps = maps;
            st.engine = 1;
        }
    }
}

// A fused leaf frame -> prep / seven-product GEMM / combine launches.
void lower_frame(const Op& op, const Field& f, double* const base[4], std::vector<Step>& steps,
                 int engine, bool direct, bool wide_plain, const View* ext = nullptr) {
    const int force = 0;
    const std::uint64_t c = op.a.rows / 2;
    auto ptr = [&](const View& v) { return base[v.region] + v.off; };
    const auto aq = quad_split(op.a), bq = quad_split(op.b), cq = quad_split(op.d);
    const bool acc = !f.is_zero(op.sb);
    // ext (accumulating frames with dead blocks to spare): S / T planes in ext[0]
    // / ext[1], raw planes in ext[2], ext[3]; C keeps C_in untouched for the combine
    const View& sh = ext ? ext[0] : acc ? cq[1] : cq[0];  // S planes host
    const View& th = ext ? ext[1] : acc ? cq[2] : cq[1];  // T planes host
    // direct-limb engine: operand planes are limb pairs (hi / lo byte rows) that
    // the GEMM loads straight into tensor-core layout; prep CTAs own whole rows
    direct = direct && c <= 2048;
    // a host row holds four plane rows of 2c bytes; plane q starts at byte 2qc
    auto plane16 = [&](const View& host, int q) {
        GemmSrc g;
        g.p = reinterpret_cast<std::uint16_t*>(ptr(host)) + q * c;
        g.ld = 4 * host.ld;
        g.fmt = 1;
        g.part = 0;
        return g;
    };
    auto plane = [&](const View& host, int q) {
        if (!direct) return plane16(host, q);
        GemmSrc g;
        g.p = reinterpret_cast<std::uint8_t*>(ptr(host)) + 2 * q * c;
        g.ld = 8 * host.ld;
        g.fmt = 2;
        g.part = c;
        return g;
    };
    auto f64 = [&](const View& v) {
        GemmSrc g;
        g.p = ptr(v);
        g.ld = v.ld;
        g.fmt = 0;
        g.part = 0;
        return g;
    };
    const double pd = static_cast<double>(f.p), pinv = 1.0 / static_cast<double>(f.p);
    Step p{};
    p.kind = Step::FPREP;
    for (int i = 0; i < 4; ++i) {
        p.fprep.A.q[i] = ptr(aq[i]);
        p.fprep.B.q[i] = ptr(bq[i]);
        p.fprep.C.q[i] = ptr(cq[i]);
    }
    p.fprep.A.ld = op.a.ld;
    p.fprep.B.ld = op.b.ld;
    p.fprep.C.ld = op.d.ld;
    p.fprep.limbs = direct ? 1 : 0;
    // raw blocks materialised as planes where a free host slot exists:
    // plain frames own C21, C22 until the combine; accumulating frames own C22
    // (its beta*C_in is packed away first), a third temporary and the spare
    // slot of the second product host.  Only B22 of a two-temporary
    // accumulating frame is left in float64 (a B operand: the direct engine
    // splits it in the GEMM).
    std::vector<std::pair<View, int>> raw_slots;
    if (ext) {
        for (int q = 0; q < 4; ++q) raw_slots.push_back({ext[2], q});
        for (int q = 0; q < 2; ++q) raw_slots.push_back({ext[3], q});
    } else if (!acc) {
        for (int q = 0; q < 4; ++q) raw_slots.push_back({cq[2], q});
        for (int q = 0; q < 4; ++q) raw_slots.push_back({cq[3], q});
    } else {
        for (int q = 0; q < 4; ++q) raw_slots.push_back({cq[3], q});
        if (op.h2.rows) for (int q = 0; q < 4; ++q) raw_slots.push_back({op.h2, q});
        raw_slots.push_back({op.h1, 3});
    }
    const View raw_view[6] = {aq[0], aq[1], aq[3], bq[0], bq[2], bq[3]};
    GemmSrc raw[6];
    for (int i = 0; i < 6; ++i) {
        if (i < static_cast<int>(raw_slots.size())) {
            raw[i] = plane(raw_slots[i].first, raw_slots[i].second);
            p.fprep.plane[PL_A11 + i] = const_cast<void*>(raw[i].p);
            p.fprep.pld[PL_A11 + i] = raw[i].ld;
        } else {
            raw[i] = f64(raw_view[i]);
            p.fprep.plane[PL_A11 + i] = nullptr;
        }
    }
    GemmSrc st[8];
    for (int q = 0; q < 4; ++q) {
        st[q] = plane(sh, q);
        st[4 + q] = plane(th, q);
    }
    for (int i = 0; i < 8; ++i) {
        p.fprep.plane[PL_S1 + i] = const_cast<void*>(st[i].p);
        p.fprep.pld[PL_S1 + i] = st[i].ld;
    }
    p.fprep.c = static_cast<std::uint32_t>(c);
    p.fprep.beta = ext ? 0 : op.sb.r;  // ext: nothing to pack, C is not touched
    p.fprep.pd = pd;
    p.fprep.pinv = pinv;
    steps.push_back(p);

    Step g{};
    g.kind = Step::FGEMM;
    GemmParams& G = g.fgemm;
    // P1 = A11 B11, P2 = A12 B21, P3 = S4 B22, P4 = A22 T4, P5 = S1 T1, P6 = S2 T2, P7 = S3 T3
    // raw[] = {A11, A12, A22, B11, B21, B22} (planes or float64 blocks)
    G.a[0] = raw[0]; G.b[0] = raw[3];
    G.a[1] = raw[1]; G.b[1] = raw[4];
    G.a[2] = st[3];  G.b[2] = raw[5];
    G.a[3] = raw[2]; G.b[3] = st[7];
    G.a[4] = st[0];  G.b[4] = st[4];
    G.a[5] = st[1];  G.b[5] = st[5];
    G.a[6] = st[2];  G.b[6] = st[6];
    for (int k = 0; k < 7; ++k) G.c[k] = k < 4 ? plane16(op.h0, k) : plane16(op.h1, k - 4);
    G.m = G.n = G.k = static_cast<std::uint32_t>(c);
    G.nprod = 7;
    G.tiles_m = static_cast<std::uint32_t>(c / 128);
    G.alpha = 1;
    G.beta = 0;
    G.pd = pd;
    G.pinv = pinv;
    if (direct) {
        g.bn = (force >= 1000 && force < 3000) ? force % 1000 + 1000 * (force / 1000 - 1)
                                                : gemm_direct_choose(G);
        // plain frames overlap their siblings (product planes in dead blocks):
        // half the CTAs at twice the width leave SMs to the sibling launches
        // (measured: config 2 4.35 -> 4.23 ms, config 3 15.24 -> 14.35 ms; at
        // c = 128 the grid is already small and it loses)
        // accumulating frames with every plane outside C (ext) overlap the same
        // way (their prep no longer waits on C_in): C2 3.96 -> 3.85 ms
        if (force == 0 && wide_plain && (!acc || ext) && g.bn == 32 && G.n % 64 == 0 && G.m >= 256)
            g.bn = 64;
        auto maps = std::make_shared<TmaMaps>();
        if (!gemm_direct_supported(G, g.bn) || !gemm_direct_encode(G, g.bn, *maps))
            fail(E_INVALID, "direct-limb frame GEMM: unsupported operands");
        g.tmaps = maps;
        g.engine = 2;
        g.split = 1;
    } else {
        finish_gemm_step(g, engine, force);
    }
    steps.push_back(g);

    Step cb{};
    cb.kind = Step::FCOMB;
    for (int k = 0; k < 7; ++k) {
        cb.fcomb.P[k] = static_cast<const std::uint16_t*>(G.c[k].p);
        cb.fcomb.pld[k] = G.c[k].ld;
    }
    for (int i = 0; i < 4; ++i) cb.fcomb.C.q[i] = ptr(cq[i]);
    cb.fcomb.C.ld = op.d.ld;
    cb.fcomb.c = static_cast<std::uint32_t>(c);
    cb.fcomb.alpha = op.sa.r;
    cb.fcomb.beta = op.sb.r;
    cb.fcomb.cin_f64 = ext ? 1 : 0;
    cb.fcomb.pd = pd;
    cb.fcomb.pinv = pinv;
    steps.push_back(cb);
}

// ---- folding a frame's operand additions into its prep ----------------------
//
// In the parent schedule a fused frame is usually preceded by the run of
// additions that forms its operands (std2 rows 1-2: S3 -> X, T3 -> Y, then
// P7 = X Y).  The prep can compute those operands from the run's sources
// itself, saving the run's launch and its round trip through HBM; it stores the
// operand back only when a later operation still reads it.

struct Fold {
    int op[2] = {-1, -1};  // plan op producing the frame's A / B
    bool writeback[2] = {true, true};
};

bool is_add(const Op& o) { return o.kind == OP_ADDSUB || o.kind == OP_COPY; }

void plan_op_sets(const Op& o, std::vector<View>& rd, std::vector<View>& wr) { op_sets(o, rd, wr); }

bool any_overlap(const std::vector<View>& xs, const View& v) {
    for (const View& x : xs)
        if (x.rows && x.phys_overlaps(v)) return true;
    return false;
}

// Is v read again after ops[i] before it is fully overwritten?
bool live_after(const Plan& plan, std::size_t i, const View& v) {
    for (std::size_t k = i + 1; k < plan.ops.size(); ++k) {
        const Op& o = plan.ops[k];
        std::vector<View> rd, wr;
        op_sets(o, rd, wr);
        if (any_overlap(rd, v)) return true;
        if (any_overlap(wr, v)) return !(is_add(o) && o.d.same_window(v));
    }
    return v.region != R_T;  // caller-visible memory keeps its value
}

// Does a fused-addition group exist for exactly the plan ops [i, i + n)?
bool group_exists(const Plan& plan, std::size_t i, std::size_t n) {
    const Op& o = plan.ops[i];
    if (!o.sched) return false;
    for (int g = 0; g < fused::kNumGroups; ++g)
        if (fused::kGroups[g].row0 == o.row && fused::kGroups[g].nins == static_cast<int>(n) &&
            std::strcmp(fused::kGroups[g].sched, o.sched) == 0)
            return true;
    return false;
}

std::vector<Fold> plan_folds(const Plan& plan) {
    std::vector<Fold> folds(plan.ops.size());
    auto srcs = [](const Op& o) {
        std::vector<View> v = {o.a};
        if (o.kind == OP_ADDSUB) v.push_back(o.b);
        return v;
    };
    for (std::size_t i = 0; i < plan.ops.size(); ++i) {
        const Op& F = plan.ops[i];
        if (F.kind != OP_FRAME || F.frame < 0 || F.a.phys_overlaps(F.b)) continue;
        // the complete run of the parent's additions just before the frame
        std::size_t j0 = i;
        while (j0 > 0 && is_add(plan.ops[j0 - 1]) && plan.ops[j0 - 1].frame == F.frame) --j0;
        if (j0 == i) continue;
        const bool acc = F.sb.r != 0;
        // what the prep itself writes (the GEMM's product planes in h0 / h1 come later)
        std::vector<View> prep_writes = {F.d};
        if (acc) prep_writes.push_back(F.h1), prep_writes.push_back(F.h2);
        // candidates: the last writer of each operand, if it writes exactly that
        // operand and may move past the run's later instructions (none reads or
        // writes its destination or writes its sources)
        Fold fd;
        for (int w = 0; w < 2; ++w) {
            const View& X = w ? F.b : F.a;
            std::size_t last = i;
            for (std::size_t j = j0; j < i; ++j)
                if (plan.ops[j].d.phys_overlaps(X)) last = j;
            if (last == i || !plan.ops[last].d.same_window(X)) continue;
            const Op& o = plan.ops[last];
            bool ok = true;
            for (const View& v : srcs(o)) {
                // per-position ownership: a source is the operand itself or disjoint from it
                if (!v.same_window(o.d) && v.phys_overlaps(o.d)) ok = false;
                if (any_overlap(prep_writes, v)) ok = false;
            }
            for (std::size_t j = last + 1; j < i && ok; ++j) {
                const Op& r = plan.ops[j];
                if (r.d.phys_overlaps(o.d) || any_overlap(srcs(r), o.d) || any_overlap(srcs(o), r.d))
                    ok = false;
            }
            if (ok) fd.op[w] = static_cast<int>(last);
        }
        // both folded: computed side by side from the state before either
        if (fd.op[0] >= 0 && fd.op[1] >= 0) {
            const Op& x = plan.ops[fd.op[0]];
            const Op& y = plan.ops[fd.op[1]];
            if (any_overlap(srcs(x), y.d) || any_overlap(srcs(y), x.d)) fd.op[1] = -1;
        }
        // an accumulating prep writes raw planes into h1 / h2: keep them off the operands
        if (acc && (any_overlap({F.h1, F.h2}, F.a) || any_overlap({F.h1, F.h2}, F.b))) continue;
        // the rest of the run must stay one launch: a contiguous fused group or a
        // single addition (else folding would split a fused run into a chain)
        auto rest_ok = [&](const Fold& f) {
            std::vector<std::size_t> rest;
            for (std::size_t j = j0; j < i; ++j)
                if (static_cast<int>(j) != f.op[0] && static_cast<int>(j) != f.op[1]) rest.push_back(j);
            if (rest.size() <= 1) return true;
            if (rest.back() - rest.front() + 1 != rest.size()) return false;
            return group_exists(plan, rest.front(), rest.size());
        };
        if (!rest_ok(fd)) {
            Fold a = fd, b = fd;
            a.op[1] = -1;
            b.op[0] = -1;
            fd = (a.op[0] >= 0 && rest_ok(a)) ? a : (b.op[1] >= 0 && rest_ok(b)) ? b : Fold();
        }
        if (fd.op[0] < 0 && fd.op[1] < 0) continue;
        for (int w = 0; w < 2; ++w)
            if (fd.op[w] >= 0) fd.writeback[w] = live_after(plan, i, w ? F.b : F.a);
        // an accumulating frame with two temporaries has no plane slot left for
        // B22: its GEMM reads that block of B as float64 (lower_frame)
        if (acc && !F.h2.rows) fd.writeback[1] = true;
        folds[i] = fd;
    }
    return folds;
}

void apply_fold(const Plan& plan, const Fold& fd, double* const base[4], Step& prep) {
    const Field& f = plan.field;
    for (int w = 0; w < 2; ++w) {
        FrameFold& ff = prep.fprep.fold[w];
        std::memset(&ff, 0, sizeof(ff));
        if (fd.op[w] < 0) continue;
        const Op& o = plan.ops[fd.op[w]];
        const auto q0 = quad_split(o.a);
        for (int k = 0; k < 4; ++k) ff.s0[k] = base[q0[k].region] + q0[k].off;
        ff.ld0 = o.a.ld;
        if (o.kind == OP_ADDSUB) {
            const auto q1 = quad_split(o.b);
            for (int k = 0; k < 4; ++k) ff.s1[k] = base[q1[k].region] + q1[k].off;
            ff.ld1 = o.b.ld;
            ff.sb = static_cast<double>(o.sb.r);
        }
        ff.sa = static_cast<double>(o.sa.r);
        ff.on = 1;
        ff.writeback = fd.writeback[w] ? 1 : 0;
        // dependency sets: the prep reads the sources instead of the operand view,
        // and writes the operand view only when it stores it back
        const View& X = o.d;
        for (auto it = prep.rd.begin(); it != prep.rd.end();)
            it = it->same_window(X) ? prep.rd.erase(it) : it + 1;
        prep.rd.push_back(o.a);
        if (o.kind == OP_ADDSUB) prep.rd.push_back(o.b);
        if (ff.writeback) prep.wr.push_back(X);
    }
    (void)f;
}

// ---- product planes in dead blocks -------------------------------------------
//
// A fused frame writes its seven product planes into two c x c blocks and its
// combine reads them back.  By default those are the frame's two temporaries,
// which every sibling frame of the same parent reuses: the next sibling's GEMM
// then waits for this frame's combine.  Any other pair of c x c blocks whose
// content is dead at the frame (the next access in plan order overwrites them
// whole) serves as well; the latest-overwritten such pair breaks that chain.

// `outer` contains `in` (same region and leading dimension)
bool view_contains(const View& outer, const View& in) {
    if (outer.region != in.region || outer.ld != in.ld || in.off < outer.off || outer.empty()) return false;
    const std::uint64_t d = in.off - outer.off, r0 = d / outer.ld, c0 = d % outer.ld;
    return r0 + in.rows <= outer.rows && c0 + in.cols <= outer.cols;
}

// Index of the next plan op after `i` that accesses `w` if that access
// overwrites all of `w` without reading it; -1 if `w` is live after op i.
// How plan op `o` accesses `w`: 0 not at all, 1 reads it (or writes part of
// it), 2 overwrites all of it without reading it.
int access_kind(const Plan& plan, const Op& o, const View& w) {
    const bool acc_like = (o.kind == OP_MUL || o.kind == OP_FRAME) && !plan.field.is_zero(o.sb);
    if (o.a.phys_overlaps(w)) return 1;
    if ((o.kind == OP_ADDSUB || o.kind == OP_MUL || o.kind == OP_FRAME) && o.b.phys_overlaps(w)) return 1;
    if (o.kind == OP_FRAME)
        for (const View* h : {&o.h0, &o.h1, &o.h2})
            if (h->rows && h->phys_overlaps(w)) return 1;
    if (o.d.phys_overlaps(w)) return !acc_like && view_contains(o.d, w) ? 2 : 1;
    return 0;
}

// Every access to each candidate block, computed once per block (physical
// identity) and shared by all frames of a plan.
struct AccessIndex {
    std::map<std::tuple<int, std::uint64_t, std::uint64_t, std::uint64_t, std::uint64_t>,
             std::vector<std::pair<std::size_t, int>>>
        acc;
    const std::vector<std::pair<std::size_t, int>>& of(const Plan& plan, const View& w) {
        const auto key = std::make_tuple(static_cast<int>(w.region), w.off, w.ld, w.rows, w.cols);
        auto it = acc.find(key);
        if (it != acc.end()) return it->second;
        std::vector<std::pair<std::size_t, int>> v;
        for (std::size_t k = 0; k < plan.ops.size(); ++k) {
            const int a = access_kind(plan, plan.ops[k], w);
            if (a) v.push_back({k, a});
        }
        return acc.emplace(key, std::move(v)).first->second;
    }
};

long next_cover(const Plan& plan, std::size_t i, const View& w, AccessIndex& ix) {
    const auto& v = ix.of(plan, w);
    auto it = std::upper_bound(v.begin(), v.end(), std::make_pair(i, 3));
    if (it == v.end()) return -1;  // reaches the end: caller memory stays live
    return it->second == 2 ? static_cast<long>(it->first) : -1;
}

// Up to `want` windows, best first; `recent` are blocks the previous frames'
// launches may still be reading (their product / raw plane hosts).
std::vector<View> choose_product_hosts(const Plan& plan, std::size_t i, const Fold* fd,
                                       const std::vector<std::size_t>& parent_ops,
                                       const std::vector<View>& recent, std::size_t want,
                                       AccessIndex& ix) {
    const Op& F = plan.ops[i];
    const std::uint64_t c = F.a.rows / 2;
    std::vector<View> excl = {F.a, F.b, F.d, F.h0, F.h1, F.h2};
    excl.insert(excl.end(), recent.begin(), recent.end());
    if (fd)
        for (int w = 0; w < 2; ++w)
            if (fd->op[w] >= 0) {
                const Op& o = plan.ops[fd->op[w]];
                excl.push_back(o.a), excl.push_back(o.b), excl.push_back(o.d);
            }
    // the next fused frame must not depend on this combine through the hosts
    std::size_t next_frame = plan.ops.size();
    for (std::size_t k = i + 1; k < plan.ops.size(); ++k)
        if (plan.ops[k].kind == OP_FRAME) {
            next_frame = k;
            break;
        }
    std::vector<std::pair<long, View>> cand;
    auto consider = [&](const View& v) {
        if (v.empty() || v.rows % c || v.cols % c || v.ld % 2) return;
        for (std::uint64_t r = 0; r < v.rows; r += c)
            for (std::uint64_t q = 0; q < v.cols; q += c) {
                const View w = v.window(r, q, c, c);
                bool clash = false;
                for (const View& x : excl) clash = clash || (x.rows && x.phys_overlaps(w));
                for (const auto& e : cand) clash = clash || e.second.phys_overlaps(w);
                if (clash) continue;
                const long nc = next_cover(plan, i, w, ix);
                if (nc > static_cast<long>(next_frame)) cand.push_back({nc, w});
            }
    };
    // blocks of the parent frame's own slots (its quadrants and temporaries)
    if (F.frame < 0) return {};
    for (std::size_t k : parent_ops) {
        const Op& o = plan.ops[k];
        consider(o.d);
        consider(o.a);
        if (o.kind != OP_COPY) consider(o.b);
    }
    // and the blocks of the operations around it (the grandparent's slots):
    // measured on the launch DAG, a window of 96 operations finds as much as 256
    {
        const std::size_t win = 96;
        const std::size_t lo = i > win ? i - win : 0, hi = std::min(plan.ops.size(), i + win);
        for (std::size_t k = lo; k < hi; ++k) {
            const Op& o = plan.ops[k];
            if (o.frame == F.frame) continue;
            consider(o.d);
            consider(o.a);
            if (o.kind != OP_COPY) consider(o.b);
        }
    }
    std::stable_sort(cand.begin(), cand.end(),
                     [](const std::pair<long, View>& x, const std::pair<long, View>& y) {
                         return x.first > y.first;
                     });
    std::vector<View> out;
    for (std::size_t t = 0; t < cand.size() && t < want; ++t) out.push_back(cand[t].second);
    return out;
}

// Lower an operation list to launches.  Additions are merged into one launch
// while they are pairwise independent (no write of one touches a read or
// write of another) and contiguous in program order.
std::vector<Step> lower(const Plan& plan, double* const base[4], const wm_ctx& ctx) {
    std::vector<Step> steps;
    const Field& f = plan.field;
    std::vector<const Op*> cur;
    auto flush = [&]() {
        if (cur.empty()) return;
        Step s{};
        s.kind = Step::ADD;
        init_batch(s.add, f);
        unsigned blk = 0;
        for (const Op* op : cur) {
            AddItem t = make_item(*op, f, base);
            t.blk0 = blk;
            blk += item_blocks(t);
            s.add.it[s.add.n++] = t;
            op_sets(*op, s.rd, s.wr);
        }
        s.blocks = blk;
        if (std::getenv("WM_LOWER_DUMP")) {
            std::fprintf(stderr, "ADD %d:", s.add.n);
            for (const Op* op : cur)
                std::fprintf(stderr, " %s/%d(%llux%llu)", op->sched ? op->sched : "-", op->row,
                             static_cast<unsigned long long>(op->d.rows),
                             static_cast<unsigned long long>(op->d.cols));
            std::fprintf(stderr, "\n");
        }
        steps.push_back(s);
        cur.clear();
    };
    auto conflicts = [&](const Op& o) {
        for (const Op* c : cur) {
            if (o.d.phys_overlaps(c->d) || o.d.phys_overlaps(c->a)) return true;
            if (c->kind == OP_ADDSUB && o.d.phys_overlaps(c->b)) return true;
            if (o.a.phys_overlaps(c->d)) return true;
            if (o.kind == OP_ADDSUB && o.b.phys_overlaps(c->d)) return true;
        }
        return false;
    };
    if (std::getenv("WM_PLAN_DUMP"))
        for (std::size_t i = 0; i < plan.ops.size(); ++i) {
            const Op& o = plan.ops[i];
            std::fprintf(stderr, "op %zu kind %d %s/%d frame %d d=%d:%llu(%llux%llu)\n", i, o.kind,
                         o.sched ? o.sched : "-", o.row, o.frame, o.d.region,
                         static_cast<unsigned long long>(o.d.off), static_cast<unsigned long long>(o.d.rows),
                         static_cast<unsigned long long>(o.d.cols));
        }
    const bool fold = ctx.fold && !f.real;
    const std::vector<Fold> folds = fold ? plan_folds(plan) : std::vector<Fold>();
    std::vector<char> folded(plan.ops.size(), 0);
    for (const Fold& fd : folds)
        for (int w = 0; w < 2; ++w)
            if (fd.op[w] >= 0) folded[fd.op[w]] = 1;
    std::map<int, std::vector<std::size_t>> by_frame;  // plan ops of each schedule frame
    std::vector<View> recent_hosts;                    // plane hosts of the previous frame
    AccessIndex access_ix;                             // accesses per candidate block
    std::vector<std::vector<View>> host_hist;          // plane hosts of the last frames
    if (ctx.dead_hosts)
        for (std::size_t k = 0; k < plan.ops.size(); ++k)
            if (plan.ops[k].frame >= 0) by_frame[plan.ops[k].frame].push_back(k);
    for (std::size_t oi = 0; oi < plan.ops.size(); ++oi) {
        const Op& op = plan.ops[oi];
        if (folded[oi]) continue;  // computed by the next frame's prep
        if ((op.kind == OP_ADDSUB || op.kind == OP_COPY) && ctx.fuse_adds) {
            const int g = find_group(plan, oi, folded);
            Step gs{};
            if (g >= 0 && try_group(plan, oi, g, base, gs)) {
                flush();
                for (int j = 0; j < fused::kGroups[g].nins; ++j) op_sets(plan.ops[oi + j], gs.rd, gs.wr);
                steps.push_back(gs);
                oi += fused::kGroups[g].nins - 1;
                continue;
            }
        }
        if (op.kind == OP_ADDSUB || op.kind == OP_COPY) {
            if (!ctx.batch_adds || static_cast<int>(cur.size()) >= kMaxAddBatch || conflicts(op))
                flush();
            cur.push_back(&op);
            continue;
        }
        flush();
        if (op.kind == OP_FRAME) {
            const std::size_t first = steps.size();
            Op fop = op;  // product (and raw) planes in dead blocks when there are some
            View ext[4];
            bool use_ext = false;
            if (ctx.dead_hosts && op.frame >= 0) {
                // accumulating frames: a third block takes the raw planes, so that
                // with two temporaries B22 is materialised too and the GEMM no
                // longer reads the frame's B (the parent's next prep rewrites it)
                const bool acc = !f.is_zero(op.sb);
                const std::vector<View> w =
                    choose_product_hosts(plan, oi, fold ? &folds[oi] : nullptr, by_frame[op.frame],
                                         recent_hosts, acc ? 6 : 2, access_ix);
                if (w.size() >= 2) {
                    fop.h0 = w[0];
                    fop.h1 = w[1];
                    if (acc && w.size() >= 6 && ctx.cin_direct) {
                        // every plane outside C: the prep neither reads nor packs C_in
                        for (int e = 0; e < 4; ++e) ext[e] = w[2 + e];
                        use_ext = true;
                    } else if (acc && w.size() >= 3) {
                        fop.h2 = w[2];
                    }
                }
                // the next frames keep off the plane hosts of the last `keep` frames
                const std::size_t keep = 2;  // launch-DAG model: 2 beats 1, 3, 4
                host_hist.push_back({fop.h0, fop.h1});
                if (fop.h2.rows) host_hist.back().push_back(fop.h2);
                if (use_ext) host_hist.back().insert(host_hist.back().end(), ext, ext + 4);
                while (host_hist.size() > keep) host_hist.erase(host_hist.begin());
                recent_hosts.clear();
                for (const auto& hv : host_hist) recent_hosts.insert(recent_hosts.end(), hv.begin(), hv.end());
            }
            lower_frame(fop, f, base, steps, ctx.gemm_engine, ctx.direct_ok && ctx.direct_frames,
                        ctx.wide_plain, use_ext ? ext : nullptr);
            frame_sets(fop, f, steps, first, use_ext ? ext : nullptr);
            if (fold && (folds[oi].op[0] >= 0 || folds[oi].op[1] >= 0))
                for (std::size_t j = first; j < steps.size(); ++j)
                    if (steps[j].kind == Step::FPREP) apply_fold(plan, folds[oi], base, steps[j]);
            continue;
        }
        Step s{};
        s.mul = make_mul(op, f, base);
        {
            s.kind = Step::MUL;
            const bool i8ok = !f.real && leaf_i8_supported(s.mul);
            s.leaf = (ctx.leaf_kernel == 1 || ctx.leaf_kernel == 2) && i8ok ? 1 : 0;
            if (s.leaf == 1) {
                s.fgemm = gemm_from_mul(s.mul);
                finish_gemm_step(s, ctx.gemm_engine);
            }
        }
        op_sets(op, s.rd, s.wr);
        steps.push_back(s);
    }
    flush();
    return steps;
}

// A launch long enough (tens of microseconds) that its successor gains nothing
// from launching early.
bool long_step(const Step& s) {
    switch (s.kind) {
        case Step::ADD: {
            std::uint64_t e = 0;
            for (int i = 0; i < s.add.n; ++i) e += static_cast<std::uint64_t>(s.add.it[i].rows) * s.add.it[i].cols;
            return e > (4ull << 20);
        }
        case Step::GROUP: return static_cast<std::uint64_t>(s.grp.rows) * s.grp.cols > (4ull << 20);
        case Step::MUL:
            return 2.0 * s.mul.m * static_cast<double>(s.mul.k) * s.mul.n > 1e9;
        case Step::FPREP: return s.fprep.c >= 1024;
        case Step::FGEMM: return s.fgemm.m >= 1024;
        case Step::FCOMB: return s.fcomb.c >= 1024;
        default: return false;
    }
}

bool g_pdl_user = true;  // the "pdl" option; per launch g_pdl = option && policy below

// Programmatic dependent launch per launch: not after a long predecessor (no
// latency left to hide), and never for a multi-CTA-per-SM compute kernel: its
// CTAs would be placed while the predecessor still fills the SMs, bunch up on
// the few SMs with room and keep that placement (measured: config 5's 1024^3
// float64 leaves, 2.88 s per multiply with PDL vs 1.68 s without).
bool use_pdl(const Step& s, const Step* prev) {
    if (!g_pdl_user || (prev && long_step(*prev))) return false;
    if (prev && (prev->kind == Step::UPLOAD || prev->kind == Step::DOWNLOAD)) return false;
    if (s.kind == Step::MUL && 2.0 * s.mul.m * static_cast<double>(s.mul.k) * s.mul.n > 1e8)
        return false;
    return true;
}

void issue_one(const Step& s, bool real, cudaStream_t st, const Step* prev = nullptr) {
    g_pdl = use_pdl(s, prev);
    switch (s.kind) {
        case Step::ADD: WM_CUDA(launch_addsub(s.add, real, s.blocks, st)); break;
        case Step::MUL:
            if (s.leaf == 1) {
                if (s.engine == 1) WM_CUDA(launch_gemm_tma(s.fgemm, *s.tmaps, s.bn, s.split, st));
                else WM_CUDA(launch_gemm_i8(s.fgemm, st));
            } else {
                WM_CUDA(launch_leaf_dmma(s.mul, real, st));
            }
            break;
        case Step::FRAME: break;
        case Step::GROUP: WM_CUDA(launch_group(s.gid, s.grp, real, st, s.tl)); break;
        case Step::FPREP: WM_CUDA(launch_frame_prep(s.fprep, st)); break;
        case Step::FGEMM:
            if (s.engine == 2) WM_CUDA(launch_gemm_direct(s.fgemm, *s.tmaps, s.bn, st));
            else if (s.engine == 1) WM_CUDA(launch_gemm_tma(s.fgemm, *s.tmaps, s.bn, s.split, st));
            else WM_CUDA(launch_gemm_i8(s.fgemm, st));
            break;
        case Step::FCOMB: WM_CUDA(launch_frame_comb(s.fcomb, st)); break;
        case Step::UPLOAD:
            WM_CUDA(cudaMemcpy2DAsync(s.sptr, s.sld * 4, s.hptr, s.hld * 4, s.io_cols * 4, s.io_rows,
                                      cudaMemcpyHostToDevice, st));
            g_pdl = false;
            WM_CUDA(launch_u32_to_f64(s.dptr, s.dld, s.sptr, s.sld, s.io_rows, s.io_cols, st, s.tl));
            break;
        case Step::DOWNLOAD:
            g_pdl = false;
            WM_CUDA(launch_f64_to_u32(s.sptr, s.sld, s.dptr, s.dld, s.io_rows, s.io_cols, s.io_p, st,
                                      s.tl));
            WM_CUDA(cudaMemcpy2DAsync(s.hptr, s.hld * 4, s.sptr, s.sld * 4, s.io_cols * 4, s.io_rows,
                                      cudaMemcpyDeviceToHost, st));
            break;
    }
}

void issue(const std::vector<Step>& steps, bool real, cudaStream_t st, int subset = 0) {
    const Step* prev = nullptr;
    for (const Step& s : steps) {
        if (subset == 1 && s.kind != Step::ADD && s.kind != Step::GROUP) continue;
        if (subset == 2 && s.kind != Step::MUL) continue;
        if (subset == 3 && s.kind != Step::FPREP && s.kind != Step::FGEMM && s.kind != Step::FCOMB)
            continue;
        if (subset == 4 && s.kind != Step::FPREP) continue;
        if (subset == 5 && s.kind != Step::FGEMM) continue;
        if (subset == 6 && s.kind != Step::FCOMB) continue;
        issue_one(s, real, st, prev);
        prev = &s;
    }
}

// Concurrent issue.  The memory-lean schedules are mostly a chain, but
// independent launches exist (about 1.2-1.5x of slack on the configurations'
// operation DAGs, wm_diag_plan_dag), and every launch here is latency-bound, so
// running them side by side pays.  Each step goes to one of kLanes streams: a
// lane whose last launch it depends on (stream order then covers that edge and
// adds no false one), else the lane whose last launch is oldest; conflicting
// launches on other lanes are joined through events.  Dependencies are
// exact within an epoch of kEpoch steps; at epoch boundaries every lane joins.
struct DagPlan {
    int nlanes = 1;                       // streams used (compute lanes + copy lanes)
    std::vector<int> lane;                // per step
    std::vector<std::vector<int>> waits;  // per step: steps (other lanes) to wait for
    std::vector<char> record;             // per step: an event is recorded after it
    std::vector<char> epoch_end;          // per step: all lanes join after it
};

constexpr int kEpoch = 512;

DagPlan plan_dag(const std::vector<Step>& steps, int nl, int epoch = kEpoch) {
    nl = nl < 1 ? 1 : nl > kLanes - 2 ? kLanes - 2 : nl;
    const int n = static_cast<int>(steps.size());
    DagPlan d;
    bool io = false;
    for (const Step& s : steps) io |= s.lane_hint >= 0;
    const int total = nl + (io ? 2 : 0);  // copy-in / copy-out lanes after the compute lanes
    d.nlanes = total;
    d.lane.assign(n, 0);
    d.waits.assign(n, {});
    d.record.assign(n, 0);
    d.epoch_end.assign(n, 0);
    int epoch0 = 0;
    int last_on[kLanes];
    int synced[kLanes][kLanes];  // synced[a][b]: latest step of lane b that lane a waited for
    for (int j = 0; j < n; ++j) {
        if (j - epoch0 == epoch) {
            d.epoch_end[j - 1] = 1;
            epoch0 = j;
        }
        if (j == epoch0)
            for (int l = 0; l < kLanes; ++l) {
                last_on[l] = l < total ? -1 : 1 << 30;
                for (int m = 0; m < kLanes; ++m) synced[l][m] = -1;
            }
        // latest conflicting step per lane (earlier ones on a lane are implied)
        int dep[kLanes];
        for (int l = 0; l < kLanes; ++l) dep[l] = -1;
        int open = total;
        for (int i = j - 1; i >= epoch0 && open > 0; --i) {
            const int l = d.lane[i];
            if (dep[l] >= 0) continue;
            if (sets_conflict(steps[i], steps[j])) {
                dep[l] = i;
                --open;
            }
        }
        // a lane whose last launch is itself a dependency adds no false edge;
        // otherwise take the lane whose last launch is oldest (most likely done)
        int best = steps[j].lane_hint >= 0 ? nl + steps[j].lane_hint : -1;
        for (int l = 0; l < nl && steps[j].lane_hint < 0; ++l)
            if (last_on[l] >= 0 && dep[l] == last_on[l] && (best < 0 || last_on[l] > last_on[best]))
                best = l;
        if (best < 0) {
            best = 0;
            for (int l = 1; l < nl; ++l)
                if (last_on[l] < last_on[best]) best = l;
        }
        d.lane[j] = best;
        for (int l = 0; l < kLanes; ++l)
            if (l != best && dep[l] > synced[best][l]) {
                d.waits[j].push_back(dep[l]);
                d.record[dep[l]] = 1;
                synced[best][l] = dep[l];
            }
        last_on[best] = j;
    }
    return d;
}

void issue_dag(const std::vector<Step>& steps, const DagPlan& d, bool real, cudaStream_t main,
               Lanes& L) {
    const int nl = d.nlanes;
    const int n = static_cast<int>(steps.size());
    L.s[0] = main;
    for (int l = 1; l < nl; ++l)
        if (!L.s[l]) WM_CUDA(cudaStreamCreateWithFlags(&L.s[l], cudaStreamNonBlocking));
    for (int l = 0; l < nl; ++l)
        if (!L.join[l]) WM_CUDA(cudaEventCreateWithFlags(&L.join[l], cudaEventDisableTiming));
    while (static_cast<int>(L.ev.size()) < n) {
        cudaEvent_t e;
        WM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        L.ev.push_back(e);
    }
    auto fork = [&]() {  // every lane starts after what is already on the main stream
        WM_CUDA(cudaEventRecord(L.join[0], main));
        for (int l = 1; l < nl; ++l) WM_CUDA(cudaStreamWaitEvent(L.s[l], L.join[0], 0));
    };
    auto join = [&]() {  // the main stream continues after every lane
        for (int l = 1; l < nl; ++l) {
            WM_CUDA(cudaEventRecord(L.join[l], L.s[l]));
            WM_CUDA(cudaStreamWaitEvent(main, L.join[l], 0));
        }
    };
    fork();
    int last[kLanes];
    for (int l = 0; l < kLanes; ++l) last[l] = -1;
    for (int j = 0; j < n; ++j) {
        cudaStream_t st = L.s[d.lane[j]];
        for (int i : d.waits[j]) WM_CUDA(cudaStreamWaitEvent(st, L.ev[i], 0));
        issue_one(steps[j], real, st, last[d.lane[j]] >= 0 ? &steps[last[d.lane[j]]] : nullptr);
        last[d.lane[j]] = j;
        if (d.record[j]) WM_CUDA(cudaEventRecord(L.ev[j], st));
        if (d.epoch_end[j]) {
            join();
            fork();
        }
    }
    join();
}

// Loads before griddepcontrol.wait.  A launch may start while the launches it
// depends on directly are still running: its predecessor on the lane, and the
// launches of other lanes it joins through events (under capture a kernel
// launched with programmatic serialization gets programmatic edges from ALL of
// them -- measured: reading a cross-lane producer's block before the wait gives
// wrong results).  Everything those launches themselves waited for has completed
// (every kernel triggers its dependents after its own wait).  So whatever none
// of the direct predecessors writes may be read ahead of the wait, under their
// tails and the launch gap: a prep's operand blocks (all or nothing per prep),
// a combine's C_in.
void mark_early_loads(std::vector<Step>& steps, const DagPlan* d, int on) {
    int last[kLanes];
    for (int l = 0; l < kLanes; ++l) last[l] = -1;
    auto hit = [](const std::vector<View>& x, const std::vector<View>& y) {
        for (const View& u : x)
            for (const View& v : y)
                if (u.phys_overlaps(v)) return true;
        return false;
    };
    for (std::size_t j = 0; j < steps.size(); ++j) {
        Step& s = steps[j];
        const int lane = d ? d->lane[j] : 0;
        if (s.kind == Step::FPREP || s.kind == Step::FCOMB) {
            // what is read ahead: the prep's whole read set, the combine's C block
            const std::vector<View>& reads = s.kind == Step::FPREP ? s.rd : s.wr;
            bool free_of = true;
            if (last[lane] >= 0) free_of = !hit(steps[last[lane]].wr, reads);
            if (d)
                for (int w : d->waits[j]) free_of = free_of && !hit(steps[w].wr, reads);
            if (s.kind == Step::FPREP) s.fprep.early = (on & 1) && s.fprep.limbs && free_of ? 1u : 0u;
            else s.fcomb.early = (on & 2) && free_of ? 1u : 0u;
        }
        last[lane] = static_cast<int>(j);
    }
    if (std::getenv("WM_EARLY_DUMP")) {  // how many launches read ahead of their wait
        int np = 0, ep = 0, nc = 0, ec = 0;
        for (const Step& s : steps) {
            np += s.kind == Step::FPREP, ep += s.kind == Step::FPREP && s.fprep.early;
            nc += s.kind == Step::FCOMB, ec += s.kind == Step::FCOMB && s.fcomb.early;
        }
        std::fprintf(stderr, "early loads: %d of %d preps, %d of %d combines\n", ep, np, ec, nc);
    }
}

void fill_report(const Plan& plan, const std::vector<Step>* steps, wm_report* r) {
    if (!r) return;
    std::memset(r, 0, sizeof(*r));
    r->mults = plan.meter.mults;
    r->adds = plan.meter.adds;
    r->peak_extra_words = plan.meter.peak;
    r->total_alloc_words = plan.meter.total;
    r->word_moves = plan.meter.word_moves;
    r->classical_calls = plan.meter.classical_calls;
    for (const auto& kv : plan.meter.schedule_calls) r->schedule_frames += kv.second;
    r->peak_extra_bytes = plan.arena_words * sizeof(double);
    r->n_ops = plan.ops.size();
    for (const auto& op : plan.ops) r->fused_frames += op.kind == OP_FRAME;
    if (steps) r->n_launches = steps->size();
    r->add_bytes = (3 * plan.meter.add2_elems + 2 * plan.meter.copy_elems) * sizeof(double);
    r->leaf_flops = plan.meter.leaf_flops;
    if (steps) {
        for (const Step& s : *steps) {
            if (s.kind == Step::ADD)
                for (int i = 0; i < s.add.n; ++i)
                    r->add_bytes_issued += (s.add.it[i].mode <= M_GEN ? 3 : 2) *
                                           static_cast<std::uint64_t>(s.add.it[i].rows) *
                                           s.add.it[i].cols * sizeof(double);
            if (s.kind == Step::FGEMM) {
                const GemmParams& G = s.fgemm;
                const std::uint64_t mk = static_cast<std::uint64_t>(G.m) * G.k,
                                    kn = static_cast<std::uint64_t>(G.k) * G.n,
                                    mn = static_cast<std::uint64_t>(G.m) * G.n;
                r->frame_leaf_flops += 2ull * G.m * G.k * G.n * G.nprod;
                for (std::uint32_t i = 0; i < G.nprod; ++i)
                    r->frame_gemm_bytes += mk * (G.a[i].fmt != 0 ? 2 : 8) +
                                           kn * (G.b[i].fmt != 0 ? 2 : 8) +
                                           mn * (G.c[i].fmt != 0 ? 2 : 8);
            }
            if (s.kind == Step::FPREP) {
                const std::uint64_t c2 = static_cast<std::uint64_t>(s.fprep.c) * s.fprep.c;
                r->frame_bytes += (4 + 4 + 4 + (s.fprep.beta ? 4 : 0)) * c2 * sizeof(double);
                int planes = 0;
                for (int i = 0; i < PL_COUNT; ++i) planes += s.fprep.plane[i] != nullptr;
                r->frame_prep_bytes += (8 + (s.fprep.beta ? 4 : 0)) * c2 * sizeof(double) +
                                       planes * c2 * 2 + (s.fprep.beta ? c2 * 8 : 0);
                for (const FrameFold& ff : s.fprep.fold)  // folded operands: second source, store
                    if (ff.on)
                        r->frame_prep_bytes += ((ff.s1[0] ? 4 : 0) + (ff.writeback ? 4 : 0)) * c2 *
                                               sizeof(double);
            }
            if (s.kind == Step::FCOMB) {
                const std::uint64_t c2 = static_cast<std::uint64_t>(s.fcomb.c) * s.fcomb.c;
                r->frame_comb_bytes += 7 * c2 * 2 + (s.fcomb.beta ? c2 * 8 : 0) + 4 * c2 * sizeof(double);
            }
            if (s.kind == Step::GROUP) {
                const fused::GroupDesc& G = fused::kGroups[s.gid];
                r->add_bytes_issued += static_cast<std::uint64_t>(G.nload + G.nstore) *
                                       s.grp.rows * s.grp.cols * sizeof(double);
            }
        }
    }
    std::ostringstream os;
    bool first = true;
    for (const auto& kv : plan.meter.schedule_calls) {
        os << (first ? "" : ",") << kv.first << ":" << kv.second;
        first = false;
    }
    g_sched_calls = os.str();
    g_alloc_log = plan.alloc_log;
}

Scalar modp_scalar(const Field& f, std::uint32_t v) {
    Scalar s;
    s.r = v % f.p;
    s.d = static_cast<double>(static_cast<std::int32_t>(v));  // REAL64 primitives: signed
    return s;
}
Scalar real_scalar(double v) {
    Scalar s;
    s.r = 0;
    s.d = v;
    return s;
}

void check_dmat(const wm_dmat& m, const char* name) {
    if (m.rows == 0 || m.cols == 0) fail(E_DIMENSION, std::string(name) + ": empty matrix");
    if (m.ld < m.cols) fail(E_DIMENSION, std::string(name) + ": ld < cols");
    if (!m.ptr) fail(E_INVALID, std::string(name) + ": null pointer");
}

// The host u32 boundary streamed through the step graph: uploads (pinned host ->
// staging -> float64) and downloads per quadrant, as steps of their own on a
// copy-in and a copy-out lane, so that the product starts as soon as the
// quadrants its first operations read are resident and a C quadrant leaves as
// soon as its last writer is done.
struct HostIO {
    std::uint32_t* h[3] = {nullptr, nullptr, nullptr};  // A, B, C (row-major, ld = cols)
    std::uint32_t* stage[3] = {nullptr, nullptr, nullptr};
    bool up[3] = {false, false, false}, down[3] = {false, false, false};
};

void add_io_steps(std::vector<Step>& steps, const HostIO& io, const wm_dmat M[3], std::uint32_t p) {
    std::vector<Step> ups, downs;
    std::vector<std::size_t> first_use;
    for (int w = 0; w < 3; ++w) {
        if (!io.up[w] && !io.down[w]) continue;
        const std::uint64_t r = M[w].rows, c = M[w].cols;
        const int parts = r % 2 == 0 && c % 2 == 0 ? 2 : 1;  // quadrants
        for (int q = 0; q < parts * parts; ++q) {
            const std::uint64_t br = r / parts, bc = c / parts;
            const std::uint64_t r0 = (q / parts) * br, c0 = (q % parts) * bc;
            Step st{};
            st.hptr = io.h[w] + r0 * c + c0;
            st.sptr = io.stage[w] + r0 * c + c0;
            st.dptr = M[w].ptr + r0 * M[w].ld + c0;
            st.hld = st.sld = c;
            st.dld = M[w].ld;
            st.io_rows = br;
            st.io_cols = bc;
            st.io_p = p;
            View v;
            v.region = static_cast<std::uint8_t>(w);
            v.origin = w;
            v.off = r0 * M[w].ld + c0;
            v.rows = br;
            v.cols = bc;
            v.ld = M[w].ld;
            if (io.up[w]) {
                Step u = st;
                u.kind = Step::UPLOAD;
                u.lane_hint = 0;
                u.wr.push_back(v);
                std::size_t fu = steps.size();
                for (std::size_t j = 0; j < steps.size() && fu == steps.size(); ++j)
                    for (const View& x : steps[j].rd)
                        if (x.phys_overlaps(v)) {
                            fu = j;
                            break;
                        }
                ups.push_back(u);
                first_use.push_back(fu);
            }
            if (io.down[w]) {
                Step d = st;
                d.kind = Step::DOWNLOAD;
                d.lane_hint = 1;
                d.rd.push_back(v);
                downs.push_back(d);
            }
        }
    }
    // copy-in in order of first use: the lane is one PCIe stream
    std::vector<std::size_t> order(ups.size());
    for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](std::size_t a, std::size_t b) { return first_use[a] < first_use[b]; });
    std::vector<Step> out;
    out.reserve(ups.size() + steps.size() + downs.size());
    for (std::size_t i : order) out.push_back(ups[i]);
    for (Step& st : steps) out.push_back(std::move(st));
    for (Step& st : downs) out.push_back(std::move(st));
    steps.swap(out);
}

// Grow the context's arena to `words` (cached plans embed its address: they
// are dropped, after the stream has drained, when it moves).
void ensure_arena(wm_ctx* ctx, std::uint64_t words) {
    if (words <= ctx->arena_words) return;
    WM_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->cache.clear();
    ctx->traced = nullptr;
    if (ctx->arena) WM_CUDA(cudaFree(ctx->arena));
    ctx->arena = nullptr;
    ctx->arena_words = 0;
    WM_CUDA(cudaMalloc(&ctx->arena, words * sizeof(double)));
    ctx->arena_words = words;
}

// A plan whose every operation is tiny (the unit-size recursions of the
// reference's test shapes) runs as ONE micro launch over its operation list
// (wm_micro.cu) instead of one launch per operation.
bool micro_plan(const wm_ctx& ctx, const Plan& plan, double* const base[4], CachedPlan& cp,
                const wm_dmat& A, const wm_dmat& B, const wm_dmat& C) {
    if (!ctx.micro || ctx.f.real || ctx.subset || ctx.trace || plan.ops.empty()) return false;
    for (const Op& op : plan.ops) {
        if (op.kind == OP_FRAME || op.d.words() > kMicroMaxWords) return false;
        if (op.kind == OP_MUL && op.a.rows * op.a.cols * op.b.cols > kMicroMaxLeafVolume) return false;
    }
    // stage the working set in shared memory when it fits: operands then carry
    // byte offsets into the image instead of addresses
    MicroImage& img = cp.micro_img;
    img = MicroImage{};
    const std::uint64_t shape[4][3] = {{A.rows, A.cols, A.ld}, {B.rows, B.cols, B.ld},
                                       {C.rows, C.cols, C.ld}, {1, plan.arena_words, plan.arena_words}};
    std::uint64_t words = 0;
    for (int r = 0; r < 4; ++r) {
        if (!shape[r][1]) continue;
        MicroRegion& R = img.region[img.nregions++];
        R = {base[r], shape[r][0], shape[r][1], shape[r][2], words, r < 3 ? 1 : 0, r < 3 ? 1 : 0};
        words += shape[r][0] * shape[r][2];
    }
    img.words = words;
    double* off[4] = {nullptr, nullptr, nullptr, nullptr};
    const bool smem = words * sizeof(double) <= micro_smem_limit();
    if (smem) {
        int i = 0;
        for (int r = 0; r < 4; ++r)
            if (shape[r][1]) off[r] = reinterpret_cast<double*>(img.region[i++].offset * sizeof(double));
    } else {
        img.nregions = 0;
    }
    double* const* addr = smem ? off : base;
    std::vector<MicroOp> ops;
    ops.reserve(plan.ops.size());
    bool small = true;
    for (const Op& op : plan.ops) {
        MicroOp m{};
        if (op.kind == OP_MUL) {
            const MulParams P = make_mul(op, ctx.f, addr);
            m.d = P.C, m.a = P.A, m.b = P.B;
            m.ldd = static_cast<std::uint32_t>(P.ldc), m.lda = static_cast<std::uint32_t>(P.lda);
            m.ldb = static_cast<std::uint32_t>(P.ldb);
            m.rows = P.m, m.cols = P.n, m.k = P.k;
            m.kind = MicroOp::MUL;
            m.sa = P.alpha, m.sb = P.beta;
            small = small && static_cast<std::uint64_t>(P.m) * P.n * P.k <= kMicroSmallLeafVolume;
        } else {
            const AddItem t = make_item(op, ctx.f, addr);
            m.d = t.d, m.a = t.a, m.b = t.b;
            m.ldd = static_cast<std::uint32_t>(t.ldd), m.lda = static_cast<std::uint32_t>(t.lda);
            m.ldb = static_cast<std::uint32_t>(t.ldb);
            m.rows = t.rows, m.cols = t.cols;
            m.kind = MicroOp::ADD;
            m.mode = t.mode, m.sa = t.sa, m.sb = t.sb;
            small = small && static_cast<std::uint64_t>(t.rows) * t.cols <= kMicroSmallWords;
        }
        m.csh = (m.cols & (m.cols - 1)) == 0 ? static_cast<std::uint32_t>(__builtin_ctz(m.cols)) : 0xFFu;
        ops.push_back(m);
    }
    WM_CUDA(cudaMalloc(&cp.micro, ops.size() * sizeof(MicroOp)));
    WM_CUDA(cudaMemcpy(cp.micro, ops.data(), ops.size() * sizeof(MicroOp), cudaMemcpyHostToDevice));
    cp.micro_n = static_cast<std::uint32_t>(ops.size());
    cp.micro_small = small;
    return true;
}

void run(wm_ctx* ctx, const std::string& variant, const wm_dmat& A, const wm_dmat& B,
         const wm_dmat& C, Scalar alpha, Scalar beta, int cutoff, wm_report* rep,
         const Schedule* parsed = nullptr, const HostIO* io = nullptr) {
    check_dmat(A, "A");
    check_dmat(B, "B");
    check_dmat(C, "C");
    if (B.rows != A.cols || C.rows != A.rows || C.cols != B.cols)
        fail(E_DIMENSION, "multiply dimensions do not conform");
    std::ostringstream key;
    if (parsed) key << "dsl:" << render_schedule(*parsed);
    key << variant << '|' << ctx->f.real << '|' << ctx->f.p << '|' << A.rows << 'x' << A.cols
        << 'x' << B.cols << '|' << A.ld << ',' << B.ld << ',' << C.ld << '|' << alpha.r << ','
        << beta.r << ',' << alpha.d << ',' << beta.d << '|' << cutoff << '|' << ctx->fuse_frames
        << ctx->batch_adds << ctx->leaf_kernel << ctx->subset << ctx->fuse_adds << ctx->gemm_engine << ctx->direct_frames << ctx->dag << ctx->fold << ctx->trace << ctx->stream_io << ctx->micro << ctx->dead_hosts << '.' << ctx->epoch << '.' << ctx->wide_plain << ctx->cin_direct << ctx->early_loads << '|' << A.ptr << ',' << B.ptr << ',' << C.ptr;
    if (io)
        for (int w = 0; w < 3; ++w)
            key << "|io" << w << ':' << io->h[w] << ',' << io->stage[w] << ',' << io->up[w] << io->down[w];
    const std::string k = key.str();
    CachedPlan* cp = nullptr;
    for (auto it = ctx->cache.begin(); it != ctx->cache.end(); ++it)
        if (it->first == k) {
            ctx->cache.splice(ctx->cache.begin(), ctx->cache, it);
            cp = ctx->cache.front().second.get();
            break;
        }
    if (!cp) {
        PlanOptions opt;
        // the fused frame kernels move 16-byte vectors and TMA boxes over the
        // caller's blocks: they need even leading dimensions and 16-B aligned
        // bases (every quadrant offset is then a multiple of 64 elements)
        const bool frame_aligned = A.ld % 2 == 0 && B.ld % 2 == 0 && C.ld % 2 == 0 &&
                                   aligned16(A.ptr) && aligned16(B.ptr) && aligned16(C.ptr);
        opt.fuse_frames = ctx->fuse_frames && frame_kernel_available() && frame_aligned;
        opt.parsed = parsed;
        auto np = std::make_unique<CachedPlan>();
        np->plan = plan_variant(variant, ctx->f, A.rows, A.cols, B.cols, A.ld, B.ld, C.ld, alpha,
                                beta, cutoff, opt);
        ensure_arena(ctx, np->plan.arena_words);
        double* base[4] = {A.ptr, B.ptr, C.ptr, ctx->arena};
        if (!io && micro_plan(*ctx, np->plan, base, *np, A, B, C)) {
            // tiny plan: nothing to lower
        } else try {
            np->steps = lower(np->plan, base, *ctx);
        } catch (const Error& e) {
            // a frame GEMM the tensor-map path cannot describe: plan again with
            // every frame unfused (nothing has been issued yet)
            if (e.code != E_INVALID || !opt.fuse_frames) throw;
            opt.fuse_frames = false;
            np->plan = plan_variant(variant, ctx->f, A.rows, A.cols, B.cols, A.ld, B.ld, C.ld,
                                    alpha, beta, cutoff, opt);
            ensure_arena(ctx, np->plan.arena_words);
            base[3] = ctx->arena;
            np->steps = lower(np->plan, base, *ctx);
        }
        if (io) {
            const wm_dmat M[3] = {A, B, C};
            add_io_steps(np->steps, *io, M, ctx->f.p);
        }
        ctx->cache.emplace_front(k, std::move(np));
        while (ctx->cache.size() > 8) ctx->cache.pop_back();
        cp = ctx->cache.front().second.get();
    }
    if (cp->micro) {
        WM_CUDA(launch_micro(cp->micro, cp->micro_n, cp->micro_img, cp->micro_small, ctx->f.p,
                             ctx->stream));
        fill_report(cp->plan, nullptr, rep);
        if (rep) rep->n_launches = 1;
        return;
    }
    // concurrent issue pays only for launches of real size; tiny problems (deep
    // recursions of the unit tests) would spend more on the dependency analysis
    const bool dag = io || (ctx->dag > 1 && ctx->subset == 0 && cp->steps.size() > 1 &&
                            std::max({A.rows, A.cols, B.cols}) >= 512 && cp->steps.size() <= 200000);
    // with the boundary in the graph, one dependency epoch spans the whole step
    // (up to 4096 launches) so C quadrants can leave while the rest computes
    if (dag && !cp->dag)
        cp->dag = std::make_shared<DagPlan>(plan_dag(
            cp->steps, std::max(1, ctx->dag),
            io ? std::max(ctx->epoch, std::min<int>(4096, static_cast<int>(cp->steps.size())))
               : ctx->epoch));
    if (!cp->exec && !cp->early_marked) {
        // (the subset replays issue other launch sequences: no early loads there)
        mark_early_loads(cp->steps, dag ? cp->dag.get() : nullptr, ctx->subset == 0 ? ctx->early_loads : 0);
        cp->early_marked = true;
    }
    if (ctx->trace) {
        // [start, end] globaltimer slots per launch, patched into the launch
        // parameters of this (trace-keyed) plan before its graph is captured
        if (!cp->tl) {
            WM_CUDA(cudaMalloc(&cp->tl, 2 * cp->steps.size() * sizeof(unsigned long long)));
            for (std::size_t j = 0; j < cp->steps.size(); ++j) {
                Step& st = cp->steps[j];
                unsigned long long* slot = cp->tl + 2 * j;
                st.add.tl = st.mul.tl = st.fprep.tl = st.fcomb.tl = st.fgemm.tl = st.tl = slot;
            }
        }
        std::vector<unsigned long long> init(2 * cp->steps.size(), 0ull);
        for (std::size_t j = 0; j < cp->steps.size(); ++j) init[2 * j] = ~0ull;
        WM_CUDA(cudaMemcpyAsync(cp->tl, init.data(), init.size() * sizeof(unsigned long long),
                                cudaMemcpyHostToDevice, ctx->stream));
        WM_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->traced = cp;
    }
    auto go = [&]() {
        if (dag)
            issue_dag(cp->steps, *cp->dag, ctx->f.real, ctx->stream, ctx->lanes);
        else issue(cp->steps, ctx->f.real, ctx->stream, ctx->subset);
    };
    // capture pays for the launch-bound plans of real problems; the 10^5-launch
    // plans of unit-size recursions (cutoff 1) are cheaper to issue directly
    if (ctx->graphs && cp->steps.size() > 1 && cp->steps.size() <= 50000) {
        if (!cp->exec) {
            WM_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
            try {
                go();
            } catch (...) {
                cudaGraph_t g = nullptr;
                cudaStreamEndCapture(ctx->stream, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            WM_CUDA(cudaStreamEndCapture(ctx->stream, &cp->graph));
            WM_CUDA(cudaGraphInstantiate(&cp->exec, cp->graph, 0));
        }
        WM_CUDA(cudaGraphLaunch(cp->exec, ctx->stream));
    } else {
        go();
    }
    fill_report(cp->plan, &cp->steps, rep);
}

double* ensure_buf(wm_ctx* ctx, int i, std::size_t words) {
    if (ctx->hbuf_words[i] < words) {
        if (ctx->hbuf[i]) WM_CUDA(cudaFree(ctx->hbuf[i]));
        ctx->hbuf[i] = nullptr;
        WM_CUDA(cudaMalloc(&ctx->hbuf[i], words * sizeof(double)));
        ctx->hbuf_words[i] = words;
    }
    return ctx->hbuf[i];
}

std::uint32_t* ensure_stage(wm_ctx* ctx, std::size_t words) {
    if (ctx->stage_words < words) {
        if (ctx->stage) WM_CUDA(cudaFree(ctx->stage));
        ctx->stage = nullptr;
        WM_CUDA(cudaMalloc(&ctx->stage, words * sizeof(std::uint32_t)));
        ctx->stage_words = words;
    }
    return ctx->stage;
}

void upload(wm_ctx* ctx, const wm_dmat& dst, const std::uint32_t* host, std::uint64_t hld) {
    check_dmat(dst, "dst");
    std::uint32_t* st = ensure_stage(ctx, dst.rows * dst.cols);
    WM_CUDA(cudaMemcpy2DAsync(st, dst.cols * 4, host, hld * 4, dst.cols * 4, dst.rows,
                              cudaMemcpyHostToDevice, ctx->stream));
    WM_CUDA(launch_u32_to_f64(dst.ptr, dst.ld, st, dst.cols, dst.rows, dst.cols, ctx->stream));
}

void download(wm_ctx* ctx, std::uint32_t* host, std::uint64_t hld, const wm_dmat& src) {
    check_dmat(src, "src");
    std::uint32_t* st = ensure_stage(ctx, src.rows * src.cols);
    WM_CUDA(launch_f64_to_u32(st, src.cols, src.ptr, src.ld, src.rows, src.cols, ctx->f.p,
                              ctx->stream));
    WM_CUDA(cudaMemcpy2DAsync(host, hld * 4, st, src.cols * 4, src.cols * 4, src.rows,
                              cudaMemcpyDeviceToHost, ctx->stream));
}

// Host u32 boundary (the reference's Matrix&): upload, run, download C and
// whatever the contract lets the schedule overwrite.  C_in is uploaded whenever
// the schedule reads it (beta != 0 or an accumulating schedule).
void host_run(wm_ctx* ctx, const std::string& v, const Schedule* parsed, uint64_t m, uint64_t k,
              uint64_t n, uint32_t* A, uint32_t* B, uint32_t* C, uint32_t alpha, uint32_t beta,
              int cutoff, wm_report* report) {
    if (ctx->f.real) fail(E_INVALID, "host u32 entry needs a MODP context");
    if (!A || !B || !C) fail(E_INVALID, "null host buffer");
    wm_dmat dA{ensure_buf(ctx, 0, m * k), m, k, k};
    wm_dmat dB{ensure_buf(ctx, 1, k * n), k, n, n};
    wm_dmat dC{ensure_buf(ctx, 2, m * n), m, n, n};
    const bool acc0 = parsed ? parsed->accumulating : (v != "classic" && variant_accumulates(v));
    const Contract c0 = parsed ? parsed->contract : variant_contract(v);
    auto pinned = [](const void* ptr) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    };
    // streamed when the copies are long enough to hide compute behind (measured:
    // config 2's e2e 9.8 -> 7.9 ms; a 1024^3 problem gains nothing)
    if (ctx->graphs && ctx->stream_io && m * k + k * n + m * n >= (8ull << 20) && pinned(A) &&
        pinned(B) && pinned(C)) {
        HostIO io;
        std::uint32_t* st = ensure_stage(ctx, m * k + k * n + m * n);
        io.h[0] = A, io.h[1] = B, io.h[2] = C;
        io.stage[0] = st, io.stage[1] = st + m * k, io.stage[2] = st + m * k + k * n;
        io.up[0] = io.up[1] = true;
        io.up[2] = beta % ctx->f.p != 0 || acc0;
        io.down[2] = true;
        io.down[0] = c0 == Contract::OverwriteA || c0 == Contract::OverwriteBoth;
        io.down[1] = c0 == Contract::OverwriteB || c0 == Contract::OverwriteBoth;
        run(ctx, v, dA, dB, dC, modp_scalar(ctx->f, alpha), modp_scalar(ctx->f, beta), cutoff,
            report, parsed, &io);
        WM_CUDA(cudaStreamSynchronize(ctx->stream));
        return;
    }
    upload(ctx, dA, A, k);
    upload(ctx, dB, B, n);
    const bool acc = parsed ? parsed->accumulating : (v != "classic" && variant_accumulates(v));
    if (beta % ctx->f.p != 0 || acc) upload(ctx, dC, C, n);
    run(ctx, v, dA, dB, dC, modp_scalar(ctx->f, alpha), modp_scalar(ctx->f, beta), cutoff, report,
        parsed);
    download(ctx, C, n, dC);
    const Contract c = parsed ? parsed->contract : variant_contract(v);
    if (c == Contract::OverwriteA || c == Contract::OverwriteBoth) download(ctx, A, k, dA);
    if (c == Contract::OverwriteB || c == Contract::OverwriteBoth) download(ctx, B, n, dB);
    WM_CUDA(cudaStreamSynchronize(ctx->stream));
}

template <class F>
int guard(F&& fn) {
    try {
        fn();
        return WM_OK;
    } catch (const Error& e) {
        return set_err(e.code, e.what());
    } catch (const std::exception& e) {
        return set_err(E_INVALID, e.what());
    }
}

// Primitive calls on raw pointers: all device memory is one "region"; views
// over distinct allocations never overlap physically, so the exact /
// span tests of MatView::overlaps apply to the addresses directly.
View raw_view(const wm_dmat& m) {
    View v;
    v.region = 0;
    v.origin = 0;
    v.base = 0;
    v.off = reinterpret_cast<std::uintptr_t>(m.ptr) / sizeof(double);
    v.rows = m.rows;
    v.cols = m.cols;
    v.ld = m.ld;
    return v;
}

}  // namespace

extern "C" {

const char* wm_version(void) { return "winomem-b200 0.1 (sm_100a)"; }
const char* wm_last_error(void) { return g_err.c_str(); }

int wm_ctx_create(int device, uint32_t p, int field, void* stream, wm_ctx** out) {
    return guard([&] {
        if (!out) fail(E_INVALID, "null out");
        *out = nullptr;
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
            fail(E_CUDA, "no CUDA device: winomem-b200 has no CPU fallback");
        if (device < 0 || device >= n) fail(E_INVALID, "bad device ordinal");
        if (field != WM_FIELD_MODP && field != WM_FIELD_REAL64) fail(E_INVALID, "bad field");
        if (field == WM_FIELD_MODP) {
            bool prime = p > 2 && (p & 1);
            for (std::uint32_t d = 3; prime && static_cast<std::uint64_t>(d) * d <= p; d += 2)
                prime = p % d != 0;
            if (!prime) fail(E_DIMENSION, "modulus must be an odd prime: " + std::to_string(p));
            if (p >= (1u << 16))
                fail(E_DIMENSION, "device path supports p < 2^16 (exact float64 accumulation)");
        }
        auto c = std::make_unique<wm_ctx>();
        c->device = device;
        c->f.real = field == WM_FIELD_REAL64;
        c->f.p = field == WM_FIELD_REAL64 ? 65521u : p;
        WM_CUDA(cudaSetDevice(device));
        WM_CUDA(leaf_i8_init());
        const bool tma_ok = gemm_tma_init() == cudaSuccess;
        c->gemm_engine = tma_ok ? 1 : 0;
        c->direct_ok = tma_ok && gemm_direct_init() == cudaSuccess;
        if (stream) {
            c->stream = static_cast<cudaStream_t>(stream);
        } else {
            WM_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            c->own_stream = true;
        }
        *out = c.release();
    });
}

int wm_ctx_destroy(wm_ctx* ctx) {
    if (ctx) {
        cudaStreamSynchronize(ctx->stream);
        delete ctx;
    }
    return WM_OK;
}

int wm_ctx_sync(wm_ctx* ctx) {
    return guard([&] { WM_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int wm_ctx_info(wm_ctx* ctx, int* device, uint32_t* p, int* field, void** stream) {
    return guard([&] {
        if (!ctx) fail(E_INVALID, "null context");
        if (device) *device = ctx->device;
        if (p) *p = ctx->f.p;
        if (field) *field = ctx->f.real ? WM_FIELD_REAL64 : WM_FIELD_MODP;
        if (stream) *stream = ctx->stream;
    });
}

int wm_ctx_set_stream(wm_ctx* ctx, void* stream) {
    return guard([&] {
        if (!ctx || !stream) fail(E_INVALID, "null context or stream");
        ctx->stream = static_cast<cudaStream_t>(stream);
    });
}

int wm_ctx_set_option(wm_ctx* ctx, const char* key, int64_t value) {
    return guard([&] {
        const std::string k = key ? key : "";
        if (k == "fuse_frames") ctx->fuse_frames = value != 0;
        else if (k == "graphs") ctx->graphs = value != 0;
        else if (k == "batch_adds") ctx->batch_adds = value != 0;
        else if (k == "leaf_kernel") ctx->leaf_kernel = static_cast<int>(value);
        else if (k == "subset") ctx->subset = static_cast<int>(value);
        else if (k == "fuse_adds") ctx->fuse_adds = value != 0;
        else if (k == "direct_frames") ctx->direct_frames = value != 0;
        else if (k == "dag") ctx->dag = static_cast<int>(value);
        else if (k == "pdl") g_pdl_user = value != 0;
        else if (k == "prep_rows") g_prep_rows = static_cast<int>(value);
        else if (k == "comb_block") g_comb_block = static_cast<unsigned>(value);
        else if (k == "fold") ctx->fold = value != 0;
        else if (k == "stream_io") ctx->stream_io = value != 0;
        else if (k == "micro") ctx->micro = value != 0;
        else if (k == "dead_hosts") ctx->dead_hosts = value != 0;
        else if (k == "epoch") ctx->epoch = value < 16 ? 16 : static_cast<int>(value);
        else if (k == "wide_plain") ctx->wide_plain = value != 0;
        else if (k == "cin_direct") ctx->cin_direct = value != 0;
        else if (k == "early_loads") ctx->early_loads = static_cast<int>(value);
        else if (k == "trace") ctx->trace = value != 0;
        else if (k == "gemm_engine") ctx->gemm_engine = static_cast<int>(value);
        else fail(E_INVALID, "unknown option " + k);
        ctx->cache.clear();
    });
}

int wm_ctx_get_option(wm_ctx* ctx, const char* key, int64_t* value) {
    return guard([&] {
        const std::string k = key ? key : "";
        if (k == "fuse_frames") *value = ctx->fuse_frames;
        else if (k == "graphs") *value = ctx->graphs;
        else if (k == "batch_adds") *value = ctx->batch_adds;
        else if (k == "leaf_kernel") *value = ctx->leaf_kernel;
        else if (k == "subset") *value = ctx->subset;
        else if (k == "fuse_adds") *value = ctx->fuse_adds;
        else if (k == "direct_frames") *value = ctx->direct_frames;
        else if (k == "dag") *value = ctx->dag;
        else if (k == "pdl") *value = g_pdl_user;
        else if (k == "prep_rows") *value = g_prep_rows;
        else if (k == "comb_block") *value = g_comb_block;
        else if (k == "fold") *value = ctx->fold;
        else if (k == "stream_io") *value = ctx->stream_io;
        else if (k == "micro") *value = ctx->micro;
        else if (k == "arena_words") *value = static_cast<int64_t>(ctx->arena_words);  // read-only
        else if (k == "dead_hosts") *value = ctx->dead_hosts;
        else if (k == "epoch") *value = ctx->epoch;
        else if (k == "wide_plain") *value = ctx->wide_plain;
        else if (k == "cin_direct") *value = ctx->cin_direct;
        else if (k == "early_loads") *value = ctx->early_loads;
        else if (k == "trace") *value = ctx->trace;
        else if (k == "gemm_engine") *value = ctx->gemm_engine;
        else fail(E_INVALID, "unknown option " + k);
    });
}

int wm_block_addsub(wm_ctx* ctx, wm_dmat dst, wm_dmat a, wm_dmat b, uint32_t sa, uint32_t sb) {
    return guard([&] {
        check_dmat(dst, "dst");
        check_dmat(a, "a");
        check_dmat(b, "b");
        const View d = raw_view(dst), va = raw_view(a), vb = raw_view(b);
        if (a.rows != b.rows || a.cols != b.cols || dst.rows != a.rows || dst.cols != a.cols)
            fail(E_DIMENSION, "block_addsub dimension mismatch");
        if (!d.same_window(va) && d.overlaps(va))
            fail(E_PARTIAL_OVERLAP, "block_addsub: dst partially overlaps a");
        if (!d.same_window(vb) && d.overlaps(vb))
            fail(E_PARTIAL_OVERLAP, "block_addsub: dst partially overlaps b");
        Op op{};
        op.kind = OP_ADDSUB;
        op.d = d;
        op.a = va;
        op.b = vb;
        op.sa = modp_scalar(ctx->f, sa);
        op.sb = modp_scalar(ctx->f, sb);
        // raw views are absolute element addresses from a null base
        op.d.region = op.a.region = op.b.region = 0;
        double* base[4] = {nullptr, nullptr, nullptr, nullptr};
        Step s{};
        s.kind = Step::ADD;
        init_batch(s.add, ctx->f);
        AddItem t = make_item(op, ctx->f, base);
        t.blk0 = 0;
        s.add.it[0] = t;
        s.add.n = 1;
        s.blocks = item_blocks(t);
        WM_CUDA(launch_addsub(s.add, ctx->f.real, s.blocks, ctx->stream));
    });
}

int wm_block_scale_copy(wm_ctx* ctx, wm_dmat dst, wm_dmat src, uint32_t s) {
    return guard([&] {
        check_dmat(dst, "dst");
        check_dmat(src, "src");
        const View d = raw_view(dst), v = raw_view(src);
        if (dst.rows != src.rows || dst.cols != src.cols)
            fail(E_DIMENSION, "block_scale_copy dimension mismatch");
        if (!d.same_window(v) && d.overlaps(v))
            fail(E_PARTIAL_OVERLAP, "block_scale_copy: dst partially overlaps src");
        if (ctx->f.is_one(modp_scalar(ctx->f, s)) && d.same_window(v)) return;
        Op op{};
        op.kind = OP_COPY;
        op.d = d;
        op.a = v;
        op.sa = modp_scalar(ctx->f, s);
        double* base[4] = {nullptr, nullptr, nullptr, nullptr};
        Step st{};
        init_batch(st.add, ctx->f);
        AddItem t = make_item(op, ctx->f, base);
        st.add.it[0] = t;
        st.add.n = 1;
        WM_CUDA(launch_addsub(st.add, ctx->f.real, item_blocks(t), ctx->stream));
    });
}

int wm_lincomb(wm_ctx* ctx, wm_dmat dst, int n, const wm_dmat* src, const uint32_t* coef) {
    return guard([&] {
        if (n < 1 || n > kMaxLincomb || !src || !coef) fail(E_INVALID, "lincomb takes 1..4 terms");
        check_dmat(dst, "dst");
        const View d = raw_view(dst);
        LincombParams L{};
        L.dst = dst.ptr;
        L.ldd = dst.ld;
        L.rows = dst.rows;
        L.cols = dst.cols;
        L.n = n;
        L.p = static_cast<double>(ctx->f.p);
        for (int t = 0; t < n; ++t) {
            check_dmat(src[t], "src");
            if (src[t].rows != dst.rows || src[t].cols != dst.cols)
                fail(E_DIMENSION, "lincomb dimension mismatch");
            const View v = raw_view(src[t]);
            if (!d.same_window(v) && d.overlaps(v))
                fail(E_PARTIAL_OVERLAP, "lincomb: dst partially overlaps a source");
            L.src[t] = src[t].ptr;
            L.lds[t] = src[t].ld;
            const Scalar sc = modp_scalar(ctx->f, coef[t]);
            L.coef[t] = ctx->f.real ? sc.d : static_cast<double>(sc.r);
        }
        WM_CUDA(launch_lincomb(L, ctx->f.real, ctx->stream));
    });
}

int wm_classical_mul(wm_ctx* ctx, wm_dmat C, wm_dmat A, wm_dmat B, uint32_t alpha, uint32_t beta) {
    return guard([&] {
        check_dmat(A, "A");
        check_dmat(B, "B");
        check_dmat(C, "C");
        if (B.rows != A.cols || C.rows != A.rows || C.cols != B.cols)
            fail(E_DIMENSION, "classical_mul dimension mismatch");
        const View vc = raw_view(C);
        if (vc.overlaps(raw_view(A)) || vc.overlaps(raw_view(B)))
            fail(E_ALIAS, "classical_mul: C must be disjoint from A and B");
        Op op{};
        op.kind = OP_MUL;
        op.d = vc;
        op.a = raw_view(A);
        op.b = raw_view(B);
        op.sa = modp_scalar(ctx->f, alpha);
        op.sb = modp_scalar(ctx->f, beta);
        double* base[4] = {nullptr, nullptr, nullptr, nullptr};
        MulParams P = make_mul(op, ctx->f, base);
        if (!ctx->f.real && (ctx->leaf_kernel == 1 || ctx->leaf_kernel == 2) && leaf_i8_supported(P))
            WM_CUDA(launch_leaf_i8(P, ctx->stream));
        else
            WM_CUDA(launch_leaf_dmma(P, ctx->f.real, ctx->stream));
    });
}

int wm_run_variant(wm_ctx* ctx, const char* variant, wm_dmat A, wm_dmat B, wm_dmat C,
                   uint32_t alpha, uint32_t beta, int cutoff, wm_report* report) {
    return guard([&] {
        if (ctx->f.real) fail(E_INVALID, "REAL64 context: use wm_run_variant_real");
        run(ctx, variant ? variant : "", A, B, C, modp_scalar(ctx->f, alpha),
            modp_scalar(ctx->f, beta), cutoff, report);
    });
}

int wm_ipmm(wm_ctx* ctx, wm_dmat A, wm_dmat B, wm_dmat C, int cutoff, wm_report* report) {
    return wm_run_variant(ctx, "ipmm", A, B, C, 1, 0, cutoff, report);
}

int wm_run_variant_real(wm_ctx* ctx, const char* variant, wm_dmat A, wm_dmat B, wm_dmat C,
                        double alpha, double beta, int cutoff, wm_report* report) {
    return guard([&] {
        if (!ctx->f.real) fail(E_INVALID, "MODP context: use wm_run_variant");
        run(ctx, variant ? variant : "", A, B, C, real_scalar(alpha), real_scalar(beta), cutoff,
            report);
    });
}

int wm_run_variant_host_u32(wm_ctx* ctx, const char* variant, uint64_t m, uint64_t k, uint64_t n,
                            uint32_t* A, uint32_t* B, uint32_t* C, uint32_t alpha, uint32_t beta,
                            int cutoff, wm_report* report) {
    return guard([&] {
        host_run(ctx, variant ? variant : "", nullptr, m, k, n, A, B, C, alpha, beta, cutoff, report);
    });
}

int wm_run_parsed_schedule_host_u32(wm_ctx* ctx, const char* text, uint64_t m, uint64_t k,
                                    uint64_t n, uint32_t* A, uint32_t* B, uint32_t* C,
                                    uint32_t alpha, uint32_t beta, int cutoff, wm_report* report) {
    return guard([&] {
        const Schedule s = parse_schedule(text ? text : "");
        host_run(ctx, s.name, &s, m, k, n, A, B, C, alpha, beta, cutoff, report);
    });
}

int wm_plan_report(const char* variant, int field, uint32_t p, uint64_t m, uint64_t k, uint64_t n,
                   uint32_t alpha, uint32_t beta, int cutoff, int fuse_frames, wm_report* report) {
    return guard([&] {
        Field f;
        f.real = field == WM_FIELD_REAL64;
        f.p = f.real ? 65521u : p;
        PlanOptions opt;
        opt.fuse_frames = fuse_frames != 0;
        Scalar a = f.real ? real_scalar(alpha) : modp_scalar(f, alpha);
        Scalar b = f.real ? real_scalar(beta) : modp_scalar(f, beta);
        Plan plan = plan_variant(variant ? variant : "", f, m, k, n, k, n, n, a, b, cutoff, opt);
        // lowered as a context would (pointer-free: counts and byte figures only)
        wm_ctx dummy;
        dummy.gemm_engine = 0;
        double* base[4] = {nullptr, nullptr, nullptr, nullptr};
        const std::vector<Step> steps = lower(plan, base, dummy);
        fill_report(plan, &steps, report);
    });
}

// The CostReport of run_parsed_schedule for DSL text, without executing.
int wm_plan_report_parsed(const char* text, uint32_t p, uint64_t m, uint64_t k, uint64_t n,
                          uint32_t alpha, uint32_t beta, int cutoff, wm_report* report) {
    return guard([&] {
        Field f;
        f.p = p;
        const Schedule s = parse_schedule(text ? text : "");
        PlanOptions opt;
        opt.parsed = &s;
        Plan plan = plan_variant(s.name, f, m, k, n, k, n, n, modp_scalar(f, alpha),
                                 modp_scalar(f, beta), cutoff, opt);
        fill_report(plan, nullptr, report);
    });
}

int wm_expected_costs(const char* variant, uint64_t m, uint64_t k, uint64_t n, int cutoff,
                      wm_report* report) {
    return guard([&] {
        Costs c = expected_costs(variant ? variant : "", m, k, n, cutoff);
        if (report) {
            std::memset(report, 0, sizeof(*report));
            report->mults = c.mults;
            report->adds = c.adds;
            report->peak_extra_words = c.peak;
            report->total_alloc_words = c.total;
            report->word_moves = c.moves;
        }
    });
}

// run_parsed_schedule (executor.hpp:304-342): a schedule given as DSL text
// executes at the top frame; its recursion tags dispatch to the builtins.
int wm_run_parsed_schedule(wm_ctx* ctx, const char* text, wm_dmat A, wm_dmat B, wm_dmat C,
                           uint32_t alpha, uint32_t beta, int cutoff, wm_report* report) {
    return guard([&] {
        if (ctx->f.real) fail(E_INVALID, "REAL64 context: parsed schedules run over Z/pZ");
        const Schedule s = parse_schedule(text ? text : "");
        run(ctx, s.name, A, B, C, modp_scalar(ctx->f, alpha), modp_scalar(ctx->f, beta), cutoff,
            report, &s);
    });
}

namespace {
int put_text(const std::string& t, char* out, int len) {
    if (out && len > 0) {
        std::strncpy(out, t.c_str(), static_cast<std::size_t>(len) - 1);
        out[len - 1] = 0;
    }
    return static_cast<int>(t.size());
}
}  // namespace

// parse_schedule + render_schedule: validates DSL text (E_PARSE,
// E_CONTRACT_VIOLATION) and writes this build's canonical rendering of it;
// *builtin_match = 1 when it is instruction-for-instruction the builtin of the
// same name.  Returns the status; *needed = rendered length.
int wm_parse_schedule(const char* text, char* out, int len, int* needed, int* builtin_match) {
    return guard([&] {
        const Schedule s = parse_schedule(text ? text : "");
        const int n = put_text(render_schedule(s), out, len);
        if (needed) *needed = n;
        if (builtin_match) *builtin_match = is_builtin(s.name) && same_schedule(s, builtin(s.name));
    });
}

// render_schedule of a builtin (E_UNKNOWN_SCHEDULE otherwise).
int wm_render_schedule(const char* name, char* out, int len, int* needed) {
    return guard([&] {
        const int n = put_text(render_schedule(builtin(name ? name : "")), out, len);
        if (needed) *needed = n;
    });
}

// ---- matrix files (ring.hpp:386-449) ---------------------------------------
int wm_matrix_file_info(const char* path, int binary, uint64_t* rows, uint64_t* cols, uint32_t* p) {
    return guard([&] {
        const MatrixFile m = read_matrix_file(path ? path : "", binary != 0, true);
        *rows = m.rows;
        *cols = m.cols;
        *p = m.p;
    });
}

int wm_matrix_read_host(const char* path, int binary, uint32_t* out, uint64_t capacity) {
    return guard([&] {
        const MatrixFile m = read_matrix_file(path ? path : "", binary != 0);
        if (m.data.size() > capacity) fail(E_INVALID, "output buffer smaller than the matrix");
        std::memcpy(out, m.data.data(), m.data.size() * sizeof(uint32_t));
    });
}

int wm_matrix_write_host(const char* path, int binary, uint64_t rows, uint64_t cols, uint32_t p,
                         const uint32_t* data) {
    return guard([&] { write_matrix_file(path ? path : "", binary != 0, rows, cols, p, data); });
}

// read straight into a device matrix (residues converted on the device); the
// file's shape must equal dst's and its modulus the context's
int wm_matrix_read_device(wm_ctx* ctx, const char* path, int binary, wm_dmat dst) {
    return guard([&] {
        if (ctx->f.real) fail(E_INVALID, "matrix files hold residues: MODP context needed");
        const MatrixFile m = read_matrix_file(path ? path : "", binary != 0);
        if (m.rows != dst.rows || m.cols != dst.cols) fail(E_DIMENSION, "file shape differs from the matrix");
        if (m.p != ctx->f.p) fail(E_DIMENSION, "file modulus differs from the context's");
        upload(ctx, dst, m.data.data(), m.cols);
        WM_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int wm_matrix_write_device(wm_ctx* ctx, const char* path, int binary, wm_dmat src) {
    return guard([&] {
        if (ctx->f.real) fail(E_INVALID, "matrix files hold residues: MODP context needed");
        std::vector<uint32_t> h(src.rows * src.cols);
        download(ctx, h.data(), src.cols, src);
        WM_CUDA(cudaStreamSynchronize(ctx->stream));
        write_matrix_file(path ? path : "", binary != 0, src.rows, src.cols, ctx->f.p, h.data());
    });
}

int wm_plan_alloc_log(char* out, int len) {
    std::ostringstream al;
    if (g_alloc_log)
        for (const auto& e : *g_alloc_log) al << e.words << ':' << e.depth << ':' << e.slot << ';';
    const std::string text = al.str();
    if (out && len > 0) {
        std::strncpy(out, text.c_str(), static_cast<std::size_t>(len) - 1);
        out[len - 1] = 0;
    }
    return static_cast<int>(text.size());
}

int wm_plan_schedule_calls(char* out, int len) {
    if (out && len > 0) {
        std::strncpy(out, g_sched_calls.c_str(), static_cast<std::size_t>(len) - 1);
        out[len - 1] = 0;
    }
    return static_cast<int>(g_sched_calls.size());
}

int wm_dev_alloc(wm_ctx* ctx, uint64_t words, double** out) {
    return guard([&] {
        if (!out || !words) fail(E_INVALID, "wm_dev_alloc: empty request");
        WM_CUDA(cudaSetDevice(ctx->device));
        WM_CUDA(cudaMalloc(out, words * sizeof(double)));
    });
}

void wm_dev_free(double* p) {
    if (p) cudaFree(p);
}

int wm_upload_u32(wm_ctx* ctx, wm_dmat dst, const uint32_t* host, uint64_t host_ld) {
    return guard([&] { upload(ctx, dst, host, host_ld); });
}

int wm_download_u32(wm_ctx* ctx, uint32_t* host, uint64_t host_ld, wm_dmat src) {
    return guard([&] {
        download(ctx, host, host_ld, src);
        WM_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

uint64_t wm_fnv1a64_u32(const uint32_t* data, uint64_t count) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (std::uint64_t i = 0; i < count; ++i) {
        h ^= data[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

int wm_fill_random(wm_ctx* ctx, wm_dmat dst, uint64_t seed) {
    return guard([&] {
        check_dmat(dst, "dst");
        WM_CUDA(launch_fill_splitmix(dst.ptr, dst.ld, dst.rows, dst.cols, seed, ctx->f.p,
                                     ctx->f.real, ctx->stream));
    });
}

#if WM_DIAG  // measurement-only exports: libwinomem_b200_diag.so (build.py)
#include "wm_runtime_diag.inc"
#endif

}  // extern "C"
