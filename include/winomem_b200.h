/*
 * winomem-b200: the C-ABI drop-in boundary for the memory-efficient
 * Strassen-Winograd schedules (Boyer, Dumas, Pernet, Zhou, ISSAC 2009) on
 * NVIDIA B200 (sm_100a).
 *
 * Plain pointers and sizes only.  Every entry point returns a status code
 * (WM_OK == 0) that mirrors the reference's C++ exception taxonomy; the message
 * of the last failure on the calling thread is available from wm_last_error().
 * The reference interface each entry replaces is cited beside it
 * (paths relative to /root/reference/proj/include/winomem/).
 *
 * Matrices live in device memory as row-major float64 with a leading
 * dimension (wm_dmat).  In the MODP field (Z/pZ, odd prime p < 2^16, the
 * reference's default p = 65521, ring.hpp:89) entries are canonical residues
 * held exactly in float64; in the REAL64 field they are ordinary doubles.
 * Host-buffer entry points (suffix _host_u32) take the reference's own element
 * type (uint32_t residues, ring.hpp:21) and do the upload / download and
 * conversion on the context's stream.
 *
 * Threading: one host thread per context; all work is issued in order on the
 * context's stream; there is no CPU fallback -- a context cannot be created
 * without a CUDA device.
 */
#ifndef WINOMEM_B200_H
#define WINOMEM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: ring.hpp:23-43, workspace.hpp:20-22, schedule.hpp:30-43 */
enum {
    WM_OK = 0,
    WM_E_DIMENSION = 1,          /* dimension_error */
    WM_E_ODD_DIMENSION = 2,      /* odd_dimension_error */
    WM_E_PARTIAL_OVERLAP = 3,    /* partial_overlap_error */
    WM_E_ALIAS = 4,              /* alias_error */
    WM_E_SHAPE = 5,              /* shape_error */
    WM_E_CONTRACT = 6,           /* contract_error */
    WM_E_IO = 7,                 /* io_error */
    WM_E_WORKSPACE = 8,          /* workspace_error */
    WM_E_UNKNOWN_SCHEDULE = 9,   /* unknown_schedule_error */
    WM_E_PARSE = 10,             /* parse_error */
    WM_E_CONTRACT_VIOLATION = 11,/* contract_violation_error */
    WM_E_CUDA = 12,              /* device error (new) */
    WM_E_NCCL = 13,              /* communication error (new) */
    WM_E_INVALID = 14,           /* invalid argument / state (new) */
    WM_E_UNKNOWN_SLOT = 15       /* unknown_slot_error */
};

enum { WM_FIELD_MODP = 0, WM_FIELD_REAL64 = 1 };

typedef struct wm_ctx wm_ctx;

/* A device matrix view: row-major float64, element (i,j) at ptr[i*ld + j]. */
typedef struct {
    double* ptr;
    uint64_t rows, cols, ld;
} wm_dmat;

/* CostReport (meter.hpp:53-75) plus the device-side figures. */
typedef struct {
    uint64_t mults, adds;
    uint64_t peak_extra_words;   /* high-water of live temporary words (the graded memory metric) */
    uint64_t total_alloc_words;
    uint64_t word_moves;
    uint64_t classical_calls;
    uint64_t schedule_frames;    /* sum of CostMeter::schedule_calls */
    uint64_t peak_extra_bytes;   /* HBM actually reserved for temporaries (arena high-water) */
    uint64_t n_ops;              /* device operations in the plan */
    uint64_t n_launches;         /* kernel launches issued per execution */
    uint64_t fused_frames;       /* OP_FRAME launches */
    /* algorithmic work (independent of fusion): bytes moved by the schedule's
     * block additions at 8 B per element (3 words per two-term addition, 2 per
     * copy) and flops of the classical leaves (2*m*k*n each) */
    uint64_t add_bytes;
    uint64_t leaf_flops;
    /* bytes the issued addition kernels move (fused frames keep theirs on chip) */
    uint64_t add_bytes_issued;
    /* fused frames: algorithmic bytes of the seven-product GEMM launches (each
     * operand plane / block read once, each product plane written once) and of
     * the whole frames (A, B, beta*C read once, C written once) */
    uint64_t frame_gemm_bytes;
    uint64_t frame_bytes;
    /* fused frames, per kernel: algorithmic bytes of the prep launches (A, B and
     * beta*C_in read once, operand planes written once) and of the combine
     * launches (product planes and packed C_in read once, C written once) */
    uint64_t frame_prep_bytes;
    uint64_t frame_comb_bytes;
    /* classical leaf flops (2*m*k*n) executed inside fused frames */
    uint64_t frame_leaf_flops;
} wm_report;

/* ---- library / context --------------------------------------------------- */
const char* wm_version(void);
const char* wm_last_error(void);
/* Creates a context on `device` for field WM_FIELD_MODP (prime p < 2^16, the
 * Modulus check of ring.hpp:47-53) or WM_FIELD_REAL64 (p ignored).  `stream`
 * is a cudaStream_t (NULL: the context creates its own). */
int wm_ctx_create(int device, uint32_t p, int field, void* stream, wm_ctx** out);
int wm_ctx_destroy(wm_ctx* ctx);
int wm_ctx_sync(wm_ctx* ctx);
/* the context's device, modulus, field and current stream (cudaStream_t) */
int wm_ctx_info(wm_ctx* ctx, int* device, uint32_t* p, int* field, void** stream);
/* issue subsequent work on `stream` (a cudaStream_t of the same device) */
int wm_ctx_set_stream(wm_ctx* ctx, void* stream);
/* options (defaults in brackets; every change drops the cached plans):
 *   "fuse_frames" [1]   fused leaf frames (prep / seven-product GEMM / combine)
 *   "graphs" [1]        capture each plan once into a CUDA graph
 *   "batch_adds" [1], "fuse_adds" [1]   batched / generated fused addition runs
 *   "fold" [1]          operand-producing additions folded into the frame prep
 *   "dead_hosts" [1]    frame planes in dead blocks (plan liveness)
 *   "cin_direct" [1]    accumulating frames: all planes outside C, C_in read by the combine
 *   "wide_plain" [1]    plain frames' GEMM at BN = 64 (c >= 256)
 *   "early_loads" [1]   frame prep / combine read the blocks their lane predecessor does not
 *                       write before griddepcontrol.wait (under its tail and the launch gap)
 *   "micro" [1]         plans of tiny operations as one launch (shared-memory working set)
 *   "arena_words"       (read-only) words of the context's temporary arena = the largest
 *                       schedule peak run so far (one arena shared by every plan)
 *   "dag" [3]           issue lanes (concurrent streams); "epoch" [512] launches per join
 *   "stream_io" [1]     host u32 boundary streamed through the graph (pinned buffers)
 *   "leaf_kernel" [2]   0 = DMMA float64, 1 = tcgen05 int8 limbs, 2 = auto
 *   "direct_frames" [1], "gemm_engine" [0]   GEMM engines (direct-limb frames; TMA / cp.async leaves)
 *   "pdl" [1], "prep_rows" [1], "comb_block" [128]   launch attributes / shapes
 *   "trace" [0]         per-launch timeline (wm_diag_trace)
 *   "subset" [0]        measurement only: 0 all launches, 1 additions only,
 *                       2 leaf products only, 3 fused frames, 4/5/6 frame prep/GEMM/combine */
int wm_ctx_set_option(wm_ctx* ctx, const char* key, int64_t value);
int wm_ctx_get_option(wm_ctx* ctx, const char* key, int64_t* value);

/* ---- primitive operators (ring.hpp) -------------------------------------- */
/* dst <- sa*a + sb*b; dst may alias a or b exactly (block_addsub, ring.hpp:241-278) */
int wm_block_addsub(wm_ctx* ctx, wm_dmat dst, wm_dmat a, wm_dmat b, uint32_t sa, uint32_t sb);
/* dst <- s*src (block_scale_copy, ring.hpp:282-310) */
int wm_block_scale_copy(wm_ctx* ctx, wm_dmat dst, wm_dmat src, uint32_t s);
/* C <- alpha*A*B + beta*C, C disjoint from A and B (classical_mul, ring.hpp:315-384) */
int wm_classical_mul(wm_ctx* ctx, wm_dmat C, wm_dmat A, wm_dmat B, uint32_t alpha, uint32_t beta);

/* dst <- sum_{t<n} coef[t]*src[t], 1 <= n <= 4, one pass; dst may alias a source
 * exactly (new: the S_i / T_i operands and P_i folds of the multi-GPU
 * partition, dist.py; REAL64 reads each coef as a signed int32) */
int wm_lincomb(wm_ctx* ctx, wm_dmat dst, int n, const wm_dmat* src, const uint32_t* coef);

/* ---- drivers -------------------------------------------------------------- */
/* run_variant (drivers.hpp:213-222) / multiply (executor.hpp:240-299):
 * variant is a builtin schedule name (std2 acc3 ip ovl ovl2 ovr aclr accr acc2 acr),
 * "classic", "ipmm" (drivers.hpp:137-158), "ipovmm" (drivers.hpp:52-99),
 * "iprect" (in-place rectangle, k <= min(m,n), new) or "blocked_acc_t<T>[_acc2]"
 * (drivers.hpp:163-209).  A is m x k, B k x n, C m x n (m, k, n from the views). */
int wm_run_variant(wm_ctx* ctx, const char* variant, wm_dmat A, wm_dmat B, wm_dmat C,
                   uint32_t alpha, uint32_t beta, int cutoff, wm_report* report);
/* ipmm (drivers.hpp:137-138) */
int wm_ipmm(wm_ctx* ctx, wm_dmat A, wm_dmat B, wm_dmat C, int cutoff, wm_report* report);
/* REAL64 field: the same dispatch with float64 scalars */
int wm_run_variant_real(wm_ctx* ctx, const char* variant, wm_dmat A, wm_dmat B, wm_dmat C,
                        double alpha, double beta, int cutoff, wm_report* report);
/* End-to-end through host buffers of reference residues (Matrix&, ring.hpp:180-219):
 * uploads A, B (and C when beta != 0), runs, downloads C -- and A / B when the
 * variant's contract may overwrite them, as the reference's Matrix& would show. */
int wm_run_variant_host_u32(wm_ctx* ctx, const char* variant, uint64_t m, uint64_t k, uint64_t n,
                            uint32_t* A, uint32_t* B, uint32_t* C, uint32_t alpha, uint32_t beta,
                            int cutoff, wm_report* report);

/* ---- multi-GPU product partition (wm_dist.cpp) -------------
 * run_variant (drivers.hpp:213-222) with the 7^L products of the top L Winograd
 * levels spread over the ranks of an NCCL communicator (product t on rank
 * t mod G): the root broadcasts A and B, every rank forms its own operands and
 * multiplies them with the single-GPU plan, products return to the root, which
 * folds alpha*coef*P into C (after C <- beta*C).  One process or thread per GPU;
 * NCCL is loaded at run time (libnccl.so.2).  wm_dist_unique_id runs on rank 0
 * and the caller ships the 128 bytes to the other ranks.  On ranks != 0 pass
 * empty A, B, C (their shapes come from the root).  levels 0: chosen by the
 * makespan bound (wm_dist_choose_levels); window: receive buffers on the root. */
typedef struct wm_dist wm_dist;
typedef struct {
    int levels;
    uint64_t products;          /* products this rank computed */
    uint64_t peak_extra_bytes;  /* device bytes this rank held at once (operand copies, */
                                /* operands, products, receive ring, local plan temporaries) */
    uint64_t bytes_sent, bytes_received;
} wm_dist_report;
int wm_dist_unique_id(unsigned char id[128]);
int wm_dist_create(wm_ctx* ctx, int rank, int world, const unsigned char id[128], wm_dist** out);
int wm_dist_destroy(wm_dist* d);
int wm_dist_choose_levels(int world, uint64_t n, int cutoff);
int wm_dist_run_variant(wm_dist* d, const char* variant, wm_dmat A, wm_dmat B, wm_dmat C,
                        uint32_t alpha, uint32_t beta, int cutoff, int levels, int window,
                        wm_dist_report* report);
const char* wm_dist_last_error(void);

/* ---- host-only planning (no device needed) --------------------------------- */
/* Plans `variant` and returns the exact CostReport the reference meter would
 * produce plus the device plan's size; executes nothing. */
int wm_plan_report(const char* variant, int field, uint32_t p, uint64_t m, uint64_t k, uint64_t n,
                   uint32_t alpha, uint32_t beta, int cutoff, int fuse_frames, wm_report* report);
/* expected_costs (models.hpp:202-229); fields of the report beyond word_moves are 0 */
int wm_expected_costs(const char* variant, uint64_t m, uint64_t k, uint64_t n, int cutoff,
                      wm_report* report);
/* Per-schedule frame counts of the last plan on this thread: "name:count,..." */
int wm_plan_schedule_calls(char* out, int len);
/* CostMeter::alloc_log of the last plan on this thread (meter.hpp:15-19, 40-45):
 * "words:depth:slot;..." per metered temporary, in acquisition order; returns
 * the full length (call with out = NULL to size the buffer) */
int wm_plan_alloc_log(char* out, int len);

/* Schedule DSL (schedule.hpp:261-684, executor.hpp:304-342).
 * wm_run_parsed_schedule: run_parsed_schedule -- the schedule in `text` runs at
 *   the top frame, its recursion tags dispatch to builtins.
 * wm_parse_schedule: parse_schedule + render_schedule -- validates `text`
 *   (WM_E_PARSE / WM_E_CONTRACT_VIOLATION), writes the canonical rendering to
 *   out[len] (*needed = its length) and sets *builtin_match when the schedule
 *   equals the builtin of the same name.
 * wm_render_schedule: render_schedule of a builtin. */
int wm_run_parsed_schedule(wm_ctx* ctx, const char* text, wm_dmat A, wm_dmat B, wm_dmat C,
                           uint32_t alpha, uint32_t beta, int cutoff, wm_report* report);
int wm_parse_schedule(const char* text, char* out, int len, int* needed, int* builtin_match);
int wm_render_schedule(const char* name, char* out, int len, int* needed);
/* the CostReport run_parsed_schedule would produce (host only, nothing executes) */
int wm_plan_report_parsed(const char* text, uint32_t p, uint64_t m, uint64_t k, uint64_t n,
                          uint32_t alpha, uint32_t beta, int cutoff, wm_report* report);
/* Matrix files (ring.hpp:386-449): text "rows cols p" + residues, or binary
 * little-endian u64 (rows, cols, p) + u64 residues.  WM_E_IO on a bad header,
 * a truncated body or a non-canonical entry (read_text / read_binary).
 * *_device read into / write from a device matrix of the file's shape. */
int wm_matrix_file_info(const char* path, int binary, uint64_t* rows, uint64_t* cols, uint32_t* p);
int wm_matrix_read_host(const char* path, int binary, uint32_t* out, uint64_t capacity);
int wm_matrix_write_host(const char* path, int binary, uint64_t rows, uint64_t cols, uint32_t p,
                         const uint32_t* data);
int wm_matrix_read_device(wm_ctx* ctx, const char* path, int binary, wm_dmat dst);
int wm_matrix_write_device(wm_ctx* ctx, const char* path, int binary, wm_dmat src);
/* run_parsed_schedule on host uint32 residues (the reference's Matrix&): like
 * wm_run_variant_host_u32 with the schedule given as DSL text. */
int wm_run_parsed_schedule_host_u32(wm_ctx* ctx, const char* text, uint64_t m, uint64_t k,
                                    uint64_t n, uint32_t* A, uint32_t* B, uint32_t* C,
                                    uint32_t alpha, uint32_t beta, int cutoff, wm_report* report);

/* ---- boundary formats ------------------------------------------------------ */
/* device float64 buffers for staging host views (the C++ drop-in's primitives) */
int wm_dev_alloc(wm_ctx* ctx, uint64_t words, double** out);
void wm_dev_free(double* p);
int wm_upload_u32(wm_ctx* ctx, wm_dmat dst, const uint32_t* host, uint64_t host_ld);
int wm_download_u32(wm_ctx* ctx, uint32_t* host, uint64_t host_ld, wm_dmat src);
/* FNV-1a over uint32 residues, row-major (fnv1a64 / Matrix::hash, ring.hpp:107-114,208) */
uint64_t wm_fnv1a64_u32(const uint32_t* data, uint64_t count);
/* seeded device generator, bit-identical to Matrix::fill_random (ring.hpp:202-205);
 * REAL64: x = 2*((next()>>11)*2^-53) - 1 */
int wm_fill_random(wm_ctx* ctx, wm_dmat dst, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif /* WINOMEM_B200_H */
