// Device launch parameters shared by the runtime and the kernels.  Every launch
// takes its parameters by value (no device-side descriptor tables), so a plan's
// launch sequence can be captured once into a CUDA graph and replayed.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace wm {

// Arithmetic mode of one elementwise item (block_addsub / block_scale_copy).
enum AddMode : std::uint32_t {
    M_ADD = 0,     // a + b
    M_SUB = 1,     // a - b
    M_RSUB = 2,    // b - a
    M_NEGADD = 3,  // -(a + b)
    M_GEN = 4,     // sa*a + sb*b
    M_COPY = 5,    // a
    M_NEG = 6,     // -a
    M_SCALE = 7,   // sa*a
};

struct AddItem {
    double* d;
    const double* a;
    const double* b;
    std::uint64_t ldd, lda, ldb;
    std::uint32_t rows, cols;
    std::uint32_t mode;
    std::uint32_t sa, sb;  // residues (MODP)
    double sad, sbd;       // values (REAL64)
    double ca, cb;         // d = ca*a + cb*b (then reduced, MODP): the branch-free form k_addsub runs
    std::uint32_t blk0;    // first block of this item within the launch
    std::uint32_t vec;     // 2: 16-byte vector path, 1: scalar path
};

constexpr int kMaxAddBatch = 8;
constexpr int kAddThreads = 256;
constexpr int kAddIlp = 4;

struct AddBatch {
    AddItem it[kMaxAddBatch];
    int n;
    std::uint32_t p;
    double pd, pinv;
    unsigned long long* tl;  // measurement timeline slot (nullptr: off)
};

// C <- alpha*A*B + beta*C on one leaf (or one fused frame).
struct MulParams {
    const double* A;
    const double* B;
    double* C;
    std::uint64_t lda, ldb, ldc;
    std::uint32_t m, k, n;
    std::uint32_t alpha, beta;  // residues (MODP)
    double alphad, betad;       // values (REAL64)
    std::uint32_t p;
    double pd, pinv;
    unsigned long long* tl;  // measurement timeline slot (nullptr: off)
};

// dst <- sum_t coef[t] * src[t] (t < n <= kMaxLincomb), one pass (wm_lincomb)
constexpr int kMaxLincomb = 4;
struct LincombParams {
    double* dst;
    const double* src[kMaxLincomb];
    std::uint64_t ldd, lds[kMaxLincomb];
    double coef[kMaxLincomb];  // MODP: residues in [0, p); REAL64: values
    std::uint64_t rows, cols;
    int n;
    double p;
};

// kernels (wm_kernels.cu, wm_dmma.cu, wm_i8.cu, wm_frame.cu)
cudaError_t launch_addsub(const AddBatch& b, bool real, unsigned blocks, cudaStream_t s);
cudaError_t launch_leaf_dmma(const MulParams& P, bool real, cudaStream_t s);
cudaError_t launch_lincomb(const LincombParams& L, bool real, cudaStream_t s);
cudaError_t launch_u32_to_f64(double* dst, std::uint64_t ldd, const std::uint32_t* src,
                              std::uint64_t lds, std::uint64_t rows, std::uint64_t cols,
                              cudaStream_t s, unsigned long long* tl = nullptr);
cudaError_t launch_f64_to_u32(std::uint32_t* dst, std::uint64_t ldd, const double* src,
                              std::uint64_t lds, std::uint64_t rows, std::uint64_t cols,
                              std::uint32_t p, cudaStream_t s, unsigned long long* tl = nullptr);
cudaError_t launch_fill_splitmix(double* dst, std::uint64_t ld, std::uint64_t rows,
                                 std::uint64_t cols, std::uint64_t seed, std::uint32_t p,
                                 bool real, cudaStream_t s);

}  // namespace wm
