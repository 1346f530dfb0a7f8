// Micro-plan executor (wm_micro.cu): a plan of tiny operations in one launch.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "wm_device.h"

namespace wm {

// One planned operation, pointers resolved at plan time (the plan cache is
// keyed on the operands' addresses).
struct MicroOp {
    enum Kind : std::uint32_t { ADD = 0, MUL = 1 };
    double* d;
    const double* a;
    const double* b;
    std::uint32_t ldd, lda, ldb;
    std::uint32_t rows, cols, k;  // ADD: d is rows x cols; MUL: C rows x cols, inner k
    std::uint32_t kind : 8;
    std::uint32_t csh : 8;        // log2(cols) when cols is a power of two, else 0xFF
    std::uint32_t : 16;
    std::uint32_t mode;           // ADD: AddMode (wm_device.h)
    std::uint32_t sa, sb;         // residues: ADD scalars, MUL alpha / beta
};
static_assert(sizeof(MicroOp) % 8 == 0, "descriptors are staged as 8-byte words");

// Plans whose every operation is at most this small run as one micro launch;
// one warp walks plans whose operations are all below the "small" bounds.
constexpr std::uint64_t kMicroMaxWords = 4096;        // per addition / leaf output
constexpr std::uint64_t kMicroMaxLeafVolume = 1 << 18;  // m * k * n per leaf
constexpr std::uint64_t kMicroSmallWords = 1024;
constexpr std::uint64_t kMicroSmallLeafVolume = 4096;

// The working set staged in shared memory (nregions == 0: operate on global
// memory): region r lives at image words [offset, offset + rows * ld).
struct MicroRegion {
    double* global;
    std::uint64_t rows, cols, ld, offset;
    int load, store;
};
struct MicroImage {
    int nregions;
    MicroRegion region[4];  // A, B, C, temporaries
    std::uint64_t words;
};

std::size_t micro_smem_limit();  // bytes available for the image
cudaError_t launch_micro(const MicroOp* ops, std::uint32_t n, const MicroImage& img, bool small,
                         std::uint32_t p, cudaStream_t s);

}  // namespace wm
