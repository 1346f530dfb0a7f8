// Generalised exact int8-limb GEMM launch parameters (wm_i8.cu): several
// independent products of one shape per launch, float64 or uint16 residue
// operands, float64 (alpha/beta) or uint16 outputs.
#pragma once

#include <cstdint>

#include <cuda.h>
#include <cuda_runtime.h>

namespace wm {

constexpr int kMaxProducts = 7;

struct GemmSrc {
    const void* p;
    std::uint64_t ld;    // in elements (fmt 2: row pitch in bytes)
    std::uint32_t fmt;   // 0 float64 residues, 1 uint16 residues, 2 limb-plane pair
    std::uint64_t part;  // fmt 2: byte offset of the low-limb plane from the high one
};

struct GemmParams {
    GemmSrc a[kMaxProducts], b[kMaxProducts], c[kMaxProducts];
    std::uint32_t m, n, k;   // shape of every product
    std::uint32_t nprod;     // products in this launch
    std::uint32_t tiles_m;   // m / 128
    std::uint32_t alpha, beta;  // float64 outputs only
    double pd, pinv;
    unsigned long long* trace;  // diagnostics: per-CTA phase timestamps (nullptr: off)
    unsigned long long* tl;     // measurement timeline slot (nullptr: off)
};

// TMA operand maps (one pair per product), encoded on the host at lowering time
struct TmaMaps {
    CUtensorMap a[kMaxProducts], b[kMaxProducts];
};

bool gemm_i8_supported(const GemmParams& P);
// (BN, K split) for a product set: aim for >= ~100 CTAs on the 148 SMs
void gemm_choose(const GemmParams& P, int* bn, int* split);
cudaError_t launch_gemm_i8(const GemmParams& P, cudaStream_t s);             // cp.async engine
cudaError_t gemm_tma_init();
bool gemm_tma_encode(const GemmParams& P, int bn, TmaMaps& M);
cudaError_t launch_gemm_tma(const GemmParams& P, const TmaMaps& M, int bn, int split,
                            cudaStream_t s);                                  // TMA engine

// Direct-limb engine (wm_direct.cu): operands are limb-plane pairs (fmt 2; B may
// also be float64), outputs uint16 planes, K a multiple of 128, no K split.
cudaError_t gemm_direct_init();
bool gemm_direct_supported(const GemmParams& P, int bn);
bool gemm_direct_encode(const GemmParams& P, int bn, TmaMaps& M);
int gemm_direct_choose(const GemmParams& P);
cudaError_t launch_gemm_direct(const GemmParams& P, const TmaMaps& M, int bn, cudaStream_t s);

}  // namespace wm
