// Fused leaf frames: one Winograd frame whose seven products are classical
// leaves, run as three launches (wm_frame.cu + the int8 GEMM of wm_i8.cu).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace wm {

struct FrameQuads {
    double* q[4];          // quadrants 11, 12, 21, 22 (float64)
    std::uint64_t ld;      // shared leading dimension (elements)
};

struct FramePrepParams {
    FrameQuads A, B, C;
    std::uint16_t* s_host;  // S1..S4 planes (4 per host row), ld = 4*s_ld
    std::uint64_t s_ld;     // host leading dimension (float64 elements)
    std::uint16_t* t_host;  // T1..T4 planes
    std::uint64_t t_ld;
    std::uint32_t c;        // quadrant size
    std::uint32_t beta;     // accumulate: pack beta*C_in into C11 slots
    double pd, pinv;
};

struct FrameCombParams {
    const std::uint16_t* P[7];  // product planes (mod p)
    std::uint64_t pld[7];       // plane leading dimensions (uint16 elements)
    FrameQuads C;
    std::uint32_t c;
    std::uint32_t alpha, beta;  // beta != 0: packed beta*C_in in the C11 slots
    double pd, pinv;
};

cudaError_t launch_frame_prep(const FramePrepParams& P, cudaStream_t s);
cudaError_t launch_frame_comb(const FrameCombParams& P, cudaStream_t s);

}  // namespace wm
