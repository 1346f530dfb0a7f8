// Fused leaf frames: one Winograd frame whose seven products are classical
// leaves, run as three launches (wm_frame.cu + the int8 GEMM of wm_i8.cu).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "wm_fused_gen.cuh"

namespace wm {

struct FrameQuads {
    double* q[4];          // quadrants 11, 12, 21, 22 (float64)
    std::uint64_t ld;      // shared leading dimension (elements)
};

// residue planes written by the prep launch, in this order
enum FramePlane { PL_S1, PL_S2, PL_S3, PL_S4, PL_T1, PL_T2, PL_T3, PL_T4,
                  PL_A11, PL_A12, PL_A22, PL_B11, PL_B21, PL_B22, PL_COUNT };

// A frame operand folded from the parent schedule's addition(s) that produce it
// (lowering pass, wm_runtime.cu): operand = sa*s0 + sb*s1 mod p, computed by the
// prep from the sources; `writeback` also stores it into the operand's own view
// when a later operation still reads it.
struct FrameFold {
    const double* s0[4];   // quadrants of the first source
    const double* s1[4];   // second source (nullptr: one-term copy / scaling)
    std::uint64_t ld0, ld1;
    double sa, sb;         // residues in [0, p)
    std::uint32_t on, writeback;
};

struct FramePrepParams {
    FrameQuads A, B, C;
    FrameFold fold[2];               // 0: A, 1: B
    void* plane[PL_COUNT];           // nullptr: not materialised (raw blocks only)
    std::uint64_t pld[PL_COUNT];     // plane row pitch: uint16 elements, or bytes if limbs
    std::uint32_t limbs;             // 1: limb-pair planes (hi bytes [0,c), lo [c,2c) per row)
    std::uint32_t c;                 // quadrant size
    std::uint32_t beta;              // accumulate: pack beta*C_in into C11 slots
    double pd, pinv;
    unsigned long long* tl;          // measurement timeline slot (nullptr: off)
    // the launch this one programmatically depends on (its predecessor on the
    // lane) writes nothing this prep reads: the loads go out BEFORE
    // griddepcontrol.wait, under the predecessor's tail and the launch gap
    std::uint32_t early;
};

struct FrameCombParams {
    const std::uint16_t* P[7];  // product planes (mod p)
    std::uint64_t pld[7];       // plane leading dimensions (uint16 elements)
    FrameQuads C;
    std::uint32_t c;
    std::uint32_t alpha, beta;  // beta != 0: packed beta*C_in in the C11 slots
    double pd, pinv;
    unsigned long long* tl;     // measurement timeline slot (nullptr: off)
    std::uint32_t cin_f64;      // beta != 0: C_in read as float64 from C (no packing)
    std::uint32_t early;        // C_in is not written by the lane predecessor: read it before the wait
};

cudaError_t launch_frame_prep(const FramePrepParams& P, cudaStream_t s);

cudaError_t launch_frame_comb(const FrameCombParams& P, cudaStream_t s);

}  // namespace wm
