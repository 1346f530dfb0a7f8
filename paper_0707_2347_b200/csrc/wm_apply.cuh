// Residue arithmetic of one block-addition element (block_addsub,
// ring.hpp:241-278) shared by the addition kernels, the generated fused runs
// and the frame combine that absorbs a following run.  Operands are canonical
// (< 2^16): a +/- b needs one conditional correction, sa*a + sb*b (< 2^33) one
// floor-based reduction.
#pragma once

#include <cstdint>

#include "wm_device.h"
#include "wm_fused_gen.cuh"

namespace wm {

template <bool REAL>
__device__ __forceinline__ double apply(double a, double b, std::uint32_t mode, double sa,
                                        double sb, double p, double pinv) {
    if (REAL) {
        switch (mode) {
            case M_ADD: return a + b;
            case M_SUB: return a - b;
            case M_RSUB: return b - a;
            case M_NEGADD: return -(a + b);
            case M_GEN: return fma(sa, a, sb * b);
            case M_COPY: return a;
            case M_NEG: return -a;
            default: return sa * a;
        }
    }
    double v;
    switch (mode) {
        case M_ADD: v = a + b; return v >= p ? v - p : v;
        case M_SUB: v = a - b; return v < 0.0 ? v + p : v;
        case M_RSUB: v = b - a; return v < 0.0 ? v + p : v;
        case M_NEGADD: v = a + b; v = v >= p ? v - p : v; return v != 0.0 ? p - v : 0.0;
        case M_COPY: return a;
        case M_NEG: return a != 0.0 ? p - a : 0.0;
        case M_GEN: v = fma(sa, a, sb * b); break;
        default: v = sa * a; break;
    }
    // v is an exact non-negative integer < 2^53
    const double q = floor(v * pinv);
    double r = fma(-q, p, v);
    r = r < 0.0 ? r + p : r;
    return r >= p ? r - p : r;
}

namespace fused {
// canonical representative in [0, p) of an exact integer value
template <bool REAL>
__device__ __forceinline__ double canon(double v, double p, double pinv) {
    if (REAL) return v;
    double r = fma(-floor(v * pinv), p, v);
    r = r < 0.0 ? r + p : r;
    return r >= p ? r - p : r;
}
}  // namespace fused

}  // namespace wm
