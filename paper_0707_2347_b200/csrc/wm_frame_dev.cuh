// Device code of the fused leaf frames (wm_frame.cu): operand loading (incl.
// folded parent additions), the limb-plane prep of one row and the U-chain
// combine of one column pair.
#pragma once

#include <cstdint>

#include "wm_apply.cuh"
#include "wm_frame.h"

namespace wm {
namespace fdev {

__device__ __forceinline__ double rmod(double v, double p, double pinv) {
    const double q = floor(v * pinv);
    double r = fma(-q, p, v);
    r = r < 0.0 ? r + p : r;
    return r >= p ? r - p : r;
}
__device__ __forceinline__ double addm(double a, double b, double p) {
    const double v = a + b;
    return v >= p ? v - p : v;
}
__device__ __forceinline__ double subm(double a, double b, double p) {
    const double v = a - b;
    return v < 0.0 ? v + p : v;
}

__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
    const double2 a = *reinterpret_cast<const double2*>(p);
    const double2 b = *reinterpret_cast<const double2*>(p + 2);
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
}

__device__ __forceinline__ uint2 pack(double a, double b, double c, double d) {
    return make_uint2(static_cast<std::uint32_t>(a) | (static_cast<std::uint32_t>(b) << 16),
                      static_cast<std::uint32_t>(c) | (static_cast<std::uint32_t>(d) << 16));
}

// The four quadrant values (row r, columns j, j+1) of a frame operand: loaded
// from its view, or -- folded -- computed from the sources of the parent
// addition(s) that produce it (sa*s0 + sb*s1 < 2^33: exact, one reduction).
__device__ __forceinline__ void load_operand(const FrameQuads& X, const FrameFold& F,
                                             std::uint64_t r, std::uint64_t j, double p,
                                             double pinv, double (&v)[4][2]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (!F.on) {
            const double2 x = *reinterpret_cast<const double2*>(X.q[k] + r * X.ld + j);
            v[k][0] = x.x;
            v[k][1] = x.y;
            continue;
        }
        const double2 a = *reinterpret_cast<const double2*>(F.s0[k] + r * F.ld0 + j);
        double2 b = make_double2(0.0, 0.0);
        if (F.s1[0]) b = *reinterpret_cast<const double2*>(F.s1[k] + r * F.ld1 + j);
        v[k][0] = rmod(fma(F.sa, a.x, F.sb * b.x), p, pinv);
        v[k][1] = rmod(fma(F.sa, a.y, F.sb * b.y), p, pinv);
    }
}

// Store a folded operand into its own view when a later operation reads it.
// Every position is written by the thread that read it (the sources are either
// this view itself, same window, or disjoint from it).
__device__ __forceinline__ void store_operand(const FrameQuads& X, const FrameFold& F,
                                              std::uint64_t r, std::uint64_t j,
                                              const double (&v)[4][2]) {
    if (!F.on || !F.writeback) return;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        *reinterpret_cast<double2*>(X.q[k] + r * X.ld + j) = make_double2(v[k][0], v[k][1]);
}

// Limb-plane prep of row r, columns j, j + 1 (FramePrepParams.limbs): phase 1
// reads everything row r needs (operands, beta*C_in); after a CTA barrier,
// phase 2 writes the operand store-backs, the S/T and raw limb planes and the
// packed beta*C_in -- every byte of it in row r of a host.
struct PrepRegs {
    double av[4][2], bv[4][2], cin[4][2];
};

__device__ __forceinline__ void prep_limbs_load(const FramePrepParams& P, std::uint64_t r,
                                                std::uint64_t j, PrepRegs& R) {
    const double p = P.pd, pinv = P.pinv;
    load_operand(P.A, P.fold[0], r, j, p, pinv, R.av);
    load_operand(P.B, P.fold[1], r, j, p, pinv, R.bv);
    if (P.beta != 0) {
        const double be = static_cast<double>(P.beta);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 x = *reinterpret_cast<const double2*>(P.C.q[k] + r * P.C.ld + j);
            R.cin[k][0] = rmod(be * x.x, p, pinv);
            R.cin[k][1] = rmod(be * x.y, p, pinv);
        }
    }
}

__device__ __forceinline__ void prep_limbs_store(const FramePrepParams& P, std::uint64_t r,
                                                 std::uint64_t j, const PrepRegs& R) {
    const double p = P.pd;
    store_operand(P.A, P.fold[0], r, j, R.av);
    store_operand(P.B, P.fold[1], r, j, R.bv);
    const double(&a11)[2] = R.av[0], (&a12)[2] = R.av[1], (&a21)[2] = R.av[2], (&a22)[2] = R.av[3];
    const double(&b11)[2] = R.bv[0], (&b12)[2] = R.bv[1], (&b21)[2] = R.bv[2], (&b22)[2] = R.bv[3];
    double s[4][2], t[4][2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const double s1 = addm(a21[e], a22[e], p), s2 = subm(s1, a11[e], p);
        s[0][e] = s1;
        s[1][e] = s2;
        s[2][e] = subm(a11[e], a21[e], p);
        s[3][e] = subm(a12[e], s2, p);
        const double t1 = subm(b12[e], b11[e], p), t2 = subm(b22[e], t1, p);
        t[0][e] = t1;
        t[1][e] = t2;
        t[2][e] = subm(b22[e], b12[e], p);
        t[3][e] = subm(t2, b21[e], p);
    }
    const std::uint32_t c = P.c;
    auto put = [&](int pl, const double (&v)[2]) {
        if (!P.plane[pl]) return;
        std::uint8_t* row = static_cast<std::uint8_t*>(P.plane[pl]) + r * P.pld[pl];
        const std::uint32_t x0 = static_cast<std::uint32_t>(v[0]), x1 = static_cast<std::uint32_t>(v[1]);
        *reinterpret_cast<std::uint16_t*>(row + j) = static_cast<std::uint16_t>((x0 >> 8) | (x1 & 0xFF00u));
        *reinterpret_cast<std::uint16_t*>(row + c + j) =
            static_cast<std::uint16_t>((x0 & 255u) | ((x1 & 255u) << 8));
    };
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        put(PL_S1 + k, s[k]);
        put(PL_T1 + k, t[k]);
    }
    put(PL_A11, a11);
    put(PL_A12, a12);
    put(PL_A22, a22);
    put(PL_B11, b11);
    put(PL_B21, b21);
    put(PL_B22, b22);
    if (P.beta != 0) {
        std::uint16_t* c11 = reinterpret_cast<std::uint16_t*>(P.C.q[0]) + 4 * (r * P.C.ld + j);
#pragma unroll
        for (int e = 0; e < 2; ++e)
            reinterpret_cast<uint2*>(c11)[e] = make_uint2(
                static_cast<std::uint32_t>(R.cin[0][e]) | (static_cast<std::uint32_t>(R.cin[1][e]) << 16),
                static_cast<std::uint32_t>(R.cin[2][e]) | (static_cast<std::uint32_t>(R.cin[3][e]) << 16));
    }
}

// U-chain combine of quadrant position (r, j), (r, j + 1): U1 = P1+P2,
// U2 = P1+P6, U3 = U2+P7, U4 = U2+P5, U5 = U4+P3, U6 = U3-P4, U7 = U3+P5 and
// C_ij = alpha*U + beta*C_in.  CG: read the product planes and the packed C_in
// through L2 (written by other CTAs of the same grid).
template <bool CG>
__device__ __forceinline__ void comb_pair(const FrameCombParams& P, std::uint64_t r, std::uint64_t j) {
    const double p = P.pd, pinv = P.pinv;
    double pv[7][2];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        const std::uint32_t* a = reinterpret_cast<const std::uint32_t*>(P.P[k] + r * P.pld[k] + j);
        const std::uint32_t w = CG ? __ldcg(a) : *a;
        pv[k][0] = static_cast<double>(w & 0xFFFFu);
        pv[k][1] = static_cast<double>(w >> 16);
    }
    double cin[2][4];  // [col e][quadrant]
    if (P.beta != 0 && P.cin_f64) {
        // C kept its float64 C_in (the planes live in dead blocks): this thread
        // reads exactly the positions it writes
        const double be = static_cast<double>(P.beta);
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
            const double2 x = *reinterpret_cast<const double2*>(P.C.q[qd] + r * P.C.ld + j);
            cin[0][qd] = rmod(be * x.x, p, pinv);
            cin[1][qd] = rmod(be * x.y, p, pinv);
        }
    } else if (P.beta != 0) {
        const std::uint16_t* c11 = reinterpret_cast<const std::uint16_t*>(P.C.q[0]);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const uint2* a = reinterpret_cast<const uint2*>(c11 + 4 * (r * P.C.ld + j + e));
            const uint2 w = CG ? __ldcg(a) : *a;
            cin[e][0] = static_cast<double>(w.x & 0xFFFFu);
            cin[e][1] = static_cast<double>(w.x >> 16);
            cin[e][2] = static_cast<double>(w.y & 0xFFFFu);
            cin[e][3] = static_cast<double>(w.y >> 16);
        }
    }
    const double al = static_cast<double>(P.alpha);
    double out[4][2];  // [quadrant][col]
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const double p1 = pv[0][e], p2 = pv[1][e], p3 = pv[2][e], p4 = pv[3][e],
                     p5 = pv[4][e], p6 = pv[5][e], p7 = pv[6][e];
        const double u2 = p1 + p6;
        const double u3 = u2 + p7;
        const double u[4] = {p1 + p2, u2 + p5 + p3, u3 + (p - p4), u3 + p5};  // < 4p
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
            double v = rmod(u[qd], p, pinv) * al;
            if (P.beta != 0) v += cin[e][qd];
            out[qd][e] = rmod(v, p, pinv);
        }
    }
#pragma unroll
    for (int qd = 0; qd < 4; ++qd)
        *reinterpret_cast<double2*>(P.C.q[qd] + r * P.C.ld + j) = make_double2(out[qd][0], out[qd][1]);
}

}  // namespace fdev
}  // namespace wm
