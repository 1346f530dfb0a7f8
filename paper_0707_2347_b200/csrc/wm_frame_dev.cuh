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

// canonical residue (an integer < 2^32 held in a float64) -> uint32 and back
// without conversion instructions: 2^52 + x keeps x in its low mantissa word
__device__ __forceinline__ std::uint32_t d2u(double x) {
    return static_cast<std::uint32_t>(__double2loint(x + 4503599627370496.0));
}
__device__ __forceinline__ double u2d(std::uint32_t u) {
    return __hiloint2double(0x43300000, static_cast<int>(u)) - 4503599627370496.0;
}
// residues on the integer pipe: a, b < p < 2^16
__device__ __forceinline__ std::uint32_t addp(std::uint32_t a, std::uint32_t b, std::uint32_t p) {
    const std::uint32_t v = a + b;
    return v >= p ? v - p : v;
}
__device__ __forceinline__ std::uint32_t subp(std::uint32_t a, std::uint32_t b, std::uint32_t p) {
    return a >= b ? a - b : a + p - b;
}
__device__ __forceinline__ std::uint32_t fold4(std::uint32_t v, std::uint32_t p) {  // v < 4p
    v = v >= 2 * p ? v - 2 * p : v;
    return v >= p ? v - p : v;
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
//
// Every load of phase 1 is issued before the first value is used (up to twenty
// 16-byte loads in flight per thread): with the loads interleaved with the
// arithmetic -- what the compiler produces under a 64-register cap -- a prep
// with folded operands waited for memory four times in a row.  Residues live in
// uint32 registers from there on.
struct PrepRegs {
    std::uint32_t av[4][2], bv[4][2], cin[4][2];
};

// the same row with the loads left where the arithmetic needs them (64 registers:
// wide CTAs, c >= 512, where occupancy matters more than loads in flight)
struct PrepRegsF64 {
    double av[4][2], bv[4][2], cin[4][2];
};

struct OperandRaw {
    double2 a[4], b[4];
};

__device__ __forceinline__ std::uint32_t negp(std::uint32_t a, std::uint32_t p) { return a ? p - a : 0u; }

__device__ __forceinline__ void operand_fetch(const FrameQuads& X, const FrameFold& F,
                                              std::uint64_t r, std::uint64_t j, OperandRaw& w) {
    const bool two = F.on && F.s1[0] != nullptr;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double* s0 = F.on ? F.s0[k] + r * F.ld0 : X.q[k] + r * X.ld;
        w.a[k] = *reinterpret_cast<const double2*>(s0 + j);
        if (two) w.b[k] = *reinterpret_cast<const double2*>(F.s1[k] + r * F.ld1 + j);
    }
}

// The operand as integers: loaded, or folded from the parent addition's sources.
// Signs (sa, sb in {1, p - 1}, or no second source) stay on the integer pipe;
// general scalars take one exact float64 reduction (sa*s0 + sb*s1 < 2^33).
__device__ __forceinline__ void operand_finish(const FrameFold& F, const OperandRaw& w, double pd,
                                               double pinv, std::uint32_t (&v)[4][2]) {
    const std::uint32_t p = static_cast<std::uint32_t>(pd);
    if (!F.on) {
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k][0] = d2u(w.a[k].x), v[k][1] = d2u(w.a[k].y);
        return;
    }
    const bool two = F.s1[0] != nullptr;
    const bool a1 = F.sa == 1.0, am = F.sa == pd - 1.0, b1 = F.sb == 1.0, bm = F.sb == pd - 1.0;
    if ((a1 || am) && (!two || b1 || bm)) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const std::uint32_t x = d2u(e ? w.a[k].y : w.a[k].x);
                const std::uint32_t y = two ? d2u(e ? w.b[k].y : w.b[k].x) : 0u;
                v[k][e] = addp(a1 ? x : negp(x, p), !two ? 0u : b1 ? y : negp(y, p), p);
            }
        return;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double bx = two ? w.b[k].x : 0.0, by = two ? w.b[k].y : 0.0;
        v[k][0] = d2u(rmod(fma(F.sa, w.a[k].x, F.sb * bx), pd, pinv));
        v[k][1] = d2u(rmod(fma(F.sa, w.a[k].y, F.sb * by), pd, pinv));
    }
}

__device__ __forceinline__ void store_operand_u32(const FrameQuads& X, const FrameFold& F,
                                                  std::uint64_t r, std::uint64_t j,
                                                  const std::uint32_t (&v)[4][2]) {
    if (!F.on || !F.writeback) return;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        *reinterpret_cast<double2*>(X.q[k] + r * X.ld + j) = make_double2(u2d(v[k][0]), u2d(v[k][1]));
}

struct PrepRaw {
    OperandRaw wa, wb;
    double2 x[4];
};

__device__ __forceinline__ void prep_limbs_fetch(const FramePrepParams& P, std::uint64_t r,
                                                 std::uint64_t j, PrepRaw& W) {
    operand_fetch(P.A, P.fold[0], r, j, W.wa);
    operand_fetch(P.B, P.fold[1], r, j, W.wb);
    if (P.beta != 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) W.x[k] = *reinterpret_cast<const double2*>(P.C.q[k] + r * P.C.ld + j);
    }
}

__device__ __forceinline__ void prep_limbs_finish(const FramePrepParams& P, const PrepRaw& W,
                                                  PrepRegs& R) {
    const double p = P.pd, pinv = P.pinv;
    operand_finish(P.fold[0], W.wa, p, pinv, R.av);
    operand_finish(P.fold[1], W.wb, p, pinv, R.bv);
    if (P.beta != 0) {
        const double be = static_cast<double>(P.beta);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            R.cin[k][0] = d2u(P.beta == 1 ? W.x[k].x : rmod(be * W.x[k].x, p, pinv));
            R.cin[k][1] = d2u(P.beta == 1 ? W.x[k].y : rmod(be * W.x[k].y, p, pinv));
        }
    }
}

// S / T and raw limb planes and the packed beta*C_in of row r, columns j, j + 1
__device__ __forceinline__ void prep_emit(const FramePrepParams& P, std::uint64_t r, std::uint64_t j,
                                          const std::uint32_t (&a)[4][2],
                                          const std::uint32_t (&b)[4][2],
                                          const std::uint32_t (&cin)[4][2]) {
    const std::uint32_t p = static_cast<std::uint32_t>(P.pd);  // a, b: quadrants 11, 12, 21, 22
    // S / T on the integer pipe (the float64 pipe is the narrow one on this part)
    std::uint32_t s[4][2], t[4][2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const std::uint32_t s1 = addp(a[2][e], a[3][e], p), s2 = subp(s1, a[0][e], p);
        s[0][e] = s1;
        s[1][e] = s2;
        s[2][e] = subp(a[0][e], a[2][e], p);
        s[3][e] = subp(a[1][e], s2, p);
        const std::uint32_t t1 = subp(b[1][e], b[0][e], p), t2 = subp(b[3][e], t1, p);
        t[0][e] = t1;
        t[1][e] = t2;
        t[2][e] = subp(b[3][e], b[1][e], p);
        t[3][e] = subp(t2, b[2][e], p);
    }
    const std::uint32_t c = P.c;
    // two residues -> their high bytes / their low bytes, one byte permute each
    auto put = [&](int pl, const std::uint32_t (&v)[2]) {
        if (!P.plane[pl]) return;
        std::uint8_t* row = static_cast<std::uint8_t*>(P.plane[pl]) + r * P.pld[pl];
        *reinterpret_cast<std::uint16_t*>(row + j) =
            static_cast<std::uint16_t>(__byte_perm(v[0], v[1], 0x2251));
        *reinterpret_cast<std::uint16_t*>(row + c + j) =
            static_cast<std::uint16_t>(__byte_perm(v[0], v[1], 0x2240));
    };
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        put(PL_S1 + k, s[k]);
        put(PL_T1 + k, t[k]);
    }
    put(PL_A11, a[0]);
    put(PL_A12, a[1]);
    put(PL_A22, a[3]);
    put(PL_B11, b[0]);
    put(PL_B21, b[2]);
    put(PL_B22, b[3]);
    if (P.beta != 0) {
        std::uint16_t* c11 = reinterpret_cast<std::uint16_t*>(P.C.q[0]) + 4 * (r * P.C.ld + j);
#pragma unroll
        for (int e = 0; e < 2; ++e)
            reinterpret_cast<uint2*>(c11)[e] =
                make_uint2(cin[0][e] | (cin[1][e] << 16), cin[2][e] | (cin[3][e] << 16));
    }
}

__device__ __forceinline__ void prep_limbs_store(const FramePrepParams& P, std::uint64_t r,
                                                 std::uint64_t j, const PrepRegs& R) {
    store_operand_u32(P.A, P.fold[0], r, j, R.av);
    store_operand_u32(P.B, P.fold[1], r, j, R.bv);
    prep_emit(P, r, j, R.av, R.bv, R.cin);
}

__device__ __forceinline__ void prep_limbs_load(const FramePrepParams& P, std::uint64_t r,
                                                std::uint64_t j, PrepRegsF64& R) {
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
                                                 std::uint64_t j, const PrepRegsF64& R) {
    store_operand(P.A, P.fold[0], r, j, R.av);
    store_operand(P.B, P.fold[1], r, j, R.bv);
    std::uint32_t a[4][2], b[4][2], cin[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            a[k][e] = d2u(R.av[k][e]);
            b[k][e] = d2u(R.bv[k][e]);
            cin[k][e] = P.beta != 0 ? d2u(R.cin[k][e]) : 0u;
        }
    prep_emit(P, r, j, a, b, cin);
}

// beta * C_in of quadrant position (r, j), (r, j + 1) as fetched: float64 pairs
// per quadrant (cin_f64) or the packed word
struct CombCin {
    double2 x[4];
    uint4 packed;
};

template <bool CG>
__device__ __forceinline__ void comb_cin_fetch(const FrameCombParams& P, std::uint64_t r,
                                               std::uint64_t j, CombCin& c) {
    if (P.beta == 0) return;
    if (P.cin_f64) {
        // C kept its float64 C_in (the planes live in dead blocks): this thread
        // reads exactly the positions it writes
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) c.x[qd] = *reinterpret_cast<const double2*>(P.C.q[qd] + r * P.C.ld + j);
    } else {
        const std::uint16_t* c11 = reinterpret_cast<const std::uint16_t*>(P.C.q[0]);
        const uint4* a = reinterpret_cast<const uint4*>(c11 + 4 * (r * P.C.ld + j));
        c.packed = CG ? __ldcg(a) : *a;  // positions j and j + 1, four quadrants each
    }
}

// U-chain combine of quadrant position (r, j), (r, j + 1): U1 = P1+P2,
// U2 = P1+P6, U3 = U2+P7, U4 = U2+P5, U5 = U4+P3, U6 = U3-P4, U7 = U3+P5 and
// C_ij = alpha*U + beta*C_in, on the integer pipe.  CG: read the product planes
// through L2 (written by other CTAs of the same grid).
template <bool CG>
__device__ __forceinline__ void comb_pair(const FrameCombParams& P, std::uint64_t r, std::uint64_t j,
                                          const CombCin& c) {
    const double pd = P.pd, pinv = P.pinv;
    const std::uint32_t p = static_cast<std::uint32_t>(pd);
    std::uint32_t w[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        const std::uint32_t* a = reinterpret_cast<const std::uint32_t*>(P.P[k] + r * P.pld[k] + j);
        w[k] = CG ? __ldcg(a) : *a;
    }
    std::uint32_t cin[2][4];  // [col e][quadrant], beta * C_in mod p
    if (P.beta != 0 && P.cin_f64) {
        const double be = static_cast<double>(P.beta);
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
            cin[0][qd] = d2u(P.beta == 1 ? c.x[qd].x : rmod(be * c.x[qd].x, pd, pinv));
            cin[1][qd] = d2u(P.beta == 1 ? c.x[qd].y : rmod(be * c.x[qd].y, pd, pinv));
        }
    } else if (P.beta != 0) {
        const uint4 v = c.packed;
        cin[0][0] = v.x & 0xFFFFu, cin[0][1] = v.x >> 16, cin[0][2] = v.y & 0xFFFFu, cin[0][3] = v.y >> 16;
        cin[1][0] = v.z & 0xFFFFu, cin[1][1] = v.z >> 16, cin[1][2] = v.w & 0xFFFFu, cin[1][3] = v.w >> 16;
    }
    double out[4][2];  // [quadrant][col]
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        std::uint32_t pv[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) pv[k] = e ? w[k] >> 16 : w[k] & 0xFFFFu;
        const std::uint32_t u2 = pv[0] + pv[5], u3 = u2 + pv[6];
        const std::uint32_t u[4] = {pv[0] + pv[1], u2 + pv[4] + pv[2], u3 + (p - pv[3]),
                                    u3 + pv[4]};  // < 4p
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
            std::uint32_t v = fold4(u[qd], p);
            if (P.alpha != 1)  // alpha v < 2^32: exact in float64
                v = d2u(rmod(static_cast<double>(P.alpha) * u2d(v), pd, pinv));
            if (P.beta != 0) v = addp(v, cin[e][qd], p);
            out[qd][e] = u2d(v);
        }
    }
#pragma unroll
    for (int qd = 0; qd < 4; ++qd)
        *reinterpret_cast<double2*>(P.C.q[qd] + r * P.C.ld + j) = make_double2(out[qd][0], out[qd][1]);
}

}  // namespace fdev
}  // namespace wm
