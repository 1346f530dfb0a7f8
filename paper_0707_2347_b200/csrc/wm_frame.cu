// Fused leaf frames.  A Winograd frame whose seven products are classical
// leaves (the bottom level of every recursion) runs as three launches instead
// of ~15-24 additions and 7 leaf products issued one after another:
//
//  prep  S1 = A21+A22, S2 = S1-A11, S3 = A11-A21, S4 = A12-S2 and
//        T1 = B12-B11, T2 = B22-T1, T3 = B22-B12, T4 = T2-B21 (Table 1) as uint16
//        residue planes; for accumulating frames beta*C_in is packed as four
//        uint16 per position into the C11 slots;
//  gemm  the seven products P1 = A11 B11, P2 = A12 B21, P3 = S4 B22,
//        P4 = A22 T4, P5 = S1 T1, P6 = S2 T2, P7 = S3 T3 in ONE int8-limb GEMM
//        launch (wm_i8.cu, blockIdx.z = product), written as uint16 planes;
//  comb  U1 = P1+P2, U2 = P1+P6, U3 = U2+P7, U4 = U2+P5, U5 = U4+P3,
//        U6 = U3-P4, U7 = U3+P5 and C_ij = alpha*U + beta*C_in, float64 out.
//
// No memory beyond the schedule's own: a "host" is a c x c float64 block whose
// rows each hold four uint16 plane rows (8c bytes).  S/T planes live in C
// blocks that are dead until the combine (C11, C12 for plain frames; C12, C21
// once beta*C_in is packed into C11), the P planes in the frame's temporaries
// or -- for ip / ovl / ovr, which have fewer -- in the A21 / B12 blocks their
// contract lets them overwrite.  Every prep / comb thread owns a fixed set of
// float64 slots (it reads them before it overwrites them), so the in-place
// packing is race-free.
#include <cstdint>

#include "wm_launch.h"
#include "wm_frame.h"

namespace wm {
namespace {

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

// thread (r, q, h), q < c/4, h in {0,1}: plane columns j = 4q + 2h, +1; the
// float64 slots (r, q + k c/4), k = 0..3, of every host / C block are owned by
// the thread pair (q, 0), (q, 1) of one CTA: both read all they need (A, B and
// beta*C_in) before a barrier, then write their halves of the slots.
__global__ void __launch_bounds__(128) k_frame_prep(const FramePrepParams P) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    WM_PDL_EARLY_M();
    const std::uint32_t c4 = P.c / 4;
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    const bool live = idx < static_cast<std::uint64_t>(P.c) * c4 * 2;
    const std::uint64_t pair = idx >> 1, h = idx & 1;
    const std::uint64_t r = live ? pair / c4 : 0, q = live ? pair - r * c4 : 0;
    const std::uint64_t j = 4 * q + 2 * h;
    const double p = P.pd, pinv = P.pinv;

    double av[4][2], bv[4][2];
    double(&a11)[2] = av[0], (&a12)[2] = av[1], (&a21)[2] = av[2], (&a22)[2] = av[3];
    double(&b11)[2] = bv[0], (&b12)[2] = bv[1], (&b21)[2] = bv[2], (&b22)[2] = bv[3];
    double cin[4][2];  // [k][quadrant 2h, 2h+1]
    if (live) {
        load_operand(P.A, P.fold[0], r, j, p, pinv, av);
        load_operand(P.B, P.fold[1], r, j, p, pinv, bv);
        if (P.beta != 0) {
            const double be = static_cast<double>(P.beta);
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    cin[k][e] = rmod(be * P.C.q[2 * h + e][r * P.C.ld + q + k * c4], p, pinv);
        }
    }
    __syncthreads();  // every owned slot has been read before any is overwritten
    if (!live) return;
    store_operand(P.A, P.fold[0], r, j, av);
    store_operand(P.B, P.fold[1], r, j, bv);
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
    // plane values (r, j..j+1) -> 4 bytes at plane + r*pld + j
    auto put = [&](int pl, const double (&v)[2]) {
        if (P.plane[pl])
            *reinterpret_cast<std::uint32_t*>(static_cast<std::uint16_t*>(P.plane[pl]) + r * P.pld[pl] + j) =
                static_cast<std::uint32_t>(v[0]) | (static_cast<std::uint32_t>(v[1]) << 16);
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
        std::uint16_t* c11 = reinterpret_cast<std::uint16_t*>(P.C.q[0]);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            *reinterpret_cast<std::uint32_t*>(c11 + 4 * (r * P.C.ld + q + k * c4) + 2 * h) =
                static_cast<std::uint32_t>(cin[k][0]) | (static_cast<std::uint32_t>(cin[k][1]) << 16);
    }
    WM_PDL_LATE_M();
}

// Limb-pair variant for the direct-limb GEMM (wm_direct.cu): one CTA per row r,
// thread t owns columns j = 2t, 2t+1.  A plane row holds the high bytes of its
// residues at [0, c) and the low bytes at [c, 2c); every byte a CTA writes lies
// in row r of its host, and every C_in value of row r is read before the
// CTA's barrier, so the in-place packing stays race-free.
__global__ void __launch_bounds__(1024) k_frame_prep_limbs(const FramePrepParams P) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    WM_PDL_EARLY_M();
    const std::uint64_t r = blockIdx.x, j = 2 * threadIdx.x;
    const double p = P.pd, pinv = P.pinv;
    double av[4][2], bv[4][2];
    double(&a11)[2] = av[0], (&a12)[2] = av[1], (&a21)[2] = av[2], (&a22)[2] = av[3];
    double(&b11)[2] = bv[0], (&b12)[2] = bv[1], (&b21)[2] = bv[2], (&b22)[2] = bv[3];
    load_operand(P.A, P.fold[0], r, j, p, pinv, av);
    load_operand(P.B, P.fold[1], r, j, p, pinv, bv);
    auto ld2 = [&](const double* ptr, double (&v)[2]) {
        const double2 x = *reinterpret_cast<const double2*>(ptr);
        v[0] = x.x;
        v[1] = x.y;
    };
    double cin[4][2];  // [quadrant][column]
    if (P.beta != 0) {
        const double be = static_cast<double>(P.beta);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            double v[2];
            ld2(P.C.q[k] + r * P.C.ld + j, v);
            cin[k][0] = rmod(be * v[0], p, pinv);
            cin[k][1] = rmod(be * v[1], p, pinv);
        }
    }
    __syncthreads();  // row r of every host has been read before any of it is overwritten
    store_operand(P.A, P.fold[0], r, j, av);
    store_operand(P.B, P.fold[1], r, j, bv);
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
                static_cast<std::uint32_t>(cin[0][e]) | (static_cast<std::uint32_t>(cin[1][e]) << 16),
                static_cast<std::uint32_t>(cin[2][e]) | (static_cast<std::uint32_t>(cin[3][e]) << 16));
    }
    WM_PDL_LATE_M();
}

// thread (r, 2 consecutive columns j, j+1) of the quadrant
__global__ void __launch_bounds__(128) k_frame_comb(const FrameCombParams P) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    WM_PDL_EARLY_M();
    const std::uint32_t c2 = P.c / 2;
    const std::uint64_t idx = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
    if (idx >= static_cast<std::uint64_t>(P.c) * c2) return;
    const std::uint64_t r = idx / c2, j = 2 * (idx - r * c2);
    const double p = P.pd, pinv = P.pinv;
    double pv[7][2];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        const std::uint32_t w = *reinterpret_cast<const std::uint32_t*>(P.P[k] + r * P.pld[k] + j);
        pv[k][0] = static_cast<double>(w & 0xFFFFu);
        pv[k][1] = static_cast<double>(w >> 16);
    }
    double cin[2][4];  // [col e][quadrant]
    if (P.beta != 0) {
        const std::uint16_t* c11 = reinterpret_cast<const std::uint16_t*>(P.C.q[0]);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const uint2 w = *reinterpret_cast<const uint2*>(c11 + 4 * (r * P.C.ld + j + e));
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
    WM_PDL_LATE_M();
}

template <class K, class Prm>
cudaError_t launch_pdl(K kern, const Prm& P, std::uint64_t threads, cudaStream_t s,
                       unsigned block = 128) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>((threads + block - 1) / block));
    cfg.blockDim = dim3(block);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, P);
}

}  // namespace

cudaError_t launch_frame_prep(const FramePrepParams& P, cudaStream_t s) {
    if (P.limbs) {
        if (P.c > 2048) return cudaErrorInvalidValue;
        return launch_pdl(k_frame_prep_limbs, P, static_cast<std::uint64_t>(P.c) * (P.c / 2), s,
                          P.c / 2);
    }
    return launch_pdl(k_frame_prep, P, static_cast<std::uint64_t>(P.c) * (P.c / 2), s);
}

cudaError_t launch_frame_comb(const FrameCombParams& P, cudaStream_t s) {
    return launch_pdl(k_frame_comb, P, static_cast<std::uint64_t>(P.c) * (P.c / 2), s);
}

bool frame_kernel_available() { return true; }

}  // namespace wm
